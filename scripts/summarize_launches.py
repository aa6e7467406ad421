"""Group an ncu launch list (`--metrics gpu__time_duration.sum --csv`) by
kernel family and print the markdown share table used in profiles/.

    python scripts/summarize_launches.py gpurun_out/launches.csv
"""
import csv
import re
import sys
from collections import defaultdict


def family(name):
    if name.startswith("void krt::") or "krt::" in name[:40]:
        m = re.search(r"krt::(?:<unnamed>::)?(\w+)", name)
        return "krt::" + (m.group(1) if m else name[:40])
    if "cutlass3x_sm100" in name or "cutlass3x" in name:
        kind = "wgrad" if "wgrad" in name else "dgrad" if "dgrad" in name else "fprop"
        return f"cuDNN conv {kind} (cutlass3x sm100 tcgen05)"
    if "nvjet" in name:
        return "nvjet / cuBLASLt GEMM"
    if "max_pool" in name:
        return "aten: " + re.search(r"(max_pool\w*)", name).group(1)
    return "aten/other: " + name[:60]


def main(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    unit_i = h.index("Metric Unit") if "Metric Unit" in h else None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[unit_i] if unit_i is not None else "ns"
        ms = v * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        f = family(r[ki])
        tot[f] += ms
        cnt[f] += 1
    total = sum(tot.values())
    print("| share | ms | launches | kernel family |\n|---:|---:|---:|---|")
    for f, ms in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| {ms / total * 100:.1f}% | {ms:.2f} | {cnt[f]} | {f} |")
    own = sum(ms for f, ms in tot.items() if f.startswith("krt::"))
    print(f"\nTotal kernel time in window: {total:.1f} ms over {sum(cnt.values())} launches. "
          f"Own kernels (`krt::`): **{own / total * 100:.1f}%** of kernel time.")


if __name__ == "__main__":
    main(sys.argv[1])
