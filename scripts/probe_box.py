"""One-off probe of the GPU box: host RAM/cores, pinned-alloc cost, PCIe H2D/D2H/duplex
bandwidth and a conv throughput sample.  Output: JSON on stdout."""
import json, os, subprocess, time
import torch

out = {}
out["nproc"] = os.cpu_count()
try:
    out["affinity"] = len(os.sched_getaffinity(0))
except Exception:
    pass
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
out["cpu"] = [l for l in open("/proc/cpuinfo").read().splitlines() if l.startswith("model name")][:1]
out["flags_avx512"] = "avx512f" in open("/proc/cpuinfo").read()
dev = torch.device("cuda:0")
torch.cuda.init()
out["gpu"] = torch.cuda.get_device_name(0)
free, total = torch.cuda.mem_get_info()
out["hbm_free_total"] = [free, total]

def pinned(nbytes):
    t0 = time.time()
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    return h, time.time() - t0

res = {}
for gb in (1, 8, 32):
    h, dt = pinned(gb << 30)
    res[f"pin_{gb}GB_s"] = dt
    del h
out["pin"] = res

n = 2 << 30
h_src, _ = pinned(n)
h_dst, _ = pinned(n)
d = torch.empty(n, dtype=torch.uint8, device=dev)
d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()

def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.time()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.time() - t0) / reps

h2d = timeit(lambda: d.copy_(h_src, non_blocking=True))
d2h = timeit(lambda: h_dst.copy_(d2, non_blocking=True))
def duplex():
    with torch.cuda.stream(s1):
        d.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d2, non_blocking=True)
dup = timeit(duplex)
out["pcie_GBps"] = {"h2d": n / h2d / 1e9, "d2h": n / d2h / 1e9, "duplex_each": n / dup / 1e9}
# chunked 64MB copies
m = 64 << 20
def chunked_h2d():
    for off in range(0, n, m):
        d[off:off+m].copy_(h_src[off:off+m], non_blocking=True)
out["pcie_GBps"]["h2d_64MB_chunks"] = n / timeit(chunked_h2d) / 1e9
del d, d2, h_src, h_dst

# conv sample: stage-3 bottleneck 3x3 conv bf16 channels_last
x = torch.randn(256, 256, 14, 14, device=dev, dtype=torch.bfloat16).to(memory_format=torch.channels_last)
w = torch.randn(256, 256, 3, 3, device=dev, dtype=torch.bfloat16).to(memory_format=torch.channels_last)
f = lambda: torch.nn.functional.conv2d(x, w, padding=1)
t = timeit(f, 20)
out["conv3x3_14x14x256_b256_TFLOPs"] = 2 * 256 * 14 * 14 * 256 * 256 * 9 / t / 1e12
x = torch.randn(256, 512, 28, 28, device=dev, dtype=torch.bfloat16).to(memory_format=torch.channels_last)
w = torch.randn(128, 512, 1, 1, device=dev, dtype=torch.bfloat16).to(memory_format=torch.channels_last)
t = timeit(lambda: torch.nn.functional.conv2d(x, w), 20)
out["conv1x1_28x28_512to128_b256_TFLOPs"] = 2 * 256 * 28 * 28 * 128 * 512 / t / 1e12
a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
t = timeit(lambda: a @ a, 10)
out["mm8192_TFLOPs"] = 2 * 8192**3 / t / 1e12
try:
    out["nvsmi"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[-1500:]
except Exception as e:
    out["nvsmi"] = str(e)
print(json.dumps(out, indent=1))
