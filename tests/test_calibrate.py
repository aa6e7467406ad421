"""calibrate.py recovers a HardwareSpec from a trace: fed the simulator's own
trace (simulator.py:364-399, same leading columns as krt_trace_csv) of a plan
made under a known spec, it must return that spec's per-kind MAC/s and its
backward_multiplier."""
import pytest

from paper_2008_11421_b200 import calibrate
from paper_2008_11421_b200 import workloads as W


@pytest.mark.parametrize("name", ["resnet200_b3072", "gpt_small_bf16", "resnet1001_2048_b2"])
def test_from_simulated_trace_recovers_the_spec(name):
    rec = W.load(name)
    b = W.bundle_for(rec)
    hw = dict(l.split(" = ") for l in rec["hardware"].strip().splitlines())
    sim = b.simulate()
    tr = calibrate.from_trace(b, sim["csv"])
    eff = {k.split(".", 1)[1]: float(v) for k, v in hw.items() if k.startswith("efficiency.")}
    rate = float(hw["compute_rate"])
    for kind, r in tr["mac_per_s_by_kind"].items():
        assert r == pytest.approx(rate * eff.get(kind, 1.0), rel=1e-6), kind
    assert tr["backward_multiplier"] == pytest.approx(float(hw["backward_multiplier"]), rel=1e-6)


def test_hw_text_round_trips_through_the_engine():
    rec = W.load("resnet200_b3072")
    cal = {"near_mem_bw": 6.5e12, "interconnect_bw": 49.8e9, "compute_rate": 7.1e14,
           "host_update_rate": 1.1e9, "backward_multiplier": 2.3, "efficiency": {"Conv": 0.41, "FullyConnected": 0.2}}
    text = calibrate.hw_text(calibrate.capacity_of(rec["hardware"]), cal)
    b = W.bundle_for(dict(rec, hardware=text))
    c = b.costs()["blocks"][0]
    assert c["bwd_seconds"] == pytest.approx(2.3 * c["fwd_seconds"], rel=1e-12)
    assert "efficiency.Conv = 0.41" in text


def test_host_update_rate_runs():
    r = calibrate.host_update_rate(n=1 << 20, threads=2, reps=1)
    assert r["elements_per_s"] > 0 and r["threads"] == 2
