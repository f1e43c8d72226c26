"""bench.py pieces that need no GPU: the --impl reference arm (the CPU oracle timed on a bounded
sample of the workload) prints the contract's JSON line, and the CPU baseline helpers run."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_the_contract_line():
    env = dict(os.environ, CLEORA_REF_STEP_S="0.2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, cwd=ROOT, env=env,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"] == "c1"


def test_cpu_baseline_helpers():
    sys.path.insert(0, ROOT)
    import bench
    import gen
    g = gen.config("c1")
    holder = []
    v, det = bench.cpu_baseline(g, holder, g.d, g.iters, budget_s=5.0)
    assert v > 0 and det["full"] and det["rows"] == g.n
    v2, det2 = bench._cpu_baseline_block(g, [], g.d, g.iters, 1.0)
    assert v2 > 0 and det2["block"] and 0 < det2["rows"] <= g.n
    cs = bench.ClockSampler(0)            # no NVML device here: an empty summary, no exception
    s = cs.summary()
    assert s["samples"] == 0 and s["sm_mhz"] is None


def test_e2e_schedule_by_memory():
    """e2e overlap schedule from the handle's footprint (B200: 180 GB): c2 (~14 GB per handle) keeps
    two whole handles, c5 (~110 GB, T 42.7 GB) trims the previous one to its result, and a handle
    that leaves no room for another T runs serially."""
    sys.path.insert(0, ROOT)
    import bench
    hbm = 180 * 10**9
    assert bench.e2e_schedule(14 * 10**9, 4.65 * 10**9, hbm) == "full"
    assert bench.e2e_schedule(110 * 10**9, 42.7 * 10**9, hbm) == "trim"
    assert bench.e2e_schedule(150 * 10**9, 42.7 * 10**9, hbm) is None
