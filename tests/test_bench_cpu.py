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


def test_gpus_flag_launches_that_many_ranks():
    """``bench.py --gpus 2`` without torchrun re-launches itself with 2 ranks (torch.distributed.run);
    --dry-launch makes every rank print its rank / world and exit before any GPU work."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-launch"],
                         capture_output=True, text=True, cwd=ROOT, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 and d["dry_launch"] for d in lines)


def test_gpus_flag_must_match_world_size():
    """Under a launcher, --gpus must equal WORLD_SIZE (a mismatch would mis-report n_gpus)."""
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-launch"],
                         capture_output=True, text=True, cwd=ROOT, env=env, timeout=120)
    assert out.returncode == 2 and "WORLD_SIZE=3" in out.stderr
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--dry-launch"],
                         capture_output=True, text=True, cwd=ROOT, env=env, timeout=120)
    assert out.returncode == 0 and json.loads(out.stdout.strip().splitlines()[-1])["world"] == 1


def test_config_l2_statement_depends_on_size():
    sys.path.insert(0, ROOT)
    import bench
    import gen
    c1 = bench.config_dict(gen.config("c1"), 1)
    assert "flushed" in c1["l2"] and "larger than L2" not in c1["l2"]
    import numpy as np
    g4 = gen.EdgeList("c4", 4847571, np.zeros(1, np.int32), np.zeros(1, np.int32), None, True, d=1024, iters=4)
    assert "larger than L2" in bench.config_dict(g4, 1)["l2"]
