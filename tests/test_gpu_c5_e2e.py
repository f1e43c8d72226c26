"""OPT-IN (CLEORA_C5_E2E=1): c5 END TO END against the whole-graph oracle.

tests/test_gpu_c5.py checks c5 step by step (the oracle's step on the GPU's own T_{i-1}); this
test checks the final embedding T_4 itself, as the BASELINE north star states the target: the
oracle builds the whole M (2.84B entries: a qsort of 68 GB of entries, ~15 min on 16 host cores)
and runs Algorithm 1 for all 41.65M rows in fp64, once; the GPU's T_4 must match
on a sample of rows -- random rows, the largest hubs, rows next to hubs and isolated rows -- within
max|d| <= 1e-5, cosine >= 0.99999, zero rows identical.

Two subprocesses keep the host memory within the GPU box's (196 GB): the GPU run writes the sampled
rows of T_4 to a file and exits; the oracle run then needs ~140 GB (M with its fp64 weights and two
T copies).  About 25 minutes in all.
"""
import json
import os
import subprocess
import sys
import tempfile

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

GPU_PHASE = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[2])
import gen, paper_2102_02302_b200 as cl
g = gen.config("c5")
n = g.n
rng = np.random.default_rng(55)
deg = np.bincount(g.src, minlength=n) + np.bincount(g.dst, minlength=n)
hubs = np.argsort(deg, kind="stable")[-16:]
nbr = np.unique(np.concatenate([g.dst[g.src == hubs[-1]][:64], g.src[g.dst == hubs[-1]][:64]]))
iso = np.flatnonzero(deg == 0)
S = np.unique(np.concatenate([rng.choice(n, 3000, replace=False), hubs, nbr,
                              rng.choice(iso, min(100, iso.size), replace=False)])).astype(np.int64)
G = cl.cleora_build(g.src, g.dst, None, n, False, device=0)
del g
cl.cleora_init(G, 256, 0)
cl.cleora_iterate(G, 4)
T = np.stack([cl.cleora_fetch(G, int(r), int(r) + 1)[0] for r in S])
G.close()
np.savez(sys.argv[1], S=S, T=T)
'''

ORACLE_PHASE = r'''
import json, sys, time, numpy as np
sys.path.insert(0, sys.argv[2])
import gen, oracle
z = np.load(sys.argv[1])
S, T = z["S"], z["T"].astype(np.float64)
g = gen.config("c5")
t0 = time.time()
M = oracle.build_csr(g.src, g.dst, None, g.n, False)
del g
t1 = time.time()
R = oracle.embed(M, 256, 0, 4)
t2 = time.time()
W = R[S].astype(np.float64)
del R
zero_ok = bool(np.array_equal(~T.any(1), ~W.any(1)))
nz = W.any(1)
err = float(np.abs(T - W).max())
cos = (T[nz] * W[nz]).sum(1) / (np.linalg.norm(T[nz], axis=1) * np.linalg.norm(W[nz], axis=1))
print(json.dumps({"rows": int(S.size), "nonzero_rows": int(nz.sum()), "max_abs": err, "min_cos": float(cos.min()),
                  "zero_rows_identical": zero_ok, "oracle_build_s": t1 - t0, "oracle_embed_s": t2 - t1,
                  "oracle_threads": oracle.num_threads(), "nnz": int(M.nnz)}))
'''


@pytest.mark.skipif(not os.environ.get("CLEORA_C5_E2E"), reason="opt-in: set CLEORA_C5_E2E=1 (~25 min, ~140 GB host)")
def test_c5_end_to_end_sampled_rows():
    import torch
    if not torch.cuda.is_available() or torch.cuda.get_device_properties(0).total_memory < 150e9:
        pytest.skip("needs a B200")
    with tempfile.TemporaryDirectory() as td:
        f = os.path.join(td, "t4.npz")
        subprocess.run([sys.executable, "-c", GPU_PHASE, f, ROOT], check=True, cwd=ROOT, timeout=3600)
        out = subprocess.run([sys.executable, "-c", ORACLE_PHASE, f, ROOT], check=True, cwd=ROOT, timeout=7200,
                             capture_output=True, text=True)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    print("c5 end to end:", res)
    assert res["nnz"] == 2_837_874_790
    assert res["zero_rows_identical"]
    assert res["max_abs"] <= 1e-5, res
    assert res["min_cos"] >= 0.99999, res
