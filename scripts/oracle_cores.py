"""The CPU oracle's throughput on one core and on all host cores (SURVEY §8(d) "oracle timing": the
1-core figure for c1 and c2 beside the all-core one).  Each measurement runs in a child process so
OMP_NUM_THREADS takes effect.  Test infrastructure only (calls oracle/).
Usage: python scripts/oracle_cores.py [configs...]   (default c1 c2)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys, time
sys.path.insert(0, %r)
import gen, oracle
g = gen.config(%r)
t0 = time.perf_counter(); M = oracle.build_from(g); t1 = time.perf_counter()
T = oracle.hash_init(g.n, g.d, 0); t2 = time.perf_counter()
for _ in range(g.iters):
    T = oracle.step(M, T)
t3 = time.perf_counter()
nnz = int(M.row_ptr[-1])
print(json.dumps({"config": %r, "threads": oracle.num_threads(), "build_s": t1 - t0, "init_s": t2 - t1,
                  "iterations_s": t3 - t2, "nnz": nnz, "d": g.d, "iters": g.iters,
                  "nnz_d_per_s": nnz * g.d * g.iters / (t3 - t0),
                  "iter_nnz_d_per_s": nnz * g.d * g.iters / (t3 - t2)}))
'''
for cfg in (sys.argv[1:] or ["c1", "c2"]):
    for threads in ("1", None):
        env = dict(os.environ)
        if threads:
            env["OMP_NUM_THREADS"] = threads
        else:
            env.pop("OMP_NUM_THREADS", None)
        out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg, cfg)], env=env, capture_output=True,
                             text=True, timeout=1800)
        print(out.stdout.strip() or out.stderr.strip()[-300:], flush=True)
