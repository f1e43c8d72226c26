"""A/B of small-graph latency on one box: per-graph build + init + 4 iterations + destroy for 400 of
f4's ER graphs, and the c1 step, with the library at <pkgroot> (argv[1]; e.g. the round-1 build)."""
import json
import os
import sys
import time

pkgroot = os.path.abspath(sys.argv[1])
sys.path.insert(0, pkgroot)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2102_02302_b200 as cl  # noqa: E402
import gen  # noqa: E402

assert os.path.dirname(cl.LIB_PATH).startswith(pkgroot), cl.LIB_PATH
rng = np.random.default_rng(0)
gs = []
for i in range(400):
    n = int(np.exp(rng.uniform(np.log(50), np.log(5000))))
    g = gen.er(n, 4 * n, seed=100 + i)
    gs.append((torch.from_numpy(g.src).cuda(), torch.from_numpy(g.dst).cuda(), n))
c1 = gen.config("c1")
c1s, c1d = torch.from_numpy(c1.src).cuda(), torch.from_numpy(c1.dst).cuda()
s = torch.cuda.Stream()
out = {"lib": cl.LIB_PATH}
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for xs, xd, xn in gs:
        G = cl.cleora_build(xs, xd, None, xn, False, device=0, stream=s.cuda_stream)
        cl.cleora_init(G, 128, 0)
        cl.cleora_iterate(G, 4)
        G.close()
    torch.cuda.synchronize()
    out[f"f4_per_graph_ms_{rep}"] = (time.perf_counter() - t0) * 1e3 / len(gs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        G = cl.cleora_build(c1s, c1d, None, c1.n, False, device=0, stream=s.cuda_stream)
        cl.cleora_init(G, 128, 0)
        cl.cleora_iterate(G, 4)
        G.close()
    torch.cuda.synchronize()
    out[f"c1_step_ms_{rep}"] = (time.perf_counter() - t0) * 1e3 / 200
print(json.dumps(out))
