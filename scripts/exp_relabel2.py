"""EXPERIMENT: SpMM time per launch with the graph's ids as generated vs relabelled by degree (hot
nodes first) -- does id locality of the hot set matter?  Usage: python exp_relabel2.py cfg"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

cfg = sys.argv[1]
g = gen.config(cfg)
deg = np.bincount(g.dst, minlength=g.n) + (0 if g.directed else np.bincount(g.src, minlength=g.n))
order = np.argsort(-deg, kind="stable")
new_of_old = np.empty(g.n, np.int32)
new_of_old[order] = np.arange(g.n, dtype=np.int32)
for mode in ("orig", "relabel"):
    src, dst = (g.src, g.dst) if mode == "orig" else (new_of_old[g.src], new_of_old[g.dst])
    w = None if g.w is None else torch.from_numpy(g.w).cuda()
    G = cl.cleora_build(torch.from_numpy(np.ascontiguousarray(src)).cuda(), torch.from_numpy(np.ascontiguousarray(dst)).cuda(),
                        w, g.n, g.directed, timing=True)
    cl.cleora_init(G, g.d, 0)
    cl.cleora_iterate(G, 4)
    st = cl.cleora_stats(G)
    print(cfg, mode, "ms/launch", round(st["spmm_ms_total"] / st["spmm_launches"], 3), "min", round(st["spmm_ms_min"], 3),
          flush=True)
    G.close()
    del src, dst
