"""Minimal driver for profiling: build + init + `iters` iterations of one config on cuda:0.
Usage: python scripts/run_spmm.py c2 [iters] [d]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = gen.config(cfg)
d = int(sys.argv[3]) if len(sys.argv) > 3 else g.d
G = cl.cleora_build(torch.from_numpy(g.src).cuda(), torch.from_numpy(g.dst).cuda(),
                    torch.from_numpy(g.w).cuda() if g.w is not None else None, g.n, g.directed, timing=True)
cl.cleora_init(G, d, 0)
cl.cleora_iterate(G, iters)
st = cl.cleora_stats(G)
info = cl.cleora_info(G)
print(cfg, "d", d, "nnz", info["nnz"], "heavy rows", info["heavy_rows"], "items", info["heavy_items"],
      "hot rows", info["hot_rows"],
      "spmm ms/launch", st["spmm_ms_total"] / max(1, st["spmm_launches"]), "min", st["spmm_ms_min"])
G.close()
