"""c4 SpMM experiments (round 2).  Prints one JSON object per case: SpMM ms per launch (CUDA events,
library timing), hot rows.
  orig            c4 as generated
  relabel         ids relabelled by in-degree (hot rows first, contiguous)
  colmod<M>       every column id taken mod M: the same rows, lengths and gather count, but all gathers
                  from an M * d * 4-byte table (L2-resident for small M) -- the kernel's own L2-bound rate
Usage: python scripts/r02_c4exp.py <case> <d> [hot_mb]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

case, d = sys.argv[1], int(sys.argv[2])
if len(sys.argv) > 3:
    os.environ["CLEORA_HOT_MB"] = sys.argv[3]
g = gen.config("c4")
src, dst = g.src, g.dst
if case == "relabel":
    indeg = np.bincount(g.dst, minlength=g.n)
    order = np.argsort(-indeg, kind="stable")
    new = np.empty(g.n, np.int32)
    new[order] = np.arange(g.n, dtype=np.int32)
    src, dst = new[g.src], new[g.dst]
elif case.startswith("colmod"):
    dst = (g.dst % int(case[6:])).astype(np.int32)
G = cl.cleora_build(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), torch.from_numpy(g.w).cuda(), g.n, True,
                    timing=True)
cl.cleora_init(G, d, 0)
cl.cleora_iterate(G, 2)
cl.cleora_stats(G, reset=True)
cl.cleora_iterate(G, 4)
st = cl.cleora_stats(G)
info = cl.cleora_info(G)
ms = st["spmm_ms_total"] / st["spmm_launches"]
gb = info["nnz"] * d * 4 / 1e9
print(json.dumps({"case": case, "d": d, "hot_mb": os.environ.get("CLEORA_HOT_MB", "72"), "nnz": info["nnz"],
                  "spmm_ms": round(ms, 3), "spmm_ms_min": round(st["spmm_ms_min"], 3), "gather_GB": round(gb, 1),
                  "gather_TBps": round(gb / ms, 2), "hot_rows": info["hot_rows"]}), flush=True)
G.close()
