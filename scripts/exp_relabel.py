"""EXPERIMENT: does a contiguous hot set (graph relabelled by degree, hot nodes first) plus a
persisting-L2 access window beat the current evict_last hints on c2?  Prints SpMM ms per launch for
(original ids), (relabelled), (relabelled + CLEORA_EXP_PERSIST_ROWS=K).  Usage: python exp_relabel.py"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch
    import gen
    import paper_2102_02302_b200 as cl
    g = gen.config("c2")
    if sys.argv[2] == "relabel":
        deg = np.bincount(np.concatenate([g.src, g.dst]), minlength=g.n)
        order = np.argsort(-deg, kind="stable")          # new id r -> old id order[r]
        new_of_old = np.empty(g.n, np.int32)
        new_of_old[order] = np.arange(g.n, dtype=np.int32)
        src, dst = new_of_old[g.src], new_of_old[g.dst]
    else:
        src, dst = g.src, g.dst
    G = cl.cleora_build(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), None, g.n, False, timing=True)
    cl.cleora_init(G, g.d, 0)
    cl.cleora_iterate(G, 8)
    st = cl.cleora_stats(G)
    print(sys.argv[2], os.environ.get("CLEORA_EXP_PERSIST_ROWS", "-"), os.environ.get("CLEORA_HOT_MB", "-"),
          "ms/launch", round(st["spmm_ms_total"] / st["spmm_launches"], 4), "min", round(st["spmm_ms_min"], 4),
          "hot", cl.cleora_info(G)["hot_rows"], flush=True)
    G.close()
    sys.exit(0)

me = os.path.abspath(__file__)
for mode, env in (("orig", {}), ("relabel", {}), ("relabel", {"CLEORA_EXP_PERSIST_ROWS": "12000"}),
                  ("relabel", {"CLEORA_EXP_PERSIST_ROWS": "18000"}), ("relabel", {"CLEORA_EXP_PERSIST_ROWS": "24000"}),
                  ("relabel", {"CLEORA_EXP_PERSIST_ROWS": "18000", "CLEORA_NO_HOT": "1"})):
    subprocess.run([sys.executable, me, "run", mode], env=dict(os.environ, **env))
