"""The f4 batch workload of scripts/bench_next.py (2,000 Erdos-Renyi graphs, d = 128, I = 4) as a
plain driver for profiling: build_batch + init + iterate.  Usage: python scripts/run_batch.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rng = np.random.default_rng(1)
ns = np.exp(rng.uniform(np.log(50), np.log(5000), 2000)).astype(np.int64)
graphs = [gen.er(int(n), int(4 * n), seed=100 + i) for i, n in enumerate(ns)]
ep = np.zeros(len(graphs) + 1, np.int64)
ep[1:] = np.cumsum([x.n_edges for x in graphs])
src = torch.from_numpy(np.concatenate([x.src for x in graphs])).cuda()
dst = torch.from_numpy(np.concatenate([x.dst for x in graphs])).cuda()
nc = np.array([x.n for x in graphs], np.int32)
B = cl.cleora_build_batch(src, dst, None, ep, nc, False, device=0, timing=True)
cl.cleora_init(B, 128, 0)
cl.cleora_iterate(B, iters)
st = cl.cleora_stats(B)
print("batch spmm ms/launch", st["spmm_ms_total"] / max(1, st["spmm_launches"]), "min", st["spmm_ms_min"])
B.close()
