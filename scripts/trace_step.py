"""Host-side phase timing of one bench step (c2 by default): build / init / iterate / destroy,
each followed by a device sync, wall clock.  Usage: python scripts/trace_step.py [cfg] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
g = gen.config(cfg)
s = torch.cuda.Stream()
src, dst = torch.from_numpy(g.src).cuda(), torch.from_numpy(g.dst).cuda()
w = torch.from_numpy(g.w).cuda() if g.w is not None else None
torch.cuda.synchronize()
for rep in range(reps):
    t0 = time.perf_counter()
    G = cl.cleora_build(src, dst, w, g.n, g.directed, stream=s.cuda_stream)
    t1 = time.perf_counter()
    cl.cleora_init(G, g.d, 0); cl.cleora_sync(G)
    t2 = time.perf_counter()
    cl.cleora_iterate(G, g.iters); cl.cleora_sync(G)
    t3 = time.perf_counter()
    G.close()
    t4 = time.perf_counter()
    print(f"{cfg} rep {rep}: build {1e3*(t1-t0):.2f} ms  init {1e3*(t2-t1):.2f}  iterate {1e3*(t3-t2):.2f}  "
          f"destroy {1e3*(t4-t3):.2f}  total {1e3*(t4-t0):.2f}", flush=True)
