"""Time cleora_init (T_0 hash into the existing buffers) on c2 at d = 1024, after a warm-up.
Usage: python scripts/time_init.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = gen.config("c2")
G = cl.cleora_build(torch.from_numpy(g.src).cuda(), torch.from_numpy(g.dst).cuda(), None, g.n, False, device=0)
cl.cleora_init(G, 1024, 0)
cl.cleora_sync(G)
ts = []
for i in range(reps):
    t0 = time.perf_counter()
    cl.cleora_init(G, 1024, i)
    cl.cleora_sync(G)
    ts.append(1e3 * (time.perf_counter() - t0))
print(f"cleora_init c2 d=1024: min {min(ts):.3f} ms, median {sorted(ts)[len(ts) // 2]:.3f} ms")
G.close()
