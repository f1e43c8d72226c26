"""D2H of the c2 result (4.65 GB) into pinned memory: torch's own copy of a device tensor vs
cleora_fetch / cleora_fetch_async of a handle's T, each timed alone (no compute running).
Usage: python scripts/d2h_fetch.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

g = gen.config("c2")
d = 1024
out = torch.empty((g.n, d), dtype=torch.float32).pin_memory()
dev = torch.empty((g.n, d), dtype=torch.float32, device="cuda")
res = {}
best = 1e9
for _ in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
res["torch_copy_ms"] = best * 1e3
G = cl.cleora_build(torch.from_numpy(g.src).cuda(), torch.from_numpy(g.dst).cuda(), None, g.n, False, device=0)
cl.cleora_init(G, d, 0)
cl.cleora_iterate(G, 4)
cl.cleora_sync(G)
for name, fn in (("cleora_fetch_ms", lambda: cl.cleora_fetch(G, 0, g.n, out)),
                 ("cleora_fetch_async_ms", lambda: (cl.cleora_fetch_async(G, 0, g.n, out), cl.cleora_sync(G)))):
    best = 1e9
    for _ in range(4):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    res[name] = best * 1e3
res["GBps_torch"] = g.n * d * 4 / res["torch_copy_ms"] / 1e6
res["GBps_fetch"] = g.n * d * 4 / res["cleora_fetch_ms"] / 1e6
G.close()
print(json.dumps(res))
