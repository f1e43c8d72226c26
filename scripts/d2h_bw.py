"""D2H bandwidth into pinned memory for the e2e fetch (c2: 4.65 GB): one copy vs the same bytes split
over 2 / 4 copies on 2 streams.  Usage: python scripts/d2h_bw.py [GB]"""
import json
import sys

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.65
n = int(gb * 1e9 / 4)
dev = torch.empty(n, dtype=torch.float32, device="cuda")
host = torch.empty(n, dtype=torch.float32).pin_memory()
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
res = {}
for parts in (1, 2, 4):
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        for s in streams[1:]:
            s.wait_event(e0)
        step = (n + parts - 1) // parts
        for p in range(parts):
            s = streams[p % 2]
            with torch.cuda.stream(s):
                host[p * step:(p + 1) * step].copy_(dev[p * step:(p + 1) * step], non_blocking=True)
        e1 = torch.cuda.Event(enable_timing=True)
        streams[0].wait_stream(streams[1])
        e1.record(streams[0])
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[parts] = {"ms": best, "GBps": n * 4 / (best / 1e3) / 1e9}
print(json.dumps(res))
