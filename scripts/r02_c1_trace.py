"""Where a small graph's step goes (c1): host time of each C-ABI call and device time between CUDA
events recorded around it, median over 200 steps after 20 warm-ups."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

g = gen.config(sys.argv[1] if len(sys.argv) > 1 else "c1")
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(device=dev)
src, dst = torch.from_numpy(g.src).to(dev), torch.from_numpy(g.dst).to(dev)
w = torch.from_numpy(g.w).to(dev) if g.w is not None else None
rec = {k: [] for k in ("h_build", "h_init", "h_iter", "h_sync", "h_close", "d_build", "d_init", "d_iter", "d_step")}
for rep in range(220):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record(st)
    G = cl.cleora_build(src, dst, w, g.n, g.directed, device=0, stream=st.cuda_stream)
    t1 = time.perf_counter()
    ev[1].record(st)
    cl.cleora_init(G, g.d, 0)
    t2 = time.perf_counter()
    ev[2].record(st)
    cl.cleora_iterate(G, g.iters)
    t3 = time.perf_counter()
    ev[3].record(st)
    ev[3].synchronize()
    t4 = time.perf_counter()
    G.close()
    t5 = time.perf_counter()
    if rep >= 20:
        for k, v in (("h_build", t1 - t0), ("h_init", t2 - t1), ("h_iter", t3 - t2), ("h_sync", t4 - t3), ("h_close", t5 - t4)):
            rec[k].append(v * 1e3)
        rec["d_build"].append(ev[0].elapsed_time(ev[1]))
        rec["d_init"].append(ev[1].elapsed_time(ev[2]))
        rec["d_iter"].append(ev[2].elapsed_time(ev[3]))
        rec["d_step"].append(ev[0].elapsed_time(ev[3]))
print(json.dumps({"config": g.name, **{k: round(statistics.median(v), 4) for k, v in rec.items()}}))
