"""Host-side timeline of the pipelined e2e loop of bench.py (c2): when each step's build / iterate
enqueue / fetch_async / previous close return.  Usage: python scripts/e2e_trace.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
g = gen.config("c2")
stream = torch.cuda.Stream()
src_h = torch.from_numpy(g.src).pin_memory()
dst_h = torch.from_numpy(g.dst).pin_memory()
outs = [torch.empty((g.n, g.d), dtype=torch.float32).pin_memory() for _ in range(2)]
for rep in range(2):
    t0 = time.perf_counter()
    ms = lambda: f"{1e3 * (time.perf_counter() - t0):8.2f}"   # noqa: E731
    prev = None
    for i in range(k):
        G = cl.cleora_build(src_h, dst_h, None, g.n, False, device=0, stream=stream.cuda_stream)
        a = ms()
        cl.cleora_init(G, g.d, 0)
        cl.cleora_iterate(G, g.iters)
        b = ms()
        cl.cleora_fetch_async(G, 0, g.n, outs[i % 2])
        c = ms()
        if prev is not None:
            prev.close()
        e = ms()
        prev = G
        print(f"rep {rep} step {i}: build {a}  iter-enq {b}  fetch-enq {c}  prev-closed {e}", flush=True)
    prev.close()
    print(f"rep {rep}: total {ms()} ms for {k} steps", flush=True)
