"""Build time (device, CUDA events around cleora_build, median of 20 after 3 warm-ups) of a config
or of the f4 batch.  Usage: python scripts/r02_build_time.py c3|f4"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

name = sys.argv[1]
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(device=dev)
if name == "f4":
    rng = np.random.default_rng(1)
    ns = np.exp(rng.uniform(np.log(50), np.log(5000), 2000)).astype(np.int64)
    graphs = [gen.er(int(n), int(4 * n), seed=100 + i) for i, n in enumerate(ns)]
    ep = np.zeros(len(graphs) + 1, np.int64)
    ep[1:] = np.cumsum([x.n_edges for x in graphs])
    src = torch.from_numpy(np.concatenate([x.src for x in graphs])).to(dev)
    dst = torch.from_numpy(np.concatenate([x.dst for x in graphs])).to(dev)
    nc = np.array([x.n for x in graphs], np.int32)
    build = lambda: cl.cleora_build_batch(src, dst, None, ep, nc, False, device=0, stream=st.cuda_stream)  # noqa: E731
else:
    g = gen.config(name)
    src, dst = torch.from_numpy(g.src).to(dev), torch.from_numpy(g.dst).to(dev)
    w = torch.from_numpy(g.w).to(dev) if g.w is not None else None
    build = lambda: cl.cleora_build(src, dst, w, g.n, g.directed, device=0, stream=st.cuda_stream)  # noqa: E731
ts = []
for rep in range(23):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    G = build()
    e1.record(st)
    e1.synchronize()
    G.close()
    if rep >= 3:
        ts.append(e0.elapsed_time(e1))
print(json.dumps({"config": name, "small_build": os.environ.get("CLEORA_SMALL_BUILD", "1"),
                  "small_max": os.environ.get("CLEORA_SMALL_MAX_ENTRIES", "default"),
                  "build_ms_median": round(statistics.median(ts), 4), "build_ms_min": round(min(ts), 4)}))
