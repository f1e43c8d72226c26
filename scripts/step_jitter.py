"""Step-time jitter diagnosis: the bench step (build -> init -> iterate(I) -> destroy) repeated,
with per-step CUDA-event times and host-side wall time of every C-ABI call, under a chosen
clock-sampling mode.  Usage: python scripts/step_jitter.py [none|nvml|smi] [steps] [cfg]"""
import json
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "none"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = sys.argv[3] if len(sys.argv) > 3 else "c2"
g = gen.config(cfg)
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
src, dst = torch.from_numpy(g.src).to(dev), torch.from_numpy(g.dst).to(dev)
w = torch.from_numpy(g.w).to(dev) if g.w is not None else None
torch.cuda.synchronize()

stop = threading.Event()
proc = None
if mode == "nvml":
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    lat = []

    def run():
        while not stop.is_set():
            t0 = time.perf_counter()
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            t1 = time.perf_counter()
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            t2 = time.perf_counter()
            lat.append((1e3 * (t1 - t0), 1e3 * (t2 - t1)))
            stop.wait(0.1)
    th = threading.Thread(target=run, daemon=True)
    th.start()
elif mode == "smi":
    proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.active", "--format=csv",
                             "-lms", "200"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)

rows = []
for i in range(steps + 3):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    G = cl.cleora_build(src, dst, w, g.n, g.directed, device=0, stream=s.cuda_stream)
    t1 = time.perf_counter()
    cl.cleora_init(G, g.d, 0)
    t2 = time.perf_counter()
    cl.cleora_iterate(G, g.iters)
    t3 = time.perf_counter()
    G.close()
    t4 = time.perf_counter()
    e1.record(s)
    e1.synchronize()
    rows.append(dict(step=i, dev_ms=round(e0.elapsed_time(e1), 3), build=round(1e3 * (t1 - t0), 3),
                     init=round(1e3 * (t2 - t1), 3), iterate=round(1e3 * (t3 - t2), 3),
                     destroy=round(1e3 * (t4 - t3), 3)))
stop.set()
if proc:
    proc.terminate()
dev_ms = [r["dev_ms"] for r in rows[3:]]
out = dict(mode=mode, cfg=cfg, steps=steps, mean=sum(dev_ms) / len(dev_ms), min=min(dev_ms), max=max(dev_ms),
           slow=[r for r in rows[3:] if r["dev_ms"] > 1.3 * min(dev_ms)][:12])
if mode == "nvml":
    out["nvml_ms_max"] = [max(x[0] for x in lat), max(x[1] for x in lat)] if lat else None
print(json.dumps(out), flush=True)
