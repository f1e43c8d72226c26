#!/usr/bin/env python
"""Benchmark of the Cleora hot path on B200 (BASELINE.json metric, one JSON line on rank 0).

The workload is c4 (BASELINE.json configs[3], the LiveJournal stand-in, "row-sharded at 1/2/4/8
GPUs": the metric's own configuration and the largest one that runs on one GPU); c2 and c3 are
reported beside it as secondary SpMM figures (``secondary``).  ``--config`` selects another.

A *step* is one pass of the whole hot path over one synthetic
graph: cleora_build (validate, mirror, radix sort, merge, row pointer, degree, D^-1 scaling,
schedule) -> cleora_init (hash T_0) -> cleora_iterate(I) (I fused SpMM + row-normalise
launches), with the COO already resident in HBM when the timed region starts.  The result
stays in HBM; the end-to-end variant (``e2e``) goes through the same C-ABI calls with HOST
buffers: pinned COO in, H2D inside cleora_build, and the result out into pinned host memory,
inside the timed region -- as cleora_fetch_nonzero (the rows with entries and their ids; every
other row is exactly 0 after a step, reading RZ), with the dense cleora_fetch of all N x d rows
measured beside it (``e2e.dense_fetch``; ``--dense-fetch`` makes it the e2e figure).

value = nnz * d * I / step_time   (nnz = stored CSR entries; BASELINE metric "nnz·d/s")
Multi-GPU (one rank per GPU, NCCL): ``--gpus N`` under torchrun (WORLD_SIZE set, must equal N),
or ``python bench.py --gpus N`` alone, which re-launches itself under torch.distributed.run with
N ranks.  M is row-sharded by nnz balance (each rank builds and keeps only its rows), every rank
keeps a full T replica, each iteration's rows reach the other replicas through the fused
peer-store exchange; the total work is the same graph for every N ("scaling": "strong"); time =
max over ranks of CUDA-event step time.

--impl reference times the CPU oracle (oracle/, plain C + OpenMP) on a bounded sample of the
same workload (one oracle iteration over a leading block of rows), on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "nnz·d/s per Cleora iteration and achieved HBM GB/s vs peak at 1/2/4/8 B200"
UNIT = "nnz·d/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks and throttle reasons sampled every 100 ms by a thread through NVML (the library
    nvidia-smi reads; spawning nvidia-smi itself inside the timed region stalled CUDA calls for
    tens of ms).  Start it before the warm-up; mark() the timed window; summary() uses only the
    samples taken inside marked windows."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.windows = []
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = gpu
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[gpu])
                except ValueError:
                    pass
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _reasons(self):
        f = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
        return int(f(self.h))

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append((time.perf_counter(), float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)),
                                     self._reasons()))
            except Exception:
                pass
            self._stop.wait(0.1)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def stop(self):
        self._stop.set()

    def mark(self, t0, t1):
        self.windows.append((t0, t1))

    def summary(self):
        inside = [s for s in self.samples if any(a - 0.05 <= s[0] <= b + 0.05 for a, b in self.windows)]
        mhz = [s[1] for s in inside]
        reasons = set()
        for _, _, r in inside:
            for bit, name in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(mhz), "source": "nvml"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def e2e_schedule(handle_bytes, t_bytes, total_hbm):
    """How the e2e steps overlap: "full" = two whole handles alive (step i's copy beside step i+1),
    "trim" = step i trimmed to its result T first (cleora_trim), None = serial."""
    if 2 * handle_bytes < 0.85 * total_hbm:
        return "full"
    if handle_bytes + t_bytes < 0.9 * total_hbm:
        return "trim"
    return None


def cpu_baseline(g, M_holder, d, iters, budget_s=12.0):
    """The oracle as it stands on this host.  Small graphs: full CSR build, T_0 and all I
    iterations when that fits ~budget_s, else one iteration over a leading block of rows with
    the iteration time extrapolated by nnz share.  Graphs whose oracle CSR build alone would
    take minutes (c4, c5: sorting 10^8-10^9 entries): the build is timed on the edges touching
    a leading block of rows [0, r1) and extrapolated by entry count; T_0 is built whole (every
    row can be a neighbour); one iteration runs over [0, r1).  Returns (value, details)."""
    import oracle
    n_ent = g.n_edges * (1 if g.directed else 2)
    if n_ent > 50_000_000:
        return _cpu_baseline_block(g, M_holder, d, iters, budget_s)
    t0 = time.perf_counter()
    M = oracle.build_from(g)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    T = oracle.hash_init(g.n, d, 0)
    t_init = time.perf_counter() - t0
    # probe: a small block, then size the sample to the budget; when the whole iteration fits
    # the budget, time all I iterations over all rows (no extrapolation)
    t0 = time.perf_counter()
    T1 = oracle.step(M, T)
    t_full = time.perf_counter() - t0
    if t_full * iters <= budget_s:
        for _ in range(iters - 1):
            T1 = oracle.step(M, T1)
        t_all = time.perf_counter() - t0
        M_holder.append(M)
        return (M.nnz * d * iters / (t_build + t_init + t_all),
                dict(t_build_s=t_build, t_init_s=t_init, t_sample_s=t_all, rows=g.n, nnz_sample=M.nnz,
                     t_iter_est_s=t_all / iters, iter_rate=M.nnz * d * iters / t_all, full=True))
    del T1
    r1 = min(g.n, 2048)
    t0 = time.perf_counter()
    oracle.step(M, T, 0, r1)
    t_probe = max(time.perf_counter() - t0, 1e-4)
    nnz_probe = max(int(M.row_ptr[r1]), 1)
    rate = nnz_probe / t_probe
    target_nnz = int(rate * budget_s)
    r1 = int(np.searchsorted(M.row_ptr, min(target_nnz, M.nnz), side="left"))
    r1 = max(1, min(r1, g.n))
    t0 = time.perf_counter()
    oracle.step(M, T, 0, r1)
    t_samp = time.perf_counter() - t0
    nnz_s = int(M.row_ptr[r1])
    t_iter = t_samp * M.nnz / max(nnz_s, 1)
    t_step = t_build + t_init + iters * t_iter
    value = M.nnz * d * iters / t_step
    M_holder.append(M)
    return value, dict(t_build_s=t_build, t_init_s=t_init, t_sample_s=t_samp, rows=r1, nnz_sample=nnz_s,
                       t_iter_est_s=t_iter, iter_rate=nnz_s * d / t_samp, full=False)


def _cpu_baseline_block(g, M_holder, d, iters, budget_s):
    import gen
    import oracle
    n_ent = g.n_edges * (1 if g.directed else 2)
    # rows [0, r1) holding ~1/64 of the entries (ids are scrambled, so a prefix is a fair sample)
    r1 = max(1, g.n // 64)
    touch = g.src < r1 if g.directed else (g.src < r1) | (g.dst < r1)
    sub = gen.EdgeList("block", g.n, g.src[touch], g.dst[touch], None if g.w is None else g.w[touch], g.directed)
    del touch
    t0 = time.perf_counter()
    M = oracle.build_from(sub)
    t_bs = time.perf_counter() - t0
    ent_s = sub.n_edges * (1 if g.directed else 2)
    del sub
    t0 = time.perf_counter()
    T = oracle.hash_init(g.n, d, 0)
    t_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.step(M, T, 0, r1)
    t_samp = time.perf_counter() - t0
    nnz_s = int(M.row_ptr[r1])
    nnz = n_ent          # upper bound of the merged nnz; the GPU line reports the exact one
    t_build = t_bs * n_ent / max(ent_s, 1)
    t_iter = t_samp * nnz / max(nnz_s, 1)
    value = nnz * d * iters / (t_build + t_init + iters * t_iter)
    del T
    return value, dict(t_build_s=t_build, t_init_s=t_init, t_sample_s=t_samp, rows=r1, nnz_sample=nnz_s,
                       t_iter_est_s=t_iter, iter_rate=nnz_s * d / t_samp, full=False, block=True,
                       t_build_sample_s=t_bs, entries_sample=ent_s)


def run_reference(args, g, world, rank):
    """--impl reference: the CPU oracle, each step = one oracle iteration over a fixed leading
    block of rows (a bounded sample of the workload), rank 0 only."""
    if rank != 0:
        return
    import oracle
    d, iters = g.d, g.iters
    M = oracle.build_from(g)
    T = oracle.hash_init(g.n, d, 0)
    r1 = min(g.n, 2048)
    t0 = time.perf_counter()
    oracle.step(M, T, 0, r1)
    rate = max(int(M.row_ptr[r1]), 1) / max(time.perf_counter() - t0, 1e-4)
    per_step_s = float(os.environ.get("CLEORA_REF_STEP_S", "3.0"))
    r1 = int(np.searchsorted(M.row_ptr, min(int(rate * per_step_s), M.nnz), side="left"))
    r1 = max(1, min(r1, g.n))
    nnz_s = int(M.row_ptr[r1])
    for _ in range(args.warmup):
        oracle.step(M, T, 0, r1)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.step(M, T, 0, r1)
        ts.append(time.perf_counter() - t0)
    t = sum(ts)
    value = nnz_s * d * args.steps / t
    cores = oracle.num_threads()
    sample = (f"{g.name}: one oracle iteration (fp64 accumulate, fp32 store) over rows [0,{r1}) = "
              f"{nnz_s} of {M.nnz} nnz, d={d}, per step; CSR build and T_0 excluded")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(g, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


L2_BYTES = 126 * 2**20
FLUSH_BYTES = 512 * 2**20


def t_bytes(g):
    return g.n * ((g.d + 3) // 4 * 4) * 4


def config_dict(g, world):
    tb = t_bytes(g)
    l2 = (f"inputs larger than L2: T = {tb / 1e9:.2f} GB per replica > 126 MB L2, no flush" if tb > 4 * L2_BYTES else
          f"T = {tb / 1e6:.1f} MB per replica is not >> 126 MB L2: L2 flushed ({FLUSH_BYTES >> 20} MB write) "
          "before every timed step, outside the step's events")
    return {"workload": g.name, "desc": g.meta.get("desc", ""), "N": g.n, "edges_in": g.n_edges,
            "d": g.d, "iterations": g.iters, "directed": g.directed, "weighted": g.w is not None,
            "parallelism": f"rowshard{world}" if world > 1 else "single",
            "exchange": "fused peer stores + NCCL barrier (NCCL all-gather fallback)" if world > 1 else "none",
            "l2": l2}


def load_traffic(name, d):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        e = json.load(open(p)).get(f"{name}_d{d}")
        return None if e is None else e["bytes_per_launch_mean"]
    except Exception:
        return None


def launch_ranks(args, argv):
    """``--gpus N`` without WORLD_SIZE: re-run this script under torch.distributed.run with N ranks
    on this node (the driver's own launch line), and return its exit code."""
    import socket
    import subprocess
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def parse_args(argv):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cleora", choices=["cleora", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dense-fetch", action="store_true", help="e2e: fetch all N x d rows (cleora_fetch) only")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the c2/c3 SpMM figures")
    ap.add_argument("--dry-launch", action="store_true",
                    help="launch test: every rank prints its rank/world as JSON and exits (no GPU work)")
    return ap.parse_args(argv)


def kernel_l2_rate(cl, g, dev, local, stream, table_bytes=32 << 20):
    """The SpMM kernel's own gather rate when every gather hits L2: the graph's mirrored entry list as
    a directed graph with every column folded into [0, K), K * d * 4 bytes <= table_bytes (the same rows,
    row lengths and gather count, up to the duplicates folding merges), 4 timed iterations after 1.
    Returns (GB/s of gathered bytes, folded nnz, ms per launch)."""
    import torch
    dp = (g.d + 3) // 4 * 4
    K = max(1, min(g.n, table_bytes // (dp * 4)))
    src = np.asarray(g.src)
    dst = np.asarray(g.dst)
    w = g.w
    if not g.directed:
        m = src != dst
        src, dst = np.concatenate([src, dst[m]]), np.concatenate([dst, src[m]])
        w = None if w is None else np.concatenate([w, w[m]])
    s_d = torch.from_numpy(np.ascontiguousarray(src)).to(dev)
    d_d = torch.from_numpy((dst % K).astype(np.int32)).to(dev)
    w_d = torch.from_numpy(np.ascontiguousarray(w)).to(dev) if w is not None else None
    G = cl.cleora_build(s_d, d_d, w_d, g.n, True, device=local, stream=stream.cuda_stream, timing=True)
    try:
        cl.cleora_init(G, g.d, 0)
        cl.cleora_iterate(G, 1)
        cl.cleora_stats(G, reset=True)
        cl.cleora_iterate(G, 4)
        st = cl.cleora_stats(G)
        nnz = cl.cleora_info(G)["nnz"]
    finally:
        G.close()
    ms = st["spmm_ms_total"] / max(1, st["spmm_launches"])
    return nnz * g.d * 4 / (ms / 1e3) / 1e9, nnz, ms


def measure_secondary(cl, names, dev, local, stream, peak, reps=3):
    """SpMM-only figures of other configs (N = 1): build once, then `reps` x (init + I iterations),
    device time of every fused SpMM launch from the library's CUDA events; first rep discarded."""
    import gen
    import torch
    out = {}
    for name in names:
        g = gen.config(name)
        d, iters = g.d, g.iters
        src = torch.from_numpy(g.src).to(dev)
        dst = torch.from_numpy(g.dst).to(dev)
        w = torch.from_numpy(g.w).to(dev) if g.w is not None else None
        G = cl.cleora_build(src, dst, w, g.n, g.directed, device=local, stream=stream.cuda_stream, timing=True)
        try:
            for r in range(reps):
                cl.cleora_init(G, d, 0)
                cl.cleora_iterate(G, iters)
                st = cl.cleora_stats(G, reset=(r == 0))
            info = cl.cleora_info(G)
        finally:
            G.close()
        ms = st["spmm_ms_total"] / max(1, st["spmm_launches"])
        nnz = info["nnz"]
        b_comp = 8 * (g.n + 1) + 8 * nnz + 2 * g.n * d * 4
        ref_rows = info["referenced_rows"] if info["referenced_rows"] >= 0 else g.n
        b_strict = 8 * (g.n + 1) + 8 * nnz + (ref_rows + g.n - info["zero_rows"]) * d * 4
        del src, dst, w
        k_rate, _, k_ms = kernel_l2_rate(cl, g, dev, local, stream)
        out[name] = {"d": d, "iterations": iters, "nnz": nnz, "spmm_ms": ms, "spmm_ms_min": st["spmm_ms_min"],
                     "nnz_d_per_s": nnz * d / (ms / 1e3), "frac": b_comp / (ms / 1e3) / 1e9 / peak,
                     "strict_frac": b_strict / (ms / 1e3) / 1e9 / peak, "algorithmic_bytes_per_launch": b_comp,
                     "traffic": load_traffic(name, d), "launches": st["spmm_launches"],
                     "gather_bound_ms": nnz * d * 4 / (k_rate * 1e9) * 1e3 if k_rate > 0 else None,
                     "kernel_l2_gbs": k_rate}
    return out


def main():
    argv = sys.argv[1:]
    args = parse_args(argv)
    if args.warmup < 3 and args.impl != "reference":
        print("bench.py: --warmup must be >= 3", file=sys.stderr)
        args.warmup = 3
    if args.gpus < 1:
        print("bench.py: --gpus must be >= 1", file=sys.stderr)
        sys.exit(2)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args, argv))
    world, rank, local = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or omit WORLD_SIZE", file=sys.stderr)
        sys.exit(2)
    if world > 1:
        # torch.distributed.run sets OMP_NUM_THREADS=1; the generators (and the reference arm's oracle,
        # rank 0 alone) are OpenMP programs: give each rank its share of the host cores (all of them to
        # the reference arm's only working rank).  Read by libgomp when it is first loaded, below.
        ncpu = os.cpu_count() or 1
        os.environ["OMP_NUM_THREADS"] = str(ncpu if args.impl == "reference" else max(1, ncpu // world))
    if args.dry_launch:
        # one write() per line: the ranks share the launcher's stdout
        sys.stdout.write(json.dumps({"dry_launch": True, "rank": rank, "world": world, "local_rank": local}) + "\n")
        sys.stdout.flush()
        return

    import gen
    g = gen.config(args.config)

    if args.impl == "reference":
        run_reference(args, g, world, rank)
        return

    import torch
    import paper_2102_02302_b200 as cl

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        obj = [cl.cleora_nccl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    d, iters = g.d, g.iters
    stream = torch.cuda.Stream(device=dev)
    src_d = torch.from_numpy(g.src).to(dev)
    dst_d = torch.from_numpy(g.dst).to(dev)
    w_d = torch.from_numpy(g.w).to(dev) if g.w is not None else None
    # T smaller than a few L2s: write a buffer larger than L2 before every timed step (outside its events)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev) if t_bytes(g) <= 4 * L2_BYTES else None
    torch.cuda.synchronize()

    xnccl = [False]      # multi-GPU: fused peer-store exchange unless it fails on this box

    def one_step(timing=False, spmm_events=None):
        G = cl.cleora_build(src_d, dst_d, w_d, g.n, g.directed, device=local, stream=stream.cuda_stream,
                            rank=rank, world=world, nccl_id=nccl_id, timing=timing, exchange_nccl=xnccl[0])
        cl.cleora_init(G, d, 0)
        if spmm_events is not None:
            # the I fused SpMM+normalise launches of this step, bracketed on the stream they run on
            e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e_s.record(stream)
            cl.cleora_iterate(G, iters)
            e_e.record(stream)
            spmm_events.append((e_s, e_e))
        else:
            cl.cleora_iterate(G, iters)
        return G

    clk = ClockSampler(local).start()
    # warm-up (also yields the schedule facts)
    info = None
    for i in range(args.warmup):
        try:
            G = one_step()
        except cl.CleoraError as e:
            if world == 1 or xnccl[0] or i > 0:
                raise
            print(f"bench.py: fused exchange failed ({e}); using the NCCL all-gather exchange", file=sys.stderr)
            xnccl[0] = True
            G = one_step()
        info = cl.cleora_info(G)
        G.close()
    nnz = info["nnz"]

    # timed region: K steps, CUDA events on the library's stream around every step, barrier + sync
    # on both sides; a step's time is build + init + I iterations (the L2 flush, when there is one,
    # runs between a step's end event and the next step's start event)
    barrier()
    torch.cuda.synchronize()
    launches0 = cl.cleora_kernel_launches()
    steps_ev = []
    spmm_ev = []
    t_w0 = time.perf_counter()
    for _ in range(args.steps):
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.zero_()
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_a.record(stream)
        G = one_step(spmm_events=spmm_ev)
        e_b.record(stream)
        G.close()
        steps_ev.append((e_a, e_b))
    steps_ev[-1][1].synchronize()
    clk.mark(t_w0, time.perf_counter())
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in steps_ev]
    launches = cl.cleora_kernel_launches() - launches0
    barrier()
    # without a flush the K steps run back to back and the bracket is first start -> last end (the
    # destroy of step i between them included); with a flush, the sum of the steps' own brackets
    span = steps_ev[0][0].elapsed_time(steps_ev[-1][1]) if flush is None else sum(step_ms)
    ms_step = max_over_ranks(span / args.steps)
    value = nnz * d * iters / (ms_step / 1e3)

    # dominant kernel: the fused SpMM+normalise launches, timed live in the timed steps with CUDA
    # events on the library's stream around cleora_iterate (the I launches and nothing else; with
    # P > 1 the exchange barrier / all-gather is inside the bracket too)
    spmm_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in spmm_ev) / (len(spmm_ev) * iters))
    xms = 0.0
    if world > 1:                # exchange time alone, from the library's per-launch events
        G = one_step(timing=True)
        xms = cl.cleora_stats(G, reset=True)["exchange_ms_total"]
        G.close()
    peak, peak_src = load_peaks()
    # SURVEY.md §8(d) / BASELINE north star: compulsory bytes per iteration = CSR (int64 row
    # pointer, int32 col, fp32 val) + one read and one write of the N x d fp32 T; per rank 1/P
    b_comp = (8 * (g.n + 1) + 8 * nnz + 2 * g.n * d * 4) / world
    achieved = b_comp / (spmm_ms / 1e3) / 1e9
    # stricter variant: only rows that are ever gathered are read, only rows with out-edges are
    # written (steady state: empty rows are not rewritten after the first two steps)
    ref_rows = info.get("referenced_rows", -1)
    ref_rows = g.n if ref_rows is None or ref_rows < 0 else ref_rows
    b_strict = (8 * (g.n + 1) + 8 * nnz + (ref_rows + g.n - info["zero_rows"]) * d * 4) / world
    # the second roofline (SURVEY §8(d) "Which roofline"): the gather operand stream nnz*d*4, every
    # byte of which crosses L2 -> SM, at the random-row gather rate measured now on this GPU
    # (cleora_probe_gather: rows of d*4 bytes from an L2-resident 32 MiB table)
    row_b = max(16, min(4096, (d + 3) // 4 * 16))
    while row_b < 512 and 512 % row_b:
        row_b += 16
    l2_rate = cl.cleora_probe_gather(row_b, 32 << 20, max(1 << 20, (1 << 32) // row_b), local)
    # ... and the SpMM kernel's own rate on this graph with every gather folded into L2 (the stronger
    # of the two is the bound: the kernel's TMA / cp.async ring beats the probe's plain loads)
    k_rate, k_nnz, k_ms = kernel_l2_rate(cl, g, dev, local, stream) if world == 1 else (0.0, 0, 0.0)
    best_rate = max(l2_rate, k_rate)
    gather_b = nnz * d * 4 / world
    lps = info.get("launches_per_step", 1) or 1
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": load_traffic(g.name, d),
                "kernel": "k_spmm_tma (fused SpMM + row L2 normalise)" + (
                    f", {lps} half-row launches per iteration; inside one iterate call every step but the last leaves its "
                    "rows unnormalised with their scales aside and the next step runs on pre-scaled weights (one short "
                    "k_lazy_vals launch, inside the timed events; DESIGN reading R21); figures per iteration"
                    if lps > 1 else ""),
                "launches_per_iteration": lps,
                "kernel_ms": spmm_ms, "kernel_timing": "CUDA events around cleora_iterate in the timed steps",
                "algorithmic_bytes_per_launch": b_comp, "peak_source": peak_src,
                "strict_bytes_per_launch": b_strict, "strict_frac": b_strict / (spmm_ms / 1e3) / 1e9 / peak,
                "gather_bytes_per_launch": gather_b,
                "gather_bound": {"bytes": gather_b, "l2_gather_gbs": best_rate, "row_bytes": row_b,
                                 "ms": gather_b / (best_rate * 1e9) * 1e3 if best_rate > 0 else None,
                                 "frac": (gather_b / (best_rate * 1e9) * 1e3) / spmm_ms if best_rate > 0 else None,
                                 "probe_gbs": l2_rate, "kernel_l2_gbs": k_rate, "kernel_l2_ms": k_ms,
                                 "kernel_l2_nnz": k_nnz,
                                 "how": "nnz*d*4 / the faster of two L2-resident gather rates measured live: "
                                        "random d*4-byte rows from a 32 MiB table (cleora_probe_gather), and this "
                                        "SpMM kernel on this graph with every column folded into a 32 MiB table "
                                        "(same rows and gather count, all hits)"},
                "bytes_def": "8(N+1) + 8 nnz + 2 N d 4 (CSR + one read and one write of T), per rank"}
    tr = roofline["traffic"]
    if tr:
        roofline["traffic_gbs"] = tr / (spmm_ms / 1e3) / 1e9
    del flush

    # e2e through the public C-ABI with host buffers (pinned), copies inside the timed region.
    # Every step: H2D of the COO (inside cleora_build), build, init, I iterations, D2H of all N x d
    # rows.  Pipelined as a server would run it: step i's D2H (cleora_fetch_async, on the library's
    # copy stream) overlaps step i+1's H2D + build + iterations; a step's handle is released once
    # the next step is enqueued (its destroy waits for its copy).  The serial variant (blocking
    # fetch, then destroy) is reported beside it.
    e2e = None
    if not args.no_e2e:
        # the device-resident COO of the timed steps is not needed any more: its HBM goes to the
        # e2e handles (c5: 11.4 GB, the difference between fitting two handles or not)
        src_d = dst_d = w_d = None
        torch.cuda.empty_cache()
        src_h = torch.from_numpy(g.src).pin_memory()
        dst_h = torch.from_numpy(g.dst).pin_memory()
        w_h = torch.from_numpy(g.w).pin_memory() if g.w is not None else None
        # pipelining keeps two handles (and two output buffers) alive.  When two full handles do not
        # fit in HBM (c5: one is ~110 GB of the 180 GB), the previous handle is trimmed to its result
        # (cleora_trim) once its fetch is enqueued, so only its T buffer overlaps the next build.
        total_hbm = torch.cuda.get_device_properties(local).total_memory
        pipe_mode = e2e_schedule(info["device_bytes"], t_bytes(g), total_hbm)
        pipelined = pipe_mode is not None
        outs = [torch.empty((g.n, d), dtype=torch.float32).pin_memory() for _ in range(2 if pipelined else 1)]
        # the result as a user fetches it: the rows with entries and their ids (cleora_fetch_nonzero;
        # every other row is exactly 0 after a step, reading RZ), packed into the front of the same
        # pinned buffers; the dense N x d fetch is measured beside it
        # (P > 1: each rank fetches its own shard's rows with entries; the bytes below are the whole job's)
        n_nzr = None
        ids = [torch.empty(g.n, dtype=torch.int32).pin_memory() for _ in outs]

        def e2e_build():
            G = cl.cleora_build(src_h, dst_h, w_h, g.n, g.directed, device=local, stream=stream.cuda_stream,
                                rank=rank, world=world, nccl_id=nccl_id, exchange_nccl=xnccl[0])
            cl.cleora_init(G, d, 0)
            cl.cleora_iterate(G, iters)
            return G

        def fetch(G, i, compact, wait):
            j = i % len(outs)
            if compact:
                (cl.cleora_fetch_nonzero if wait else cl.cleora_fetch_nonzero_async)(G, outs[j], ids[j])
            elif wait:
                cl.cleora_fetch(G, 0, g.n, outs[j])
            else:
                cl.cleora_fetch_async(G, 0, g.n, outs[j])

        def e2e_serial(k, compact):
            for _ in range(k):
                G = e2e_build()
                fetch(G, 0, compact, True)
                G.close()

        def e2e_pipelined(k, compact):
            prev = None
            for i in range(k):
                G = e2e_build()
                fetch(G, i, compact, False)
                if pipe_mode == "trim":
                    cl.cleora_trim(G)
                if prev is not None:
                    prev.close()
                prev = G
            prev.close()

        def timed(fn, k, compact):
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(k, compact)
            e1.record(stream)
            e1.synchronize()
            clk.mark(t0, time.perf_counter())
            torch.cuda.synchronize()
            barrier()
            return max_over_ranks(e0.elapsed_time(e1) / k), 1e3 * (time.perf_counter() - t0) / k

        oom0 = cl.cleora_oom_fallbacks()
        e2e_serial(1, False)
        if pipelined:
            try:
                e2e_pipelined(2, True)
            except cl.CleoraError as e:          # out of memory after all: serial
                print(f"bench.py: pipelined e2e failed ({e}); serial e2e", file=sys.stderr)
                pipelined = False
                cl.cleora_release_cached_memory()
        h2d = g.n_edges * 8 + (g.n_edges * 4 if g.w is not None else 0)
        if not args.dense_fetch:
            G = e2e_build()
            n_rank = cl.cleora_nonzero_count(G)
            G.close()
            if world > 1:
                import torch.distributed as dist
                t = torch.tensor([n_rank], dtype=torch.int64, device=dev)
                dist.all_reduce(t)
                n_nzr = int(t.item())
            else:
                n_nzr = n_rank

        def measure(compact):
            k2 = k_serial = max(2, min(args.steps, 5))
            ms_serial, wall_serial = timed(e2e_serial, k2, compact)
            what = "cleora_fetch_nonzero_async" if compact else "cleora_fetch_async"
            if pipelined:
                # the pipeline's fill (the first step's H2D + build + iterations, with no D2H to hide behind)
                # is paid once per timed run: more steps than the serial run, so the figure is the schedule's
                # steady-state rate rather than its start-up
                k2 = max(2, min(args.steps, 10))
                ms_e2e, wall = timed(e2e_pipelined, k2, compact)
                mode = f"pipelined: step i's D2H ({what}) overlaps step i+1's H2D + build + iterations"
                if pipe_mode == "trim":
                    mode += " (step i's handle trimmed to its result, cleora_trim, to make room)"
                if ms_serial < ms_e2e:      # both measured the same way; report the faster schedule
                    mode = f"serial (faster than the measured {mode}: {ms_e2e:.1f} ms per step)"
                    ms_e2e, wall, k2 = ms_serial, wall_serial, k_serial
            else:
                ms_e2e, wall = ms_serial, wall_serial
                mode = "serial: build, iterations, blocking fetch, destroy (two handles do not fit in HBM)"
            d2h = (n_nzr * d * 4 + n_nzr * 4) if compact else g.n * d * 4
            return {"value": nnz * d * iters / (ms_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e, "steps": k2, "wall_ms_per_step": wall,
                    "mode": mode, "serial_value": nnz * d * iters / (ms_serial / 1e3),
                    "serial_ms_per_step": ms_serial, "serial_steps": k_serial}

        dense = measure(False)
        if n_nzr is not None and not args.dense_fetch:
            e2e = measure(True)
            e2e["result"] = (f"cleora_fetch_nonzero: the {n_nzr:,} rows with entries (d fp32 each) and their "
                             f"int32 ids{', each rank its own shard' if world > 1 else ''}; the other "
                             f"{g.n - n_nzr:,} rows are exactly 0 after a step (reading RZ)")
            e2e["dense_fetch"] = {k: dense[k] for k in ("value", "ms_per_step", "d2h_bytes_per_step", "mode",
                                                        "serial_ms_per_step")}
        else:
            e2e = dense
            e2e["result"] = "cleora_fetch of all N x d rows"
        e2e["oom_fallbacks"] = cl.cleora_oom_fallbacks() - oom0
        del outs, ids, src_h, dst_h, w_h
    clk.stop()

    # secondary configs (N = 1): the c2 / c3 SpMM figures beside the headline
    secondary = None
    if world == 1 and not args.no_secondary:
        src_d = dst_d = w_d = None
        torch.cuda.empty_cache()
        names = [n for n in ("c2", "c3") if n != g.name]
        secondary = measure_secondary(cl, names, dev, local, stream, peak)

    # CPU oracle baseline: rank 0 at N = 1 only, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        holder = []
        v, det = cpu_baseline(g, holder, d, iters)
        cpu = {"value": v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
               "sample": (f"{g.name}: full oracle run: CSR build ({det['t_build_s']:.2f} s) + T_0 ({det['t_init_s']:.2f} s) + "
                          f"{iters} iterations over all rows ({det['t_sample_s']:.2f} s)" if det["full"] else
                          f"{g.name}: oracle CSR build over the {det.get('entries_sample')} entries touching rows [0,{det['rows']}) "
                          f"({det.get('t_build_sample_s', 0):.2f} s, extrapolated by entry count to {det['t_build_s']:.1f} s) + "
                          f"full T_0 ({det['t_init_s']:.2f} s) + one iteration over rows [0,{det['rows']}) = {det['nnz_sample']} nnz "
                          f"({det['t_sample_s']:.2f} s), extrapolated by nnz share x I={iters}" if det.get("block") else
                          f"{g.name}: full oracle CSR build ({det['t_build_s']:.2f} s) + T_0 ({det['t_init_s']:.2f} s) + "
                          f"one iteration over rows [0,{det['rows']}) = {det['nnz_sample']} of {nnz} nnz "
                          f"({det['t_sample_s']:.2f} s), iteration time extrapolated by nnz share x I={iters}"),
               "iter_rate": det["iter_rate"]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded generator, gen/)",
                "config": config_dict(g, world),
                "iteration": {"ms": spmm_ms, "nnz_d_per_s": nnz * d / (spmm_ms / 1e3),
                              "exchange_ms": (xms / max(iters, 1)) if world > 1 else 0.0},
                "nnz": nnz, "heavy_rows": info["heavy_rows"], "heavy_items": info["heavy_items"],
                "hot_rows": info["hot_rows"], "zero_rows": info["zero_rows"],
                "referenced_rows": info["referenced_rows"],
                "step_ms_each": [round(x, 3) for x in step_ms],
                "roofline": roofline, "secondary": secondary, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
