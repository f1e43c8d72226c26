"""Measurement of the SURVEY §8(f) rows on one B200 (one JSON line):

f1 -- chunked embedding of c2 with Q chunks: per-chunk build + init + I iterations, then
      cleora_merge_chunks into device memory.  The merge kernel is HBM-bound: its algorithmic
      bytes are Q*N*dp*4 (chunk rows read) + Q*N*4 (occurrences) + N*dp*4 (merged rows written);
      achieved = bytes / (CUDA-event time of the merge call, device output, no D2H).
f2 -- cleora_reconstruct of n_new unseen nodes against c2's T_{I-1}, device inputs and output:
      new nodes/s and nnz*d/s of the one fused SpMM step it runs.
f3 -- the paper's pipeline for YouTube: every adjacency row of c2 (node v and its
      neighbours, non-isolated nodes) as a hyperedge, star-expanded on the device, then build + init
      + I iterations of the expanded graph (d = 1024); and c1's rows clique-expanded.
f4 -- many small graphs (2,000 Erdos-Renyi graphs, N log-uniform in [50, 5000], 4N edges each,
      d = 128, I = 4): one batched handle (block-diagonal M, one launch per step) against the same
      graphs one handle at a time (a prefix of 200 graphs, scaled), device-resident inputs.
Usage: python scripts/bench_next.py [--chunks 4] [--new 200000] [--reps 5]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2102_02302_b200 as cl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--chunks", type=int, default=4)
ap.add_argument("--new", type=int, default=200_000)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6650.0
g = gen.config(args.config)
d, iters, Q = g.d, g.iters, args.chunks
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
src, dst = torch.from_numpy(g.src).to(dev), torch.from_numpy(g.dst).to(dev)
w = torch.from_numpy(g.w).to(dev) if g.w is not None else None
torch.cuda.synchronize()


def ev():
    return torch.cuda.Event(enable_timing=True)


# ---------------------------------------------------------------- f1
hs = []
e0, e1 = ev(), ev()
e0.record(s)
for q in range(Q):
    G = cl.cleora_build(src, dst, w, g.n, g.directed, device=0, stream=s.cuda_stream, n_chunks=Q, chunk=q, chunk_seed=1)
    cl.cleora_init(G, d, 0)
    cl.cleora_iterate(G, iters)
    hs.append(G)
e1.record(s)
e1.synchronize()
chunks_ms = e0.elapsed_time(e1)
nnz_chunks = sum(cl.cleora_info(G)["nnz"] for G in hs)
out = torch.empty((g.n, d), dtype=torch.float32, device=dev)
cl.cleora_merge_chunks(hs, out)            # warm-up
ts = []
for _ in range(args.reps):
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(s)
    cl.cleora_merge_chunks(hs, out)        # enqueued on chunk 0's stream (s), synchronous
    b.record(s)
    b.synchronize()
    ts.append(a.elapsed_time(b))
merge_ms = min(ts)
dp = (d + 3) // 4 * 4
merge_bytes = Q * g.n * dp * 4 + Q * g.n * 4 + g.n * dp * 4
for G in hs:
    G.close()
del out

# ---------------------------------------------------------------- f2
rng = np.random.default_rng(0)
deg = np.bincount(np.concatenate([g.src, g.dst]), minlength=g.n)
k = rng.geometric(1 / max(1.0, deg[deg > 0].mean()), args.new).astype(np.int64)      # new-node degrees
new_idx = torch.from_numpy(np.repeat(np.arange(args.new, dtype=np.int32), k)).to(dev)
p = deg / deg.sum()                                                                   # preferential attachment
known = torch.from_numpy(rng.choice(g.n, int(k.sum()), p=p).astype(np.int32)).to(dev)
G = cl.cleora_build(src, dst, w, g.n, g.directed, device=0, stream=s.cuda_stream)
cl.cleora_init(G, d, 0)
cl.cleora_iterate(G, iters - 1)
rout = torch.empty((args.new, d), dtype=torch.float32, device=dev)
cl.cleora_reconstruct(G, new_idx, known, None, args.new, rout)
ts = []
for _ in range(args.reps):
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(s)
    cl.cleora_reconstruct(G, new_idx, known, None, args.new, rout)
    b.record(s)
    b.synchronize()
    ts.append(a.elapsed_time(b))
rec_ms = min(ts)
G.close()

# ---------------------------------------------------------------- f3
def rows_as_hyperedges(x):
    Gx = cl.cleora_build(x.src, x.dst, None, x.n, x.directed, device=0)
    csr = cl.cleora_fetch_csr(Gx)
    Gx.close()
    rp, col = csr["row_ptr"], csr["col"]
    k = np.diff(rp)
    live = np.flatnonzero(k > 0)
    ptr = np.concatenate([[0], np.cumsum(k[live] + 1)]).astype(np.int64)
    nodes = np.empty(ptr[-1], np.int32)
    nodes[ptr[:-1]] = live                                   # the row's own node first
    mask = np.ones(ptr[-1], bool)
    mask[ptr[:-1]] = False
    nodes[mask] = np.concatenate([col[rp[v]:rp[v + 1]] for v in live]) if live.size < 20000 else \
        col[np.concatenate([np.arange(rp[v], rp[v + 1]) for v in live])]
    return torch.from_numpy(ptr).to(dev), torch.from_numpy(nodes).to(dev), x.n


f3 = {}
for name, x, mode, d3 in (("c2_star", g, cl.EXPAND_STAR, 1024), ("c1_clique", gen.config("c1"), cl.EXPAND_CLIQUE, 128)):
    hp, hn, n0 = rows_as_hyperedges(x)
    es, ed = cl.cleora_expand(hp, hn, n0, mode, stream=s.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        a, b = ev(), ev()
        a.record(s)
        es, ed = cl.cleora_expand(hp, hn, n0, mode, stream=s.cuda_stream)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    nn = n0 + (hp.numel() - 1 if mode == cl.EXPAND_STAR else 0)
    pts = []
    for _ in range(3):                  # the first run allocates the expanded graph's buffers
        a, b = ev(), ev()
        a.record(s)
        es, ed = cl.cleora_expand(hp, hn, n0, mode, stream=s.cuda_stream)
        G3 = cl.cleora_build(es, ed, None, nn, False, device=0, stream=s.cuda_stream)
        cl.cleora_init(G3, d3, 0)
        cl.cleora_iterate(G3, 4)
        b.record(s)
        b.synchronize()
        pts.append(a.elapsed_time(b))
        nnz3 = cl.cleora_info(G3)["nnz"]
        G3.close()
    print(f"f3 {name} pipeline ms per run: {pts}", file=sys.stderr)
    f3[name] = {"hyperedges": hp.numel() - 1, "members": int(hn.numel()), "expanded_edges": int(es.numel()),
                "expanded_nodes": nn, "nnz": nnz3, "d": d3, "expand_ms": min(ts),
                "expanded_edges_per_s": es.numel() / (min(ts) / 1e3),
                "pipeline_ms": min(pts[1:]), "pipeline_first_run_ms": pts[0],
                "pipeline": "expand + build + init + 4 iterations (min of 2 runs after a first, allocating one)"}

# ---------------------------------------------------------------- f4
rng = np.random.default_rng(1)
ns = np.exp(rng.uniform(np.log(50), np.log(5000), 2000)).astype(np.int64)
graphs = [gen.er(int(n), int(4 * n), seed=100 + i) for i, n in enumerate(ns)]
ep = np.zeros(len(graphs) + 1, np.int64)
ep[1:] = np.cumsum([x.n_edges for x in graphs])
bsrc = torch.from_numpy(np.concatenate([x.src for x in graphs])).to(dev)
bdst = torch.from_numpy(np.concatenate([x.dst for x in graphs])).to(dev)
nc = np.array([x.n for x in graphs], np.int32)
d4, it4 = 128, 4


def batch_step(timing=False):
    B = cl.cleora_build_batch(bsrc, bdst, None, ep, nc, False, device=0, stream=s.cuda_stream, timing=timing)
    cl.cleora_init(B, d4, 0)
    cl.cleora_iterate(B, it4)
    return B


batch_step().close()
ts = []
for _ in range(args.reps):
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(s)
    B = batch_step()
    B.close()
    b.record(s)
    b.synchronize()
    ts.append(a.elapsed_time(b))
batch_ms = min(ts)
B = batch_step(timing=True)
st = cl.cleora_stats(B)
info = cl.cleora_info(B)
B.close()
nnz4 = info["nnz"]
spmm4 = st["spmm_ms_total"] / max(1, st["spmm_launches"])
b4 = 8 * (info["n_nodes"] + 1) + 8 * nnz4 + 2 * info["n_nodes"] * d4 * 4
gs = [(torch.from_numpy(x.src).to(dev), torch.from_numpy(x.dst).to(dev), x.n) for x in graphs[:200]]
torch.cuda.synchronize()
a, b = ev(), ev()
a.record(s)
for xs, xd, xn in gs:
    G = cl.cleora_build(xs, xd, None, xn, False, device=0, stream=s.cuda_stream)
    cl.cleora_init(G, d4, 0)
    cl.cleora_iterate(G, it4)
    G.close()
b.record(s)
b.synchronize()
seq_ms = a.elapsed_time(b) * len(graphs) / len(gs)

line = {"what": "SURVEY 8(f) f1 chunked embedding + merge, f2 inductive reconstruction, f3 expansion, f4 batched graphs",
        "config": g.name, "d": d,
        "f1": {"chunks": Q, "nnz_all_chunks": nnz_chunks, "chunks_build_init_iterate_ms": chunks_ms,
               "merge_ms": merge_ms, "merge_bytes": merge_bytes,
               "merge_roofline": {"bound": "hbm", "achieved": merge_bytes / (merge_ms / 1e3) / 1e9, "peak": peak,
                                  "unit": "GB/s", "frac": merge_bytes / (merge_ms / 1e3) / 1e9 / peak}},
        "f2": {"new_nodes": args.new, "edges": int(k.sum()), "ms": rec_ms, "new_nodes_per_s": args.new / (rec_ms / 1e3),
               "nnz_d_per_s": int(k.sum()) * d / (rec_ms / 1e3),
               "includes": "device-side CSR build of the new nodes' rows + one fused SpMM step + D2D copy"},
        "f3": f3,
        "f4": {"graphs": len(graphs), "nodes": info["n_nodes"], "nnz": nnz4, "d": d4, "iterations": it4,
               "batched_step_ms": batch_ms, "batched_graphs_per_s": len(graphs) / (batch_ms / 1e3),
               "batched_nnz_d_per_s": nnz4 * d4 * it4 / (batch_ms / 1e3),
               "one_at_a_time_ms": seq_ms, "speedup": seq_ms / batch_ms,
               "spmm_ms_per_launch": spmm4,
               "spmm_roofline": {"bound": "hbm", "achieved": b4 / (spmm4 / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                                 "frac": b4 / (spmm4 / 1e3) / 1e9 / peak}}}
print(json.dumps(line), flush=True)
