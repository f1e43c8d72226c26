"""Multi-rank (N > 1) host logic on CPU with the gloo backend, world_size 2 and 3.

The multi-GPU path row-shards M by nnz balance (cleora_plan_shards), every rank
computes normalize(M T) for its rows, and the rows reach every replica either through the fused
peer stores of the SpMM epilogue (protocol "peer": stores into all replicas, empty rows skipped once
clean, a barrier per step) or through the NCCL fallback, an all-gather-v of one broadcast per rank
(protocol "nccl", exactly the calls of api.cu's exchange()).  Here each rank computes its rows with the oracle and exchanges them with the same
protocol over gloo; the result must be bitwise equal to the single-process oracle, which pins
the cut planning, the exchange offsets and the row independence the sharding relies on.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        import oracle
        import paper_2102_02302_b200 as cl
        g = gen.chung_lu(3000, 9000, 2.1, 9.5388, 233115.5 * 3000 / 1134890, seed=cfg["seed"]) \
            if cfg["kind"] == "cl" else gen.rmat_directed(2048, 11, 20000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=cfg["seed"])
        M_full = oracle.build_from(g)
        if cfg.get("cuts") == "entries":
            # the row-sharded build (cleora_build, world > 1): cuts from the mirrored entry counts,
            # and this rank builds M from its rows' entries only; its rows must be bit-identical
            # to the whole M's, and the rest empty
            from tests import _shard
            cuts = _shard.cuts(g, world)
            r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
            s_, d_, w_ = _shard.shard_edges(g, r0, r1)
            M = oracle.build_csr(s_, d_, w_, g.n, True)
            a, b = int(M_full.row_ptr[r0]), int(M_full.row_ptr[r1])
            assert np.array_equal(M.row_ptr[r0:r1 + 1] + a, M_full.row_ptr[r0:r1 + 1])
            assert M.row_ptr[r0] == 0 and M.row_ptr[-1] == b - a
            assert np.array_equal(M.col, M_full.col[a:b])
            assert M.val.tobytes() == M_full.val[a:b].tobytes()
            assert M.deg[r0:r1].tobytes() == M_full.deg[r0:r1].tobytes()
            assert not M.deg[:r0].any() and not M.deg[r1:].any()
        else:
            M = M_full
            cuts = cl.cleora_plan_shards(M.row_ptr, world)
            r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        T = torch.from_numpy(oracle.hash_init(g.n, cfg["d"], 0))
        if cfg.get("protocol") == "peer":
            T = _peer_protocol(M, T, cuts, rank, world, cfg["iters"])
            if rank == 0:
                ref = oracle.embed(M_full, cfg["d"], 0, cfg["iters"])
                q.put((T.numpy().tobytes() == ref.tobytes(), [int(c) for c in cuts]))
            return
        for _ in range(cfg["iters"]):
            out = torch.empty_like(T)
            out[r0:r1] = torch.from_numpy(oracle.step(M, T.numpy(), r0, r1))
            # all-gather-v: every rank broadcasts its block [cuts[p], cuts[p+1]) in place
            for p in range(world):
                b, e = int(cuts[p]), int(cuts[p + 1])
                if e > b:
                    blk = out[b:e].contiguous()
                    dist.broadcast(blk, src=p)
                    out[b:e] = blk
            T = out
        if rank == 0:
            ref = oracle.embed(M_full, cfg["d"], 0, cfg["iters"])
            q.put((T.numpy().tobytes() == ref.tobytes(), [int(c) for c in cuts]))
    finally:
        dist.destroy_process_group()


def _peer_protocol(M, T0, cuts, rank, world, iters):
    """The fused exchange of api.cu (X_PEER) on CPU: each rank holds two replica buffers; in a
    step it computes its rows [cuts[rank], cuts[rank+1]) from its replica of T_in and stores them
    into EVERY rank's replica of T_out (here: all_gather_object of the stored rows), skipping rows
    without entries once that buffer already holds their zeros (zclean bookkeeping), then a
    barrier orders the steps.  Buffer 1 starts as garbage, so a missed store shows."""
    import oracle
    bufs = [T0.clone(), torch.full_like(T0, 7.0)]
    zclean = [False, False]
    cur = 0
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    empty = (M.row_ptr[1:] == M.row_ptr[:-1])[r0:r1]
    for _ in range(iters):
        out = 1 - cur
        mine = oracle.step(M, bufs[cur].numpy(), r0, r1)
        write = ~empty if zclean[out] else np.ones(r1 - r0, bool)
        stores = [None] * world
        dist.all_gather_object(stores, (r0, r1, write, mine[write]))
        for b, e, w, vals in stores:
            blk = bufs[out][b:e]
            blk[torch.from_numpy(w)] = torch.from_numpy(vals)
        dist.barrier()
        zclean[out] = True
        cur = out
    return bufs[cur]


@pytest.mark.parametrize("world,kind,protocol,cut", [(2, "cl", "nccl", "nnz"), (3, "rmat", "nccl", "nnz"),
                                                     (2, "rmat", "peer", "nnz"), (3, "cl", "peer", "nnz"),
                                                     (2, "cl", "peer", "entries"), (3, "rmat", "peer", "entries"),
                                                     (4, "rmat", "nccl", "entries")])
def test_sharded_iteration_equals_single_process(world, kind, protocol, cut):
    """Each rank holds only its shard's CSR when cut == "entries" (the row-sharded build)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    cfg = dict(kind=kind, seed=world, d=16, iters=4, protocol=protocol, cuts=cut)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    same, cuts = q.get(timeout=10)
    assert same, f"sharded result differs (cuts {cuts})"
    assert cuts[0] == 0 and len(cuts) == world + 1
