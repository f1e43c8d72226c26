"""The multi-GPU path on one GPU: loopback emulation of `world` ranks (CLEORA_F_LOOPBACK).

Each emulated rank owns a full replica pair and computes its nnz-balanced row shard with the
SAME fused kernel the real multi-GPU path runs; its epilogue stores every finished row into all
replicas (on a real box these are NVLink peer pointers opened with CUDA IPC).  The ranks run one
after another, so no launch ever waits for another (task rule: no cross-rank spinning on one
GPU).  SURVEY.md §8(e): per-row arithmetic does not depend on the number of GPUs, so every
replica must be BITWISE equal to the 1-GPU result, which is itself held to the oracle.
Also: rows without out-edges are not rewritten once both buffers hold their zeros -- the
result is bitwise the same as rewriting them (CLEORA_WRITE_ZERO_ROWS=1).
"""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2102_02302_b200 as m
    return m


def _graphs():
    rng = np.random.default_rng(7)
    n = 6000
    # a hub (5000 leaves) plus random edges: heavy items, shard cuts inside the hub's row range
    hub = gen.EdgeList("hub", n, np.concatenate([np.zeros(5000, np.int32), rng.integers(0, n, 20000).astype(np.int32)]),
                       np.concatenate([np.arange(1, 5001, dtype=np.int32), rng.integers(0, n, 20000).astype(np.int32)]),
                       None, False)
    rm = gen.rmat_directed(8192, 13, 120000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=4)   # sinks, weights
    return [gen.config("c1"), hub, rm,
            gen.chung_lu(20000, 60000, 2.1, 9.5388, 233115.5 * 20000 / 1134890, seed=2)]


def _run(cl, g, d, iters, **kw):
    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0, **kw)
    try:
        cl.cleora_init(G, d, 0)
        cl.cleora_iterate(G, iters)
        if kw.get("loopback"):
            return [cl.cleora_fetch_replica(G, p) for p in range(kw["world"])], cl.cleora_info(G)
        return cl.cleora_fetch(G), cl.cleora_info(G)
    finally:
        G.close()


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("d", [64, 256, 1100])
def test_loopback_replicas_equal_single_gpu(cl, world, d):
    for g in _graphs():
        ref, _ = _run(cl, g, d, 3)
        reps, info = _run(cl, g, d, 3, loopback=True, world=world, rank=world - 1)
        assert info["world"] == world
        for p, T in enumerate(reps):
            assert T.tobytes() == ref.tobytes(), f"{g.name} world={world} d={d}: replica {p} differs from 1 GPU"


def test_loopback_parity_and_shards(cl):
    g = gen.config("c1")
    M = oracle.build_from(g)
    R = oracle.embed(M, 128, 0, 4)
    reps, info = _run(cl, g, 128, 4, loopback=True, world=4, rank=2)
    cuts = cl.cleora_plan_shards(M.row_ptr, 4)
    assert (info["shard_begin"], info["shard_end"]) == (cuts[2], cuts[3])
    err = float(np.abs(reps[2].astype(np.float64) - R).max())
    assert err <= 1e-5


def test_zero_rows_not_rewritten_same_bytes(cl, monkeypatch):
    """Directed R-MAT: about half the rows have no out-edges.  Split iterate calls, a set_rows in
    between (which makes the current buffer's zero rows dirty), with and without the skip."""
    g = gen.rmat_directed(8192, 13, 60000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=9)
    outs = []
    for write_all in (False, True):
        if write_all:
            monkeypatch.setenv("CLEORA_WRITE_ZERO_ROWS", "1")
        G = cl.cleora_build(g.src, g.dst, g.w, g.n, True, device=0)
        cl.cleora_init(G, 96, 3)
        cl.cleora_iterate(G, 3)
        T = cl.cleora_fetch(G)
        T[:500] = 0.25                      # overwrite rows, zero rows included
        cl.cleora_set_rows(G, 0, T[:500])
        cl.cleora_iterate(G, 1)
        cl.cleora_iterate(G, 2)
        outs.append(cl.cleora_fetch(G))
        info = cl.cleora_info(G)
        G.close()
    assert info["zero_rows"] > 1000
    assert outs[0].tobytes() == outs[1].tobytes()
    M = oracle.build_from(g)
    R = oracle.embed(M, 96, 3, 3)
    R[:500] = 0.25
    for _ in range(3):
        R = oracle.step(M, R)
    assert float(np.abs(outs[0].astype(np.float64) - R).max()) <= 1e-5
    assert np.array_equal(~outs[0].any(1), ~R.any(1))


def _nccl_worker(rank, world, port, exchange_nccl, q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import gen as gen_
    import paper_2102_02302_b200 as cl_
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        obj = [cl_.cleora_nccl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        g = gen_.chung_lu(20000, 60000, 2.1, 9.5388, 233115.5 * 20000 / 1134890, seed=2)
        outs = []
        for _ in range(2):   # a second handle from the same unique id reuses the communicator
            G = cl_.cleora_build(g.src, g.dst, None, g.n, False, device=rank, rank=rank, world=world,
                                 nccl_id=obj[0], exchange_nccl=exchange_nccl)
            cl_.cleora_init(G, 256, 0)
            cl_.cleora_iterate(G, 3)
            outs.append(cl_.cleora_fetch(G))
            mode = cl_.cleora_info(G)["exchange"]
            G.close()
        assert outs[0].tobytes() == outs[1].tobytes()
        q.put((rank, mode, outs[1].tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange_nccl", [False, True])
def test_real_multi_gpu_if_available(cl, exchange_nccl):
    """On a box with >= 2 GPUs: torchrun-style ranks over NCCL, the fused peer-store exchange (or
    the NCCL all-gather fallback); every rank's replica is bitwise the 1-GPU result."""
    import socket
    import torch
    import torch.multiprocessing as mp
    world = min(4, torch.cuda.device_count())
    if world < 2:
        pytest.skip("needs >= 2 GPUs (this pool has one; covered by the loopback tests above)")
    g = gen.chung_lu(20000, 60000, 2.1, 9.5388, 233115.5 * 20000 / 1134890, seed=2)
    ref, _ = _run(cl, g, 256, 3)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nccl_worker, args=(r, world, port, exchange_nccl, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, mode, T in res:
        assert mode == 1 if exchange_nccl else mode in (1, 2)      # 2: peer stores, 1: NCCL (fallback)
        assert T == ref.tobytes(), f"rank {rank} (exchange mode {mode}) differs from 1 GPU"
