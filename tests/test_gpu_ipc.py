"""The real multi-process exchange on ONE GPU: two or three processes, each a rank of one handle,
collectives through the caller's host all-gather (gloo; NCCL refuses two ranks on one device), the
fused peer-store exchange through CUDA IPC mappings of each other's T buffers (X_PEER).

This runs, on hardware, what the loopback emulation cannot: cudaIpcGetMemHandle on blocks of the
library's block cache, cudaIpcOpenMemHandle in another process, stores through those mappings with
__threadfence_system, the barrier ordering of the steps (stream synchronise + host all-gather), the
mapping cache (a second handle of the same shape reuses the same blocks: no new IPC opens), and a
rank destroying its handle while the other still maps its blocks.  No kernel ever waits for another
process's kernel (the barrier is on the host), so the two ranks can share the GPU.  Every rank's
embedding must be BITWISE the 1-GPU result."""
import os
import socket
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist
    import gen
    import paper_2102_02302_b200 as cl
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        torch.cuda.set_device(0)
        ag = cl.host_allgather_from()
        g = gen.rmat_directed(8192, 13, 120000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=4)
        u = gen.chung_lu(20000, 60000, 2.1, 9.5388, 233115.5 * 20000 / 1134890, seed=2)
        res = []
        # (g, 1024): nnz = 14 N, so half-row passes with lazy steps (reading R21) through the peer mappings
        for gr, d, calls in ((g, 256, [3]), (g, 256, [1, 2]), (u, 1024, [4]), (u, 64, [2, 2]), (g, 1024, [4]),
                             (g, 1024, [1, 3])):
            opens0 = cl.cleora_ipc_opens()
            G = cl.cleora_build(gr.src, gr.dst, gr.w, gr.n, gr.directed, device=0, rank=rank, world=world,
                                host_allgather=ag)
            cl.cleora_init(G, d, 0)
            for k in calls:
                cl.cleora_iterate(G, k)
            info = cl.cleora_info(G)
            T = cl.cleora_fetch(G)
            res.append((gr.name, d, calls, info["exchange"], info["shard_begin"], info["shard_end"],
                        cl.cleora_ipc_opens() - opens0, T.tobytes()))
            if rank == 0:
                G.close()                 # the other ranks still map this rank's blocks (back in its cache)
            dist.barrier()
            if rank != 0:
                T2 = cl.cleora_fetch(G)   # their own replicas are untouched by rank 0's destroy
                assert T2.tobytes() == T.tobytes()
                G.close()
            dist.barrier()
        # 1-GPU references, computed by rank 0 in its own process
        # (the same call split: lazy steps are placed by the calls)
        if rank == 0:
            for gr, d, calls in ((g, 256, [3]), (u, 1024, [4]), (u, 64, [4]), (g, 1024, [4]), (g, 1024, [1, 3])):
                G = cl.cleora_build(gr.src, gr.dst, gr.w, gr.n, gr.directed, device=0)
                cl.cleora_init(G, d, 0)
                for k in calls:
                    cl.cleora_iterate(G, k)
                out[(gr.name, d, tuple(calls))] = cl.cleora_fetch(G).tobytes()
                G.close()
        q.put((rank, res, out))
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put((rank, "error", traceback.format_exc() + repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_processes_one_gpu_peer_exchange(world):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, res, out = q.get(timeout=900)
        assert res != "error", out
        got[rank] = (res, out)
    for p in procs:
        p.join(timeout=120)
    refs = got[0][1]
    for rank in range(world):
        res = got[rank][0]
        for i, (name, d, calls, mode, b, e, opens, T) in enumerate(res):
            assert mode == 2, f"rank {rank}: exchange mode {mode}, expected fused peer stores (2)"
            key = (name, d, tuple(calls)) if (name, d, tuple(calls)) in refs else (name, d, (sum(calls),))
            assert T == refs[key], f"rank {rank} {name} d={d} calls={calls}: differs from 1 GPU"
            if i == 1:      # same graph and d as case 0: the peer's blocks come back from its cache
                assert opens == 0, f"rank {rank}: {opens} new IPC mappings for a repeated handle"
        assert res[0][4] == (0 if rank == 0 else res[0][4]) and res[0][5] > res[0][4]


def _fail_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import gen
    import paper_2102_02302_b200 as cl
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), CLEORA_TEST_FAIL_T_RANK="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        ag = cl.host_allgather_from()
        g = gen.chung_lu(20000, 60000, 2.1, 9.5388, 233115.5 * 20000 / 1134890, seed=2)
        G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0, rank=rank, world=world, host_allgather=ag)
        try:
            cl.cleora_init(G, 256, 0)
            q.put((rank, "no error"))
        except cl.CleoraError as e:
            q.put((rank, str(e)))
        G.close()
    except Exception as e:
        q.put((rank, "unexpected: " + repr(e)))
    finally:
        dist.destroy_process_group()


def test_one_rank_failing_fails_every_rank():
    """Failure agreement: rank 1's T allocation fails (injected); instead of the others
    blocking in the next collective (the IPC handle exchange), every rank's cleora_init returns an
    error -- rank 1 its own, the others "rank 1 of 3 failed"."""
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_fail_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(3))
    for p in procs:
        p.join(timeout=60)
    assert "injected" in got[1], got
    assert "rank 1 of 3 failed" in got[0] and "rank 1 of 3 failed" in got[2], got
