"""Multi-rank (N > 1) host logic on CPU with the gloo backend, world_size 2 and 3.

The multi-GPU path row-shards M by nnz balance (cleora_plan_shards), every
rank computes normalize(M T) for its rows, and each iteration ends with an all-gather-v: one
broadcast per rank of its row block into every replica (exactly the NCCL calls of api.cu's
exchange()).  Here each rank computes its rows with the oracle and exchanges them with the same
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
        M = oracle.build_from(g)
        cuts = cl.cleora_plan_shards(M.row_ptr, world)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        T = torch.from_numpy(oracle.hash_init(g.n, cfg["d"], 0))
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
            ref = oracle.embed(M, cfg["d"], 0, cfg["iters"])
            q.put((T.numpy().tobytes() == ref.tobytes(), [int(c) for c in cuts]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "cl"), (3, "rmat")])
def test_sharded_iteration_equals_single_process(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    cfg = dict(kind=kind, seed=world, d=16, iters=3)
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
