"""cleora_fetch_nonzero: the result without the rows that are 0 by construction -- needs a B200.

A row of M without entries has y = 0 in every step (Algorithm 1 line 7; reading RZ), so
after the first step it is exactly 0 in T.  The compact fetch must return exactly the rows with
entries (ids from the ORACLE's CSR), each bitwise equal to the dense fetch's row (itself checked
against the oracle within the north-star bars), and every row it leaves out must be exactly 0 in the
dense fetch.  Before the first step and after cleora_set_rows every row comes back.  Covered: several
staging slices (> 256 MB of rows), the asynchronous form with cleora_trim (bench.py's e2e pipeline),
device outputs, rows of d not a multiple of 4, row shards (loopback), and the usage errors.
"""
import numpy as np
import pytest

import gen
import oracle
from tests import _shard
from tests.test_gpu_parity import compare, ill_conditioned

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2102_02302_b200 as m
    return m


def _rows_with_entries(M, r0=0, r1=None):
    r1 = M.n if r1 is None else r1
    nz = np.flatnonzero(np.diff(M.row_ptr) > 0).astype(np.int32)
    return nz[(nz >= r0) & (nz < r1)]


def _check(cl, G, M, stepped, r0=0, r1=None):
    r1 = M.n if r1 is None else r1
    dense = cl.cleora_fetch(G)
    rows, ids = cl.cleora_fetch_nonzero(G)
    want = _rows_with_entries(M, r0, r1) if stepped else np.arange(r0, r1, dtype=np.int32)
    assert np.array_equal(ids, want), "ids are not the rows with entries"
    assert cl.cleora_nonzero_count(G) == want.size
    assert np.array_equal(rows.view(np.uint32), dense[ids].view(np.uint32)), "packed rows differ from T"
    if stepped:
        rest = np.ones(M.n, bool)
        rest[ids] = False
        rest[:r0] = rest[r1:] = False
        assert not dense[rest].any(), "a row left out is not 0"
    return dense


@pytest.mark.parametrize("seed", range(24))
def test_tiny_graphs(cl, seed):
    g = gen.tiny_graph(seed)
    d = [1, 3, 4, 5, 8, 33, 128, 1024][seed % 8]
    M = oracle.build_from(g)
    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
    try:
        cl.cleora_init(G, d, seed)
        R = oracle.hash_init(g.n, d, seed)
        T = _check(cl, G, M, stepped=False)
        assert np.array_equal(T.view(np.uint32), R.view(np.uint32))
        for k in (1, 2):
            ok = not ill_conditioned(M, R)
            cl.cleora_iterate(G, k)
            for _ in range(k):
                ok = ok and not ill_conditioned(M, R)
                R = oracle.step(M, R)
            T = _check(cl, G, M, stepped=True)
            if ok:
                compare(T, R, f"{g.name} d={d}")
    finally:
        G.close()


@pytest.mark.parametrize("slices", ["0", "1"])
def test_directed_sinks_several_slices_async_trim_and_device_outputs(cl, slices, monkeypatch):
    """A directed R-MAT graph (most rows are sinks, c4's kind) at d = 1024 whose rows with entries
    exceed one 256 MB staging slice; the async form into pinned memory followed by cleora_trim (the
    bench's e2e pipeline) and the device-output form give the same bits as the synchronous fetch.
    slices = "1": the sliced path (CLEORA_FETCH_SLICES=1) instead of one whole-result staging buffer."""
    import torch
    monkeypatch.setenv("CLEORA_FETCH_SLICES", slices)
    g = gen.rmat_directed(400_000, 19, 1_600_000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=7)
    M = oracle.build_from(g)
    want = _rows_with_entries(M)
    assert want.size * 1024 * 4 > (256 << 20) and want.size < g.n
    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
    try:
        cl.cleora_init(G, 1024, 3)
        cl.cleora_iterate(G, 2)
        R = oracle.step(M, oracle.step(M, oracle.hash_init(g.n, 1024, 3)))
        compare(_check(cl, G, M, stepped=True), R, "rmat d=1024")
        rows_s, ids_s = cl.cleora_fetch_nonzero(G)
        rd = torch.empty((want.size, 1024), dtype=torch.float32, device="cuda:0")
        idd = torch.empty(want.size, dtype=torch.int32, device="cuda:0")
        cl.cleora_fetch_nonzero(G, rd, idd)
        assert np.array_equal(rd.cpu().numpy().view(np.uint32), rows_s.view(np.uint32))
        assert np.array_equal(idd.cpu().numpy(), ids_s)
    finally:
        G.close()
    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
    try:
        cl.cleora_init(G, 1024, 3)
        cl.cleora_iterate(G, 2)
        rp = torch.empty((want.size, 1024), dtype=torch.float32).pin_memory()
        ip = torch.empty(want.size, dtype=torch.int32).pin_memory()
        cl.cleora_fetch_nonzero_async(G, rp, ip)
        cl.cleora_trim(G)
        cl.cleora_sync(G)
        assert np.array_equal(rp.numpy().view(np.uint32), rows_s.view(np.uint32))
        assert np.array_equal(ip.numpy(), ids_s)
        # the selection survives the trim: a second call after it still answers
        r2, i2 = cl.cleora_fetch_nonzero(G)
        assert np.array_equal(r2.view(np.uint32), rows_s.view(np.uint32)) and np.array_equal(i2, ids_s)
    finally:
        G.close()


def test_set_rows_returns_every_row_until_the_next_step(cl):
    g = gen.rmat_directed(4096, 12, 20000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=2)
    M = oracle.build_from(g)
    sink = int(np.flatnonzero(np.diff(M.row_ptr) == 0)[0])
    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
    try:
        cl.cleora_init(G, 64, 0)
        cl.cleora_iterate(G, 1)
        _check(cl, G, M, stepped=True)
        cl.cleora_set_rows(G, sink, np.ones((1, 64), np.float32))
        T = _check(cl, G, M, stepped=False)
        assert (T[sink] == 1).all()
        cl.cleora_iterate(G, 1)
        _check(cl, G, M, stepped=True)
    finally:
        G.close()


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_shards(cl, world):
    """Each rank returns its own shard's rows with entries; together the ranks cover the graph."""
    g = gen.rmat_directed(8192, 13, 60000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=4)
    M = oracle.build_from(g)
    cuts = _shard.cuts(g, world)
    got = []
    for p in range(world):
        G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0, loopback=True, world=world, rank=p)
        try:
            cl.cleora_init(G, 128, 1)
            cl.cleora_iterate(G, 2)
            _check(cl, G, M, stepped=True, r0=int(cuts[p]), r1=int(cuts[p + 1]))
            got.append(cl.cleora_fetch_nonzero(G)[1])
        finally:
            G.close()
    assert np.array_equal(np.concatenate(got), _rows_with_entries(M))


def test_c4_full(cl):
    """The bench configuration: iterate(4) in one call, then the compact fetch -- ids bit-exact against
    the oracle's CSR, rows bitwise the dense fetch's (whose parity test_gpu_parity.py::test_c4_full
    checks), every row left out exactly 0."""
    import torch
    g = gen.config("c4")
    M = oracle.build_from(g)
    want = _rows_with_entries(M)
    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
    try:
        cl.cleora_init(G, g.d, 0)
        cl.cleora_iterate(G, g.iters)
        rp = torch.empty((want.size, g.d), dtype=torch.float32).pin_memory()
        ip = torch.empty(want.size, dtype=torch.int32).pin_memory()
        rows, ids = cl.cleora_fetch_nonzero(G, rp, ip)
        assert np.array_equal(ids.numpy(), want)
        chunk = 1 << 16
        for r0 in range(0, g.n, chunk):
            T = cl.cleora_fetch(G, r0, min(g.n, r0 + chunk))
            a, b = np.searchsorted(want, [r0, r0 + chunk])
            assert np.array_equal(rows[a:b].numpy().view(np.uint32), T[want[a:b] - r0].view(np.uint32))
            rest = np.ones(T.shape[0], bool)
            rest[want[a:b] - r0] = False
            assert not T[rest].any()
    finally:
        G.close()


def test_usage_errors(cl):
    g = gen.rmat_directed(4096, 12, 20000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=3)
    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
    try:
        cl.cleora_init(G, 16, 0)
        cl.cleora_iterate(G, 1)
        n = cl.cleora_nonzero_count(G)
        assert 0 < n < g.n
        with pytest.raises(cl.CleoraError):
            cl.cleora_fetch_nonzero(G, np.empty((n - 1, 16), np.float32), np.empty(n - 1, np.int32))
        cl.cleora_trim(G)
        with pytest.raises(cl.CleoraError):         # trimmed before the rows were selected
            cl.cleora_fetch_nonzero(G)
    finally:
        G.close()
