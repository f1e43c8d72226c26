"""Row-sharded builds (world > 1) on one GPU, through the C ABI.

Loopback emulation (CLEORA_F_LOOPBACK) builds every emulated rank's shard exactly as a real rank
builds its own: the cuts come from the mirrored entry counts, and each shard's CSR is sorted, merged
and scaled from that rank's entries only.  Every shard must be BIT-EXACT against the
whole-graph oracle's rows [r0, r1) (tests/_shard.py restates the cut rule), the handle's whole-M facts
(nnz, zero rows, max degree) must be the oracle's, and the embeddings bitwise the 1-GPU result.
The deferred exchange (only gathered rows reach the peers before the last step of a call) is
checked against the undeferred one (CLEORA_NO_DEFER=1), bitwise.
"""
import numpy as np
import pytest

import gen
import oracle
from tests import _shard

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2102_02302_b200 as m
    return m


def _graphs():
    rng = np.random.default_rng(11)
    n = 5000
    hub = gen.EdgeList("hub", n, np.concatenate([np.zeros(4000, np.int32), rng.integers(0, n, 15000).astype(np.int32)]),
                       np.concatenate([np.arange(1, 4001, dtype=np.int32), rng.integers(0, n, 15000).astype(np.int32)]),
                       None, False)
    # weighted multigraph: duplicates (summed in input order, B2), self-loops (stored once, R5)
    s = rng.integers(0, 300, 6000).astype(np.int32)
    d = rng.integers(0, 300, 6000).astype(np.int32)
    d[:200] = s[:200]
    w = rng.lognormal(0, 1, 6000).astype(np.float32)
    multi = gen.EdgeList("multi", 400, s, d, w, False)
    return [gen.config("c1"), hub, multi,
            gen.rmat_directed(8192, 13, 120000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=4),
            gen.chung_lu(20000, 60000, 2.1, 9.5388, 233115.5 * 20000 / 1134890, seed=2)]


@pytest.mark.parametrize("world", [2, 3, 5])
def test_loopback_shards_bit_exact(cl, world):
    for g in _graphs():
        M = oracle.build_from(g)
        cuts = _shard.cuts(g, world)
        for p in range(world):
            G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0, loopback=True, world=world, rank=p)
            try:
                info = cl.cleora_info(G)
                csr = cl.cleora_fetch_csr(G)
            finally:
                G.close()
            r0, r1 = int(cuts[p]), int(cuts[p + 1])
            assert (info["shard_begin"], info["shard_end"]) == (r0, r1), (g.name, world, p)
            assert info["nnz"] == M.nnz and info["world"] == world
            assert info["zero_rows"] == int((M.row_ptr[1:] == M.row_ptr[:-1]).sum())
            assert info["max_degree"] == int(np.diff(M.row_ptr).max())
            a, b = int(M.row_ptr[r0]), int(M.row_ptr[r1])
            assert info["shard_nnz"] == b - a
            rp = csr["row_ptr"]
            assert not rp[:r0 + 1].any() and (rp[r1:] == b - a).all()
            assert np.array_equal(rp[r0:r1 + 1] + a, M.row_ptr[r0:r1 + 1])
            assert np.array_equal(csr["col"], M.col[a:b])
            assert csr["val"].tobytes() == M.val[a:b].tobytes(), f"{g.name} shard {p}/{world}: val not bit-exact"
            assert csr["deg"][r0:r1].tobytes() == M.deg[r0:r1].tobytes()
            assert not csr["deg"][:r0].any() and not csr["deg"][r1:].any()


def _close(a, b, tol=1e-5):
    """within the parity bars (max|d| <= 1e-5, cosine >= 0.99999 per non-zero row), same zero rows"""
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    assert np.abs(a64 - b64).max() <= tol
    nz = b64.any(1)
    assert np.array_equal(a64.any(1), nz)
    cos = (a64[nz] * b64[nz]).sum(1) / (np.linalg.norm(a64[nz], axis=1) * np.linalg.norm(b64[nz], axis=1))
    assert cos.min() >= 0.99999


def _embed(cl, g, d, calls, **kw):
    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0, **kw)
    try:
        cl.cleora_init(G, d, 0)
        for k in calls:
            cl.cleora_iterate(G, k)
        if kw.get("loopback"):
            return [cl.cleora_fetch_replica(G, p) for p in range(kw["world"])]
        return [cl.cleora_fetch(G)]
    finally:
        G.close()


@pytest.mark.parametrize("lazy", ["1", "0"])
@pytest.mark.parametrize("d", [96, 512, 1024])
def test_deferred_exchange_bitwise(cl, d, lazy, monkeypatch):
    """iterate(4) (3 deferred steps + a full one), iterate(1) x 4 (every step full) and the undeferred
    exchange all give every replica the 1-GPU bits -- with lazy half-row steps at d = 1024 (reading R21:
    the peers receive the unnormalised halves and the row scales like any row) and with every step
    normalised (CLEORA_LAZY=0)."""
    monkeypatch.setenv("CLEORA_LAZY", lazy)
    g = gen.rmat_directed(8192, 13, 120000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=4)   # 50% never-gathered rows
    ref = _embed(cl, g, d, [4])[0]
    for calls in ([4], [1, 1, 1, 1], [3, 1], [2, 2]):
        ref_c = ref if lazy == "0" or calls == [4] else _embed(cl, g, d, calls)[0]
        for T in _embed(cl, g, d, calls, loopback=True, world=3, rank=1):
            assert T.tobytes() == ref_c.tobytes(), calls
        _close(ref_c, ref)
    monkeypatch.setenv("CLEORA_NO_DEFER", "1")
    for T in _embed(cl, g, d, [4], loopback=True, world=3, rank=0):
        assert T.tobytes() == ref.tobytes()


def test_chunked_sharded_equals_single(cl):
    """A chunk (Algorithm 1, Q > 1) of a row-sharded build: the same rows, merge weights and bits."""
    g = gen.config("c1")
    G1 = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0, n_chunks=3, chunk=1, chunk_seed=5)
    cl.cleora_init(G1, 64, 0)
    cl.cleora_iterate(G1, 3)
    ref = cl.cleora_fetch(G1)
    G1.close()
    for T in _embed(cl, g, 64, [3], loopback=True, world=2, rank=0, n_chunks=3, chunk=1, chunk_seed=5):
        assert T.tobytes() == ref.tobytes()


@pytest.mark.parametrize("name,world", [("c2", 4), ("c4", 2)])
def test_full_size_sharded_bitwise(cl, name, world):
    """The bench configs row-sharded in loopback (every replica of every emulated rank) against one
    GPU, bitwise, on row blocks across the graph (host memory: a few GB per replica block); c4 with
    its lazy half-row steps (reading R21) on both sides."""
    import torch
    g = gen.config(name)
    dev = torch.device("cuda", 0)
    src, dst = torch.from_numpy(g.src).to(dev), torch.from_numpy(g.dst).to(dev)
    w = torch.from_numpy(g.w).to(dev) if g.w is not None else None
    blocks = [(0, 60000), (g.n // 2, g.n // 2 + 60000), (g.n - 60000, g.n)]
    G = cl.cleora_build(src, dst, w, g.n, g.directed, device=0)
    cl.cleora_init(G, g.d, 0)
    cl.cleora_iterate(G, g.iters)
    ref = [cl.cleora_fetch(G, a, b) for a, b in blocks]
    info1 = cl.cleora_info(G)
    G.close()
    cl.cleora_release_cached_memory()
    G = cl.cleora_build(src, dst, w, g.n, g.directed, device=0, loopback=True, world=world, rank=world - 1)
    try:
        cl.cleora_init(G, g.d, 0)
        cl.cleora_iterate(G, g.iters)
        info = cl.cleora_info(G)
        assert info["nnz"] == info1["nnz"] and info["zero_rows"] == info1["zero_rows"]
        for p in range(world):
            for (a, b), R in zip(blocks, ref):
                assert cl.cleora_fetch_replica(G, p, a, b).tobytes() == R.tobytes(), f"{name} replica {p} rows [{a},{b})"
    finally:
        G.close()
        cl.cleora_release_cached_memory()


@pytest.mark.parametrize("world", [3, 5, 8])
def test_degenerate_shards(cl, world):
    """More ranks than rows with entries: empty shards (no rows, or rows without entries), a shard made
    of one hub row, self-loops only -- every replica still bitwise the 1-GPU result, every shard's CSR
    bit-exact against the oracle's rows."""
    cases = [
        gen.EdgeList("three", 3, np.array([0, 1], np.int32), np.array([1, 2], np.int32), None, False),
        gen.EdgeList("loops", 6, np.arange(6, dtype=np.int32), np.arange(6, dtype=np.int32), None, True),
        gen.EdgeList("star", 2000, np.zeros(1999, np.int32), np.arange(1, 2000, dtype=np.int32),
                     np.linspace(0.5, 2.0, 1999).astype(np.float32), True),     # one row holds every entry
        gen.EdgeList("sparse", 50000, np.array([7, 49999], np.int32), np.array([49999, 7], np.int32), None, True),
    ]
    for g in cases:
        M = oracle.build_from(g)
        ref = _embed(cl, g, 33, [3])[0]
        for T in _embed(cl, g, 33, [2, 1], loopback=True, world=world, rank=world - 1):
            assert T.tobytes() == ref.tobytes(), g.name
        cuts = _shard.cuts(g, world)
        for p in range(world):
            G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0, loopback=True, world=world, rank=p)
            try:
                csr = cl.cleora_fetch_csr(G)
                info = cl.cleora_info(G)
            finally:
                G.close()
            r0, r1 = int(cuts[p]), int(cuts[p + 1])
            a, b = int(M.row_ptr[r0]), int(M.row_ptr[r1])
            assert (info["shard_begin"], info["shard_end"], info["shard_nnz"]) == (r0, r1, b - a), (g.name, p)
            assert np.array_equal(csr["col"], M.col[a:b]) and csr["val"].tobytes() == M.val[a:b].tobytes()
            assert np.array_equal(csr["row_ptr"][r0:r1 + 1] + a, M.row_ptr[r0:r1 + 1])
