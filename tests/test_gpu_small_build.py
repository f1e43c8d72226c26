"""The one-kernel build of small graphs (build.cu k_build_small) against the general build and the
oracle -- needs a B200.

Small whole graphs (<= 2^21 mirrored entries, no row longer than 256 entries) are built by one
cooperative kernel instead of ~20 launches (validate, radix sort, run merge, row pointer, degree,
values).  Both paths must give the SAME bytes: row_ptr, col, val bits, deg bits (readings B1-B4 of
DESIGN §2: stable (src, dst) order, run sums in list order, sequential degree fold, one rounding of
e_ab / deg -- PAPER.md:79-81), the same graph facts (entries, zero rows, longest row) and the same
error verdicts.  A graph with a longer row falls back to the general path inside the same call.
``CLEORA_SMALL_BUILD=0`` forces the general path.
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


def _build(cl, g, small, monkeypatch):
    monkeypatch.setenv("CLEORA_SMALL_BUILD", "1" if small else "0")
    n0 = cl.cleora_kernel_launches()
    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
    launches = cl.cleora_kernel_launches() - n0
    try:
        csr = cl.cleora_fetch_csr(G)
        info = cl.cleora_info(G)
    finally:
        G.close()
    return csr, {k: info[k] for k in ("nnz", "zero_rows", "max_degree")}, launches


def _same(a, b, what):
    assert np.array_equal(a["row_ptr"], b["row_ptr"]), f"{what}: row_ptr"
    assert np.array_equal(a["col"], b["col"]), f"{what}: col"
    assert a["val"].view(np.uint32).tobytes() == b["val"].view(np.uint32).tobytes(), f"{what}: val bits"
    assert a["deg"].view(np.uint64).tobytes() == b["deg"].view(np.uint64).tobytes(), f"{what}: deg bits"


def _row_graph(n, length, directed, weighted, seed):
    """node 0 with `length` out-entries (after mirroring), duplicates among them, plus a random tail."""
    rng = np.random.default_rng(seed)
    per = length if directed else length
    src = np.concatenate([np.zeros(per, np.int32), rng.integers(1, n, 300).astype(np.int32)])
    dst = np.concatenate([rng.integers(1, n, per).astype(np.int32), rng.integers(1, n, 300).astype(np.int32)])
    w = rng.lognormal(0, 1, src.size).astype(np.float32) if weighted else None
    return gen.EdgeList(f"row{length}", n, src, dst, w, directed)


def _graphs():
    gs = [gen.tiny_graph(s, n_max=400, e_max=3000) for s in range(40)]
    gs += [gen.tiny_graph(500 + s, n_max=20, e_max=400) for s in range(10)]     # many duplicates per row
    rng = np.random.default_rng(3)
    # heavy duplication with lognormal weights: run sums in list order decide the bits
    s = rng.integers(0, 60, 3000).astype(np.int32)
    d = rng.integers(0, 60, 3000).astype(np.int32)
    gs.append(gen.EdgeList("dups", 60, s, d, rng.lognormal(0, 2, 3000).astype(np.float32), False))
    gs.append(gen.EdgeList("dups_dir", 60, s, d, rng.lognormal(0, 2, 3000).astype(np.float32), True))
    gs.append(gen.EdgeList("dups_long", 30, s % 30, d % 30, rng.lognormal(0, 2, 3000).astype(np.float32), False))
    gs.append(gen.EdgeList("selfloops", 5, np.arange(5, dtype=np.int32), np.arange(5, dtype=np.int32), None, False))
    gs.append(gen.EdgeList("one", 1, np.zeros(1, np.int32), np.zeros(1, np.int32), None, True))
    gs.append(gen.EdgeList("isolated", 100000, np.array([7, 99999], np.int32), np.array([99999, 7], np.int32),
                           None, True))
    gs.append(gen.er(30001, 90000, seed=4))
    gs.append(gen.rmat_directed(8192, 13, 50000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=5))
    gs.append(gen.lattice(90, 0.3, 0.02, seed=6))
    for length in (255, 256):                                  # the longest row the kernel sorts
        for directed in (False, True):
            gs.append(_row_graph(2000, length, directed, True, length))
    return gs


def _longest_row(g):
    """entries of the longest row after mirroring, before merging (what the one-kernel build sorts)"""
    r = g.src if g.directed else np.concatenate([g.src, g.dst[g.src != g.dst]])
    return int(np.bincount(r, minlength=g.n).max()) if r.size else 0


def test_small_build_bitwise_vs_general(cl, monkeypatch):
    n_small = 0
    for g in _graphs():
        a, fa, la = _build(cl, g, True, monkeypatch)
        b, fb, lb = _build(cl, g, False, monkeypatch)
        _same(a, b, g.name)
        assert fa == fb, f"{g.name}: facts {fa} vs {fb}"
        if _longest_row(g) <= 256:
            n_small += 1
            assert la < lb, f"{g.name}: one-kernel build launched {la} kernels, general {lb}"
        else:                                   # the one-kernel attempt + its readback, then the general build
            assert la == lb + 2, f"{g.name}: fallback launched {la} kernels, general {lb}"
    assert n_small >= 50


def test_small_build_matches_oracle(cl, monkeypatch):
    monkeypatch.setenv("CLEORA_SMALL_BUILD", "1")
    for g in _graphs()[::3] + [gen.config("c1")]:
        M = oracle.build_from(g)
        G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
        try:
            c = cl.cleora_fetch_csr(G)
        finally:
            G.close()
        assert np.array_equal(c["row_ptr"], M.row_ptr), g.name
        assert np.array_equal(c["col"], M.col), g.name
        assert np.array_equal(c["val"].view(np.uint32), M.val.view(np.uint32)), g.name
        assert np.array_equal(c["deg"].view(np.uint64), M.deg.view(np.uint64)), g.name


@pytest.mark.parametrize("length", [257, 3000])
@pytest.mark.parametrize("directed", [False, True])
def test_long_row_falls_back_to_the_general_build(cl, monkeypatch, length, directed):
    g = _row_graph(5000, length, directed, True, length + directed)
    a, fa, la = _build(cl, g, True, monkeypatch)
    b, fb, lb = _build(cl, g, False, monkeypatch)
    _same(a, b, g.name)
    assert fa == fb and _longest_row(g) == length
    assert la == lb + 2, f"fallback: the one-kernel attempt and its readback, then the general build ({la} vs {lb})"


def test_small_build_error_verdicts(cl, monkeypatch):
    src = np.array([0, 1, 2, 3, 4], np.int32)
    dst = np.array([1, 2, 3, 4, 0], np.int32)
    cases = []
    bad_id = dst.copy(); bad_id[3] = 5
    cases.append((src, bad_id, None))
    bad_neg = src.copy(); bad_neg[1] = -1
    cases.append((bad_neg, dst, None))
    w = np.ones(5, np.float32); w[2] = np.nan
    cases.append((src, dst, w))
    w0 = np.ones(5, np.float32); w0[4] = 0.0; w0[1] = -2.0
    cases.append((src, dst, w0))
    both = dst.copy(); both[2] = 9
    wb = np.ones(5, np.float32); wb[0] = np.inf
    cases.append((src, both, wb))
    for s, d, w in cases:
        msgs = []
        for small in (True, False):
            monkeypatch.setenv("CLEORA_SMALL_BUILD", "1" if small else "0")
            with pytest.raises(cl.CleoraError) as ei:
                cl.cleora_build(s, d, w, 5, False, device=0)
            assert ei.value.code == cl.EDATA
            msgs.append(str(ei.value))
        assert msgs[0] == msgs[1]


def test_small_build_then_iterate_equals_general(cl, monkeypatch):
    """The embedding computed from either build is the same bytes (same CSR, same schedule)."""
    for g in (gen.config("c1"), gen.tiny_graph(7, n_max=300, e_max=2000, weighted=True)):
        outs = []
        for small in (True, False):
            monkeypatch.setenv("CLEORA_SMALL_BUILD", "1" if small else "0")
            G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
            try:
                cl.cleora_init(G, 128, 3)
                cl.cleora_iterate(G, 4)
                outs.append(cl.cleora_fetch(G))
            finally:
                G.close()
        assert outs[0].tobytes() == outs[1].tobytes(), g.name


def test_small_batch_build_bitwise(cl, monkeypatch):
    graphs = [gen.tiny_graph(900 + i, n_max=200, e_max=1500) for i in range(30)]
    graphs = [gen.EdgeList(x.name, x.n, x.src, x.dst, None, False) for x in graphs]
    ep = np.zeros(len(graphs) + 1, np.int64)
    ep[1:] = np.cumsum([x.n_edges for x in graphs])
    src = np.concatenate([x.src for x in graphs])
    dst = np.concatenate([x.dst for x in graphs])
    nc = np.array([x.n for x in graphs], np.int32)
    res = []
    for small in (True, False):
        monkeypatch.setenv("CLEORA_SMALL_BUILD", "1" if small else "0")
        B = cl.cleora_build_batch(src, dst, None, ep, nc, False, device=0)
        try:
            res.append(cl.cleora_fetch_csr(B))
        finally:
            B.close()
    _same(res[0], res[1], "batch")
