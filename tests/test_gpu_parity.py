"""Parity of the CUDA path (through the C ABI) against the CPU oracle -- needs a B200.

Bars (BASELINE.json north_star): CSR structure, values and degrees bit-exact; T_0 bit-exact;
every iterate within max|d| <= 1e-5 per element and cosine >= 0.99999 per non-zero row; the
zero-row sets identical.  Inputs are the seeded generators of gen/ (DESIGN.md "Input recipe").
"""
import os

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

TOL_ABS = 1e-5
TOL_COS = 0.99999


@pytest.fixture(scope="module")
def cl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2102_02302_b200 as m
    return m


def check_csr(csr, M):
    assert np.array_equal(csr["row_ptr"], M.row_ptr), "row_ptr"
    assert np.array_equal(csr["col"], M.col), "col"
    assert np.array_equal(csr["val"].view(np.uint32), M.val.view(np.uint32)), "val bits"
    assert np.array_equal(csr["deg"].view(np.uint64), M.deg.view(np.uint64)), "deg bits"


def compare(T, R, what="", chunk=1 << 16):
    """max|d| and min cosine over non-zero rows; zero-row sets must be identical.
    Row-chunked so that full-size configs (c4: 2 x 19.9 GB) fit in host memory."""
    err, mc = 0.0, 1.0
    for r0 in range(0, T.shape[0], chunk):
        t = T[r0:r0 + chunk].astype(np.float64)
        r = R[r0:r0 + chunk].astype(np.float64)
        if t.size:
            err = max(err, float(np.abs(t - r).max()))
        zt, zr = ~t.any(1), ~r.any(1)
        assert np.array_equal(zt, zr), f"{what}: zero-row sets differ in rows [{r0}, {r0 + chunk})"
        nz = ~zr
        if nz.any():
            cos = (t[nz] * r[nz]).sum(1) / (np.linalg.norm(t[nz], axis=1) * np.linalg.norm(r[nz], axis=1))
            mc = min(mc, float(cos.min()))
    assert err <= TOL_ABS, f"{what}: max|d| = {err:.3e}"
    assert mc >= TOL_COS, f"{what}: min cos = {mc:.9f}"
    return err, mc


def ill_conditioned(M, T_prev):
    """True if some row's pre-normalisation vector is (near) zero although it has live
    neighbours: normalising it is ill-defined, so any rounding may flip it (d=1 graphs).
    Only evaluated on small cases (random-init graphs of real size never cancel)."""
    if M.nnz == 0 or M.nnz * T_prev.shape[1] > 5e7:
        return False
    rows = np.repeat(np.arange(M.n), np.diff(M.row_ptr))
    Y = np.zeros_like(T_prev, dtype=np.float64)
    np.add.at(Y, rows, M.val[:, None].astype(np.float64) * T_prev[M.col].astype(np.float64))
    live = np.zeros(M.n, bool)
    np.logical_or.at(live, rows, T_prev[M.col].any(1))
    nr = np.linalg.norm(Y, axis=1)
    return bool(live.any() and nr[live].min() < 1e-4)


def run_case(cl, g, d, iters, seed=0, per_iter=True, one_call=False):
    """one_call: the GPU runs cleora_iterate(iters) once -- the launch sequence bench.py times (with
    half-row passes every step but the last is lazy, reading R21) -- against the oracle's T_iters."""
    M = oracle.build_from(g)
    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
    try:
        check_csr(cl.cleora_fetch_csr(G), M)
        cl.cleora_init(G, d, seed)
        R = oracle.hash_init(g.n, d, seed)
        T = cl.cleora_fetch(G)
        assert np.array_equal(T.view(np.uint32), R.view(np.uint32)), "T_0 not bit-exact"
        worst = (0.0, 1.0)
        del T
        if one_call:
            cl.cleora_iterate(G, iters)
            for i in range(iters):
                R = oracle.step(M, R)
            return compare(cl.cleora_fetch(G), R, f"{g.name} d={d} iterate({iters})")
        for i in range(1, iters + 1):
            if ill_conditioned(M, R):
                break
            cl.cleora_iterate(G, 1)
            R = oracle.step(M, R)
            if per_iter or i == iters:
                e, c = compare(cl.cleora_fetch(G), R, f"{g.name} d={d} iteration {i}")
                worst = (max(worst[0], e), min(worst[1], c))
        return worst
    finally:
        G.close()


DIMS = [1, 2, 3, 4, 5, 7, 8, 16, 31, 33, 64, 100, 128, 129, 200, 256, 257, 384, 512, 513, 768, 1000, 1024,
        1025, 1500, 2048, 3000, 4096]


@pytest.mark.parametrize("seed", range(100))
def test_tiny_random_graphs(cl, seed):
    g = gen.tiny_graph(seed)
    d = DIMS[seed % len(DIMS)]
    run_case(cl, g, d, iters=1 + seed % 6, seed=seed)


@pytest.mark.parametrize("d", [1, 4, 17, 128, 256, 1024, 1100])
@pytest.mark.parametrize("directed,weighted", [(False, False), (True, True)])
def test_hub_rows_multi_part(cl, d, directed, weighted):
    """Power-law hubs: a star of 5000 leaves plus a random graph, so the hub row is split into
    several CTA items (heavy path with the last-CTA fp64 finalisation)."""
    rng = np.random.default_rng(d)
    n = 6000
    src = np.concatenate([np.zeros(5000, np.int32), rng.integers(0, n, 20000).astype(np.int32)])
    dst = np.concatenate([np.arange(1, 5001, dtype=np.int32), rng.integers(0, n, 20000).astype(np.int32)])
    w = rng.lognormal(0, 1, src.size).astype(np.float32) if weighted else None
    g = gen.EdgeList("hub", n, src, dst, w, directed)
    run_case(cl, g, d, iters=4)


@pytest.mark.parametrize("thresh", ["8", "16", "64", "4096"])
def test_schedule_threshold_does_not_change_results(cl, thresh, monkeypatch):
    monkeypatch.setenv("CLEORA_HEAVY_THRESH", thresh)
    g = gen.chung_lu(20000, 60000, 2.1, 9.5388, 233115.5 * 20000 / 1134890, seed=1)
    run_case(cl, g, 256, iters=4)


def _record(name, worst):
    """Worst max|d| / min cosine of a full-config case, printed and (CLEORA_PARITY_LOG=file) logged."""
    import json
    line = json.dumps({"config": name, "max_abs": worst[0], "min_cos": worst[1]})
    print(line)
    if os.environ.get("CLEORA_PARITY_LOG"):
        with open(os.environ["CLEORA_PARITY_LOG"], "a") as f:
            f.write(line + "\n")


def test_degree_of_long_weighted_rows_bit_exact(cl):
    """deg(a) is the sequential fp64 fold over ascending b (reading B3).  Rows of > 32 entries take a
    parallel sum when it provably equals that fold (every e_ab a multiple of 2^q and the total below
    2^(53+q): no partial sum in any order rounds), else the sequential fold.  Rows built to fall on
    either side -- dyadic weights, fp32 lognormal weights (c4's kind), weights spanning 1e-7..1e7 whose
    partial sums round, duplicates merged first -- must give the oracle's bits, through both builds."""
    rng = np.random.default_rng(61)
    n, m = 3000, 6000
    rows = []
    ws = [rng.integers(1, 4096, m).astype(np.float32) / np.float32(8.0),          # multiples of 1/8
          rng.lognormal(0.0, 1.0, m).astype(np.float32),                         # c4-like
          (10.0 ** rng.uniform(-7, 7, m)).astype(np.float32),                    # rounds: sequential fold
          np.float32(2.0 ** 100) * rng.integers(1, 9, m).astype(np.float32),     # large dyadic
          rng.lognormal(0.0, 1.0, m).astype(np.float32)]
    src = np.concatenate([np.full(m, r, np.int32) for r in range(len(ws))])
    dst = np.concatenate([rng.integers(0, n, m).astype(np.int32) for _ in ws])
    dst[-m:] = rng.integers(0, 40, m).astype(np.int32)                           # many duplicates per run
    g = gen.EdgeList("longw", n, src, dst, np.concatenate(ws), True)
    M = oracle.build_from(g)
    import os
    for small in ("1", "0"):
        os.environ["CLEORA_SMALL_BUILD"] = small
        try:
            G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
            check_csr(cl.cleora_fetch_csr(G), M)
            G.close()
        finally:
            os.environ.pop("CLEORA_SMALL_BUILD", None)


def test_c1_full(cl):
    g = gen.config("c1")
    _record("c1", run_case(cl, g, g.d, g.iters))


def test_c3_full(cl):
    g = gen.config("c3")
    _record("c3", run_case(cl, g, g.d, g.iters, per_iter=False))


def test_c2_full(cl):
    g = gen.config("c2")
    _record("c2", run_case(cl, g, g.d, g.iters, per_iter=False))


def test_c4_full(cl):
    """c4 as bench.py runs it: iterate(4) in one call (half-row passes, lazy normalisation in steps 1-3)"""
    g = gen.config("c4")
    _record("c4", run_case(cl, g, g.d, g.iters, one_call=True))


def test_determinism_and_composability(cl):
    """Same bytes on repeated runs; iterate(1)+iterate(2) == iterate(3) bit for bit."""
    g = gen.config("c1")
    outs = []
    for split in ([3], [1, 2], [3]):
        G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
        cl.cleora_init(G, 64, 5)
        for k in split:
            cl.cleora_iterate(G, k)
        outs.append(cl.cleora_fetch(G).tobytes())
        G.close()
    assert outs[0] == outs[1] == outs[2]


def test_device_resident_inputs_and_stream(cl):
    """The same result when the COO is already in HBM (torch CUDA tensors) and a caller stream is used."""
    import torch
    g = gen.config("c1")
    s = torch.cuda.Stream()
    G1 = cl.cleora_build(g.src, g.dst, g.w, g.n, False, device=0)
    G2 = cl.cleora_build(torch.from_numpy(g.src).cuda(), torch.from_numpy(g.dst).cuda(), None, g.n, False,
                         stream=s)
    for G in (G1, G2):
        cl.cleora_init(G, 128, 0)
        cl.cleora_iterate(G, 2)
    a, b = cl.cleora_fetch(G1), cl.cleora_fetch(G2)
    out = torch.empty_like(torch.from_numpy(a)).cuda()
    cl.cleora_fetch(G2, 0, g.n, out)
    assert a.tobytes() == b.tobytes() == out.cpu().numpy().tobytes()
    G1.close(); G2.close()


def test_set_rows_and_partial_fetch(cl):
    g = gen.config("c1")
    M = oracle.build_from(g)
    G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
    cl.cleora_init(G, 20, 1)
    T0 = np.random.default_rng(0).standard_normal((g.n, 20)).astype(np.float32)
    cl.cleora_set_rows(G, 0, T0)
    np.testing.assert_array_equal(cl.cleora_fetch(G, 100, 300), T0[100:300])
    cl.cleora_iterate(G, 1)
    compare(cl.cleora_fetch(G), oracle.step(M, T0), "custom T0")
    assert cl.cleora_fetch(G, 5, 5).shape == (0, 20)
    G.close()


def test_error_codes(cl):
    i32 = lambda *a: np.array(a, np.int32)
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_build(i32(0, 1), i32(1, 5), None, 3)
    assert e.value.code == cl.EDATA and "edge 1" in str(e.value)
    for bad in (0.0, -2.0, np.nan, np.inf):
        with pytest.raises(cl.CleoraError) as e:
            cl.cleora_build(i32(0, 1), i32(1, 2), np.array([1.0, bad], np.float32), 3)
        assert e.value.code == cl.EDATA
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_build(i32(), i32(), None, 3)
    assert e.value.code == cl.EUSAGE
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_build(i32(0), i32(1), None, 0)
    assert e.value.code == cl.EUSAGE
    G = cl.cleora_build(i32(0), i32(1), None, 2, device=0)
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_iterate(G, 1)                      # before init
    assert e.value.code == cl.EUSAGE
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_init(G, 0, 0)
    assert e.value.code == cl.EUSAGE
    cl.cleora_init(G, 8, 0)
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_iterate(G, -1)
    assert e.value.code == cl.EUSAGE
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_fetch(G, 0, 3)
    assert e.value.code == cl.EUSAGE
    cl.cleora_iterate(G, 0)
    assert cl.cleora_info(G)["iterations"] == 0
    G.close()


def test_info_and_stats(cl):
    g = gen.config("c2")
    G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0, timing=True)
    info = cl.cleora_info(G)
    assert info["n_nodes"] == g.n and info["nnz"] == 2 * g.n_edges
    deg = np.bincount(np.concatenate([g.src, g.dst]), minlength=g.n)
    assert info["zero_rows"] == int((deg == 0).sum()) and info["max_degree"] == int(deg.max())
    cl.cleora_init(G, 128, 0)
    assert cl.cleora_info(G)["heavy_rows"] == int((deg > 256).sum())    # LDG / cp.async gathers: > 256 entries
    cl.cleora_init(G, 1024, 0)
    assert cl.cleora_info(G)["heavy_rows"] == int((deg > 64).sum())     # TMA bulk gathers: > 64 entries
    cl.cleora_iterate(G, 3)
    st = cl.cleora_stats(G, reset=True)
    assert st["spmm_launches"] == 3 and st["spmm_ms_total"] > 0
    assert cl.cleora_stats(G)["spmm_launches"] == 0
    G.close()


@pytest.mark.parametrize("d", [100, 256, 600, 1024])
def test_gather_engines_bitwise_equal(cl, d, monkeypatch):
    """The three gather engines -- TMA bulk copies, per-lane cp.async into the same shared-memory
    ring (spmm_tma.cu), and register LDGs (spmm_norm.cu) -- run the same per-row arithmetic in the
    same order, so their outputs are bitwise identical."""
    g = gen.chung_lu(30000, 90000, 2.1, 9.5388, 233115.5 * 30000 / 1134890, seed=3)
    monkeypatch.setenv("CLEORA_HEAVY_THRESH", "64")       # the same schedule for every engine
    outs = []
    for mode in ("bulk", "async", "ldg"):
        monkeypatch.setenv("CLEORA_GATHER", mode)
        G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
        cl.cleora_init(G, d, 0)
        cl.cleora_iterate(G, 3)
        outs.append(cl.cleora_fetch(G))
        G.close()
    assert outs[0].tobytes() == outs[1].tobytes() == outs[2].tobytes()


def test_fetch_async_overlaps_and_is_ordered(cl):
    """cleora_fetch_async copies the current T while later work runs; later iterations of the same
    handle are ordered after the copy (the copied rows are T_2, not a mix with T_3 / T_4)."""
    import torch
    g = gen.config("c1")
    G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
    cl.cleora_init(G, 128, 0)
    cl.cleora_iterate(G, 2)
    ref2 = cl.cleora_fetch(G)
    out = torch.empty((g.n, 128), dtype=torch.float32).pin_memory()
    cl.cleora_fetch_async(G, 0, g.n, out)
    cl.cleora_iterate(G, 2)                           # overwrites both buffers after the copy
    cl.cleora_sync(G)
    assert out.numpy().tobytes() == ref2.tobytes()
    ref4 = cl.cleora_fetch(G)
    G2 = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
    cl.cleora_init(G2, 128, 0)
    cl.cleora_iterate(G2, 4)
    assert cl.cleora_fetch(G2).tobytes() == ref4.tobytes()
    part = torch.empty((100, 128), dtype=torch.float32, device="cuda")
    cl.cleora_fetch_async(G2, 50, 150, part)          # device destination, row range
    G2.close()                                        # destroy waits for the copy
    assert part.cpu().numpy().tobytes() == ref4[50:150].tobytes()
    G.close()


def _degenerate_graphs():
    rng = np.random.default_rng(11)
    out = []
    n = 50                                                # every edge a self-loop
    out.append(gen.EdgeList("self_loops", n, np.arange(n, dtype=np.int32), np.arange(n, dtype=np.int32), None, False))
    # one edge listed 10,000 times with weights: a single merged entry per direction (reading B2)
    out.append(gen.EdgeList("dup10k", 3, np.zeros(10000, np.int32), np.ones(10000, np.int32),
                            rng.lognormal(0, 2, 10000).astype(np.float32), False))
    # in-star: 100,000 leaves point at node 0 (directed): node 0's column is gathered by every leaf,
    # node 0's own row is empty (a sink); plus the out-star from node 1 (a 100,000-entry heavy row)
    leaves = np.arange(2, 100002, dtype=np.int32)
    out.append(gen.EdgeList("stars", 100002, np.concatenate([leaves, np.ones(100000, np.int32)]),
                            np.concatenate([np.zeros(100000, np.int32), leaves]), None, True))
    out.append(gen.EdgeList("chain", 5000, np.arange(4999, dtype=np.int32), np.arange(1, 5000, dtype=np.int32),
                            None, False))
    out.append(gen.EdgeList("one_node", 1, np.zeros(1, np.int32), np.zeros(1, np.int32), None, True))
    a, b = np.meshgrid(np.arange(50), np.arange(50, 100))
    out.append(gen.EdgeList("K50_50", 100, a.ravel().astype(np.int32), b.ravel().astype(np.int32), None, False))
    return out


@pytest.mark.parametrize("d", [1, 7, 128, 1024])
def test_degenerate_graphs(cl, d):
    for g in _degenerate_graphs():
        run_case(cl, g, d, iters=4)


def test_c2_repeatable_bitwise(cl):
    """Two runs of the bench workload give the same bytes (no floating-point atomics anywhere; heavy
    rows are combined in part order whichever CTA finishes last)."""
    g = gen.config("c2")
    outs = []
    for _ in range(2):
        G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
        cl.cleora_init(G, g.d, 0)
        cl.cleora_iterate(G, g.iters)
        outs.append(cl.cleora_fetch(G))
        G.close()
    assert outs[0].tobytes() == outs[1].tobytes()


def test_cached_memory_release_and_reuse(cl):
    """Blocks freed by destroy are reused by the next handle of the same shape; releasing the cache
    returns them to the driver and everything still works afterwards."""
    import torch
    g = gen.config("c1")
    ref = None
    for release in (False, True, False):
        G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
        cl.cleora_init(G, 256, 0)
        cl.cleora_iterate(G, 2)
        T = cl.cleora_fetch(G)
        G.close()
        ref = T if ref is None else ref
        assert T.tobytes() == ref.tobytes()
        if release:
            free_before = torch.cuda.mem_get_info()[0]
            cl.cleora_release_cached_memory()
            assert torch.cuda.mem_get_info()[0] >= free_before


@pytest.mark.parametrize("mode,d", [("bulk", 1024), ("async", 512), ("ldg", 256), ("ldg", 100)])
def test_light_chunk_rows_do_not_change_bytes(cl, mode, d, monkeypatch):
    """Light rows are computed one at a time in entry order whatever the light-chunk length, so the
    per-engine chunk-row caps (6 / 8 / 31) change only the processing order of rows, never
    a value: 1-, 6- and 31-row chunks give bitwise the same T.  Graphs large enough (300k+ rows)
    that the caps bind, a lattice (the row-order locality case) and a power law (heavy rows)."""
    import torch
    monkeypatch.setenv("CLEORA_GATHER", mode)
    graphs = [gen.lattice(560, 0.3, 0.02, seed=5),
              gen.chung_lu(320000, 900000, 2.1, 9.5388, 233115.5 * 320000 / 1134890, seed=6)]
    for g in graphs:
        outs = []
        for rows in ("1", "6", "31"):
            monkeypatch.setenv("CLEORA_CHUNK_ROWS", rows)
            G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
            cl.cleora_init(G, d, 0)
            cl.cleora_iterate(G, 2)
            outs.append(cl.cleora_fetch(G, out=torch.empty((g.n, d), dtype=torch.float32, device="cuda")))
            G.close()
        assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2]), f"{g.name} {mode} d={d}"


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("heavy", ["64", "8"])
def test_short_row_pairs_bitwise_vs_tma_engines(cl, d, heavy, monkeypatch):
    """At d <= 128 the register kernel runs two short rows per warp (one per half-warp); its result
    must be bitwise the cp.async / TMA-bulk kernels' (one row per warp, different code).  Graphs mix
    odd chunk tails, short rows next to long and heavy ones, and rows without out-edges (directed
    R-MAT: the zero-row skip from iteration 2 on); heavy threshold 8 makes rows of 9-16 entries
    heavy items, so pairs and heavy rows interleave."""
    monkeypatch.setenv("CLEORA_HEAVY_THRESH", heavy)
    rng = np.random.default_rng(11)
    n = 5000
    hub = gen.EdgeList("hub", n, np.concatenate([np.zeros(3000, np.int32), rng.integers(0, n, 15000).astype(np.int32)]),
                       np.concatenate([np.arange(1, 3001, dtype=np.int32), rng.integers(0, n, 15000).astype(np.int32)]),
                       None, False)
    graphs = [hub, gen.rmat_directed(8192, 13, 50000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=12),
              gen.lattice(90, 0.3, 0.02, seed=13), gen.er(3001, 9000, seed=14)]
    for g in graphs:
        outs = []
        for mode in ("ldg", "async", "bulk"):
            monkeypatch.setenv("CLEORA_GATHER", mode)
            G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
            cl.cleora_init(G, d, 5)
            cl.cleora_iterate(G, 3)
            outs.append(cl.cleora_fetch(G))
            G.close()
        assert outs[0].tobytes() == outs[1].tobytes() == outs[2].tobytes(), f"{g.name} d={d} heavy={heavy}"


def test_trim_keeps_the_embedding_and_frees_the_rest(cl):
    """cleora_trim keeps only T_I: an asynchronous fetch enqueued before it completes with the same
    bytes, a blocking fetch after it too, device_bytes drops to one T buffer, and every call that
    needs the CSR or the other buffer is a usage error.  Odd and even iteration counts (the kept
    buffer is T[1] or T[0])."""
    import torch
    g = gen.config("c1")
    for iters in (3, 4):
        G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
        cl.cleora_init(G, 128, 0)
        cl.cleora_iterate(G, iters)
        ref = cl.cleora_fetch(G)
        out = torch.empty((g.n, 128), dtype=torch.float32).pin_memory()
        cl.cleora_fetch_async(G, 0, g.n, out)
        before = cl.cleora_info(G)["device_bytes"]
        cl.cleora_trim(G)
        cl.cleora_trim(G)                                   # no-op
        after = cl.cleora_info(G)["device_bytes"]
        assert after == g.n * 128 * 4 < before
        cl.cleora_sync(G)
        assert out.numpy().tobytes() == ref.tobytes()
        assert cl.cleora_fetch(G).tobytes() == ref.tobytes()
        for call in (lambda: cl.cleora_iterate(G, 1), lambda: cl.cleora_init(G, 128, 0),
                     lambda: cl.cleora_fetch_csr(G), lambda: cl.cleora_set_rows(G, 0, ref[:4])):
            with pytest.raises(cl.CleoraError) as e:
                call()
            assert e.value.code == 2
        G.close()


@pytest.mark.parametrize("heavy", ["64", "8"])
def test_half_row_passes_bitwise(cl, heavy, monkeypatch):
    """dp = 1024 steps as two half-row passes (CLEORA_HALVES=1; the default where nnz >= 8 N, e.g. c4)
    give bitwise the whole-row kernel's result (CLEORA_HALVES=0): light rows, single- and multi-part
    heavy rows (threshold 8 makes most rows heavy), rows without out-edges (the zero-row skip from
    step 3 on), weights, split iterate calls, and the loopback exchange (peer stores in pass 2)."""
    monkeypatch.setenv("CLEORA_HEAVY_THRESH", heavy)
    monkeypatch.setenv("CLEORA_LAZY", "0")          # bitwise: every step normalised (lazy steps: below)
    rng = np.random.default_rng(21)
    n = 6000
    hub = gen.EdgeList("hub", n, np.concatenate([np.zeros(5000, np.int32), rng.integers(0, n, 20000).astype(np.int32)]),
                       np.concatenate([np.arange(1, 5001, dtype=np.int32), rng.integers(0, n, 20000).astype(np.int32)]),
                       rng.lognormal(0, 1, 25000).astype(np.float32), True)
    graphs = [hub, gen.rmat_directed(8192, 13, 120000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=22), gen.config("c1")]
    for g in graphs:
        outs = {}
        for halves in ("0", "1"):
            monkeypatch.setenv("CLEORA_HALVES", halves)
            for mode in ("bulk", "async"):
                monkeypatch.setenv("CLEORA_GATHER", mode)
                for lb in (False, True):
                    kw = dict(loopback=True, world=3, rank=1) if lb else {}
                    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0, **kw)
                    cl.cleora_init(G, 1024, 3)
                    cl.cleora_iterate(G, 2)
                    cl.cleora_iterate(G, 2)
                    outs[(halves, mode, lb)] = [cl.cleora_fetch_replica(G, p).tobytes() for p in range(3)] if lb else \
                        [cl.cleora_fetch(G).tobytes()]
                    G.close()
        ref = outs[("0", "bulk", False)][0]
        for key, reps in outs.items():
            for b in reps:
                assert b == ref, f"{g.name} heavy={heavy}: {key} differs from the whole-row kernel"
    M = oracle.build_from(graphs[1])
    monkeypatch.setenv("CLEORA_HALVES", "1")
    monkeypatch.delenv("CLEORA_GATHER")
    G = cl.cleora_build(graphs[1].src, graphs[1].dst, graphs[1].w, graphs[1].n, True, device=0)
    cl.cleora_init(G, 1024, 3)
    cl.cleora_iterate(G, 4)
    compare(cl.cleora_fetch(G), oracle.embed(M, 1024, 3, 4), "halves vs oracle")
    G.close()


@pytest.mark.parametrize("heavy", ["256", "8"])
def test_lazy_normalisation_between_steps(cl, heavy, monkeypatch):
    """Half-row steps inside one iterate call leave their rows unnormalised with the row scales aside
    and the next step folds the scales into its weights; only the call's last step normalises (reading
    R21).  Against the oracle's T_k within the bars, against every-step-normalised (CLEORA_LAZY=0)
    within rounding, bitwise reproducible, and split calls (each call's last step normalises) agree:
    light rows, single- and multi-part heavy rows (threshold 8), rows without out-edges, weights, both
    gather engines."""
    monkeypatch.setenv("CLEORA_HEAVY_THRESH", heavy)
    monkeypatch.setenv("CLEORA_HALVES", "1")
    rng = np.random.default_rng(31)
    n = 6000
    hub = gen.EdgeList("hub", n, np.concatenate([np.zeros(5000, np.int32), rng.integers(0, n, 20000).astype(np.int32)]),
                       np.concatenate([np.arange(1, 5001, dtype=np.int32), rng.integers(0, n, 20000).astype(np.int32)]),
                       rng.lognormal(0, 1, 25000).astype(np.float32), True)
    graphs = [hub, gen.rmat_directed(8192, 13, 120000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=32), gen.config("c1")]
    for g in graphs:
        M = oracle.build_from(g)
        R_all = oracle.embed(M, 1024, 3, 4, keep_all=True)
        R4 = R_all[4]
        for mode in ("async", "bulk"):
            monkeypatch.setenv("CLEORA_GATHER", mode)
            outs = {}
            for lazy, split in (("1", (4,)), ("1", (4,)), ("0", (4,)), ("1", (1, 3)), ("1", (2, 2))):
                monkeypatch.setenv("CLEORA_LAZY", lazy)
                G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
                try:
                    cl.cleora_init(G, 1024, 3)
                    done = 0
                    for k in split:
                        cl.cleora_iterate(G, k)
                        done += k
                        T = cl.cleora_fetch(G)          # between calls T is T_done: normalised rows, and the
                        nz = T.any(1)                   # rows without entries 0 (inner steps skip the ungathered)
                        assert np.allclose(np.linalg.norm(T[nz].astype(np.float64), axis=1), 1.0, atol=1e-6)
                        compare(T, R_all[done], f"{g.name} {mode} after {done} steps ({split})")
                    key = (lazy, split)
                    if key in outs:
                        assert outs[key].tobytes() == T.tobytes(), f"{g.name}: lazy run not reproducible"
                    outs[key] = T
                finally:
                    G.close()
            for key, T in outs.items():
                compare(T, R4, f"{g.name} {mode} heavy={heavy} lazy={key}")
            compare(outs[("1", (4,))], outs[("0", (4,))], f"{g.name} {mode}: lazy vs every step normalised")



@pytest.mark.parametrize("heavy", ["256", "8"])
def test_lazy_steps_skip_never_gathered_rows(cl, heavy, monkeypatch):
    """A lazy step stores nothing for a row with entries that no row gathers (in-degree 0): no later
    step of the call reads it and the call's last step computes it anew.  Forced on small graphs
    (CLEORA_HOT_MB tiny makes the in-degree available); the result of every call split is bitwise the
    one with those rows stored (CLEORA_KEEP_UNGATHERED=1) and within the bars of the oracle: light,
    single- and multi-part heavy source-only rows (threshold 8), both gather engines."""
    monkeypatch.setenv("CLEORA_HOT_MB", "0.001")
    monkeypatch.setenv("CLEORA_HALVES", "1")
    monkeypatch.setenv("CLEORA_HEAVY_THRESH", heavy)
    rng = np.random.default_rng(41)
    n = 6000
    # node n - 1: a source-only hub (3,000 out-edges, nothing points at it) -- a heavy never-gathered row
    src = np.concatenate([np.full(3000, n - 1, np.int32), rng.integers(0, n - 1, 20000).astype(np.int32)])
    dst = np.concatenate([rng.integers(0, n - 1, 3000).astype(np.int32), rng.integers(0, n - 1, 20000).astype(np.int32)])
    hub = gen.EdgeList("srchub", n, src, dst, rng.lognormal(0, 1, src.size).astype(np.float32), True)
    graphs = [hub, gen.rmat_directed(8192, 13, 60000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=42)]
    for g in graphs:
        M = oracle.build_from(g)
        ind = np.bincount(M.col, minlength=g.n)
        assert ((np.diff(M.row_ptr) > 0) & (ind == 0)).any(), "no never-gathered row with entries"
        R_all = oracle.embed(M, 1024, 5, 4, keep_all=True)
        for mode in ("async", "bulk"):
            monkeypatch.setenv("CLEORA_GATHER", mode)
            for split in ((4,), (2, 2), (3, 1)):
                outs = []
                for keep in ("0", "1"):
                    monkeypatch.setenv("CLEORA_KEEP_UNGATHERED", keep)
                    G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0)
                    try:
                        cl.cleora_init(G, 1024, 5)
                        for k in split:
                            cl.cleora_iterate(G, k)
                        outs.append(cl.cleora_fetch(G))
                    finally:
                        G.close()
                assert outs[0].tobytes() == outs[1].tobytes(), f"{g.name} {mode} {split}: differs from keeping them"
                compare(outs[0], R_all[4], f"{g.name} {mode} heavy={heavy} {split}")

def test_partial_t0_is_completed_on_every_read(cl, monkeypatch):
    """On graphs whose T exceeds the hot-row budget, cleora_init writes T_0 only for rows a step can
    gather (in-degree > 0) and fills in the others when T_0 itself is read.  Forced here on small
    graphs (CLEORA_HOT_MB tiny): every read before the first step -- fetch, partial fetch, async fetch,
    set_rows, trim, reconstruct, merge of chunks, loopback replicas, batches -- sees the full T_0 (bit-
    exact vs the oracle), and every embedding is bitwise the one from a fully written T_0
    (CLEORA_T0_ALL=1)."""
    import torch
    monkeypatch.setenv("CLEORA_HOT_MB", "0.001")
    rng = np.random.default_rng(71)
    graphs = [gen.rmat_directed(8192, 13, 50000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=72),   # many rows unreferenced
              gen.chung_lu(20000, 60000, 2.1, 9.5388, 233115.5 * 20000 / 1134890, seed=73),  # isolated nodes
              gen.tiny_graph(74, n_max=400, e_max=600, directed=True, weighted=True)]
    d, seed = 96, 3

    def mk(g, **kw):
        G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0, **kw)
        cl.cleora_init(G, d, seed)
        return G

    for g in graphs:
        R0 = oracle.hash_init(g.n, d, seed)
        G = mk(g)
        assert cl.cleora_fetch(G).tobytes() == R0.tobytes(), g.name
        G.close()
        G = mk(g)
        a, b = g.n // 3, min(g.n, g.n // 3 + 777)
        assert cl.cleora_fetch(G, a, b).tobytes() == R0[a:b].tobytes()
        G.close()
        G = mk(g)
        buf = torch.empty((g.n, d), dtype=torch.float32).pin_memory()
        cl.cleora_fetch_async(G, 0, g.n, buf)
        cl.cleora_sync(G)
        assert buf.numpy().tobytes() == R0.tobytes()
        G.close()
        G = mk(g)
        X = rng.standard_normal((5, d)).astype(np.float32)
        cl.cleora_set_rows(G, 10, X)
        R = R0.copy()
        R[10:15] = X
        assert cl.cleora_fetch(G).tobytes() == R.tobytes()
        G.close()
        G = mk(g)
        cl.cleora_trim(G)
        assert cl.cleora_fetch(G).tobytes() == R0.tobytes()
        G.close()
        new = np.arange(3, dtype=np.int32).repeat(4)
        known = rng.integers(0, g.n, new.size).astype(np.int32)
        outs = {}
        for full in ("0", "1"):
            monkeypatch.setenv("CLEORA_T0_ALL", full)
            G = mk(g)
            rec = cl.cleora_reconstruct(G, new, known, None, 3)
            G.close()
            G = mk(g)
            cl.cleora_iterate(G, 3)
            T3 = cl.cleora_fetch(G)
            G.close()
            G = mk(g)
            cl.cleora_iterate(G, 1)
            cl.cleora_iterate(G, 2)
            T12 = cl.cleora_fetch(G)
            G.close()
            G = mk(g, loopback=True, world=3, rank=1)
            reps0 = [cl.cleora_fetch_replica(G, p) for p in range(3)]
            G.close()
            G = mk(g, loopback=True, world=3, rank=2)
            cl.cleora_iterate(G, 2)
            reps2 = [cl.cleora_fetch_replica(G, p) for p in range(3)]
            G.close()
            hs = [mk(g, n_chunks=2, chunk=q, chunk_seed=5) for q in range(2)]
            merged = cl.cleora_merge_chunks(hs)
            for h in hs:
                h.close()
            outs[full] = (rec, T3, T12, reps0, reps2, merged)
        monkeypatch.delenv("CLEORA_T0_ALL")
        p, f = outs["0"], outs["1"]
        assert p[0].tobytes() == f[0].tobytes(), f"{g.name}: reconstruct on T_0"
        assert p[1].tobytes() == f[1].tobytes() and p[2].tobytes() == f[2].tobytes(), f"{g.name}: iterate"
        for x, y in zip(p[3], f[3]):
            assert x.tobytes() == y.tobytes() == R0.tobytes(), f"{g.name}: loopback T_0 replicas"
        for x, y in zip(p[4], f[4]):
            assert x.tobytes() == y.tobytes(), f"{g.name}: loopback iterate"
        assert p[5].tobytes() == f[5].tobytes(), f"{g.name}: merge of T_0 chunks"
    # a batch: T_0 keyed on local ids, rows left out by init filled in on the read
    bg = [gen.tiny_graph(800 + i, n_max=300, e_max=400, directed=True) for i in range(10)]
    ep = np.zeros(len(bg) + 1, np.int64)
    ep[1:] = np.cumsum([x.n_edges for x in bg])
    B = cl.cleora_build_batch(np.concatenate([x.src for x in bg]), np.concatenate([x.dst for x in bg]), None, ep,
                              np.array([x.n for x in bg], np.int32), True, device=0)
    cl.cleora_init(B, d, seed)
    T0 = cl.cleora_fetch(B)
    B.close()
    base = 0
    for x in bg:
        assert T0[base:base + x.n].tobytes() == oracle.hash_init(x.n, d, seed).tobytes()
        base += x.n
