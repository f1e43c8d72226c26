"""SURVEY §8(f) rows on the GPU, through the C ABI, against the oracle (f4 batches: test_gpu_batch.py):

f1 -- Algorithm 1 with Q chunks: every chunk handle's CSR bit-exact against the
      oracle's build of the same edge subset (reading R13), chunk embeddings within the bars, the
      merge bit-exact against the oracle's merge of the same chunk embeddings (reading R14), and
      the whole chunked pipeline within the bars of oracle.embed_chunked.  Q = 1 is bit-identical
      to the unchunked GPU path.
f2 -- inductive embedding of new nodes: cleora_reconstruct against
      oracle.reconstruct on the GPU's own T_{I-1}; the training-consistency identity
      reconstruct(every node from its own edges, T_{I-1}) == T_I, bitwise on the GPU.
f3 -- hypergraph clique / star expansion on the device: edge lists byte-identical to the oracle's
      (readings R16/R17), host and device paths, and expand -> build -> embed within the bars.
"""
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


def close(T, R, what):
    T = T.astype(np.float64)
    R = R.astype(np.float64)
    assert np.array_equal(~T.any(1), ~R.any(1)), f"{what}: zero rows differ"
    err = float(np.abs(T - R).max()) if T.size else 0.0
    assert err <= TOL_ABS, f"{what}: max|d| {err:.3e}"
    nz = R.any(1)
    if nz.any():
        cos = (T[nz] * R[nz]).sum(1) / (np.linalg.norm(T[nz], axis=1) * np.linalg.norm(R[nz], axis=1))
        assert cos.min() >= TOL_COS, f"{what}: min cos {cos.min():.9f}"


def _graphs():
    rng = np.random.default_rng(3)
    n = 4000
    hub = gen.EdgeList("hub", n, np.concatenate([np.zeros(3000, np.int32), rng.integers(0, n, 9000).astype(np.int32)]),
                       np.concatenate([np.arange(1, 3001, dtype=np.int32), rng.integers(0, n, 9000).astype(np.int32)]),
                       rng.lognormal(0, 1, 12000).astype(np.float32), False)
    return [gen.config("c1"), hub, gen.rmat_directed(4096, 12, 50000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=6)] + \
        [gen.tiny_graph(s) for s in range(12)]


@pytest.mark.parametrize("Q", [1, 2, 3, 5])
def test_chunked_pipeline(cl, Q):
    for gi, g in enumerate(_graphs()):
        d, iters, seed, cseed = [17, 64, 128, 256][(gi + Q) % 4], 1 + (gi + Q) % 4, 3, 100 + gi
        chunk = oracle.chunk_assign(g.n_edges, Q, cseed)
        hs = []
        try:
            for q in range(Q):
                G = cl.cleora_build(g.src, g.dst, g.w, g.n, g.directed, device=0, n_chunks=Q, chunk=q, chunk_seed=cseed)
                hs.append(G)
                m = chunk == q
                if m.any():          # the chunk's CSR: bit-exact against the oracle's build of the subset
                    M = oracle.build_csr(g.src[m], g.dst[m], None if g.w is None else g.w[m], g.n, g.directed)
                    csr = cl.cleora_fetch_csr(G)
                    assert np.array_equal(csr["row_ptr"], M.row_ptr) and np.array_equal(csr["col"], M.col)
                    assert np.array_equal(csr["val"].view(np.uint32), M.val.view(np.uint32))
                    assert np.array_equal(csr["deg"].view(np.uint64), M.deg.view(np.uint64))
                else:
                    assert cl.cleora_info(G)["nnz"] == 0
                cl.cleora_init(G, d, seed)
                cl.cleora_iterate(G, iters)
            parts = [cl.cleora_fetch(G) for G in hs]
            merged = cl.cleora_merge_chunks(hs)
        finally:
            for G in hs:
                G.close()
        T_ref, parts_ref, occ, _ = oracle.embed_chunked(g.src, g.dst, g.w, g.n, g.directed, Q, cseed, d, seed, iters,
                                                        return_parts=True)
        for q in range(Q):
            close(parts[q], parts_ref[q], f"{g.name} Q={Q} chunk {q}")
        # the merge itself: bit-exact with the oracle's merge of the GPU's own chunk embeddings
        assert merged.tobytes() == oracle.merge(parts, occ).tobytes(), f"{g.name} Q={Q}: merge not bit-exact"
        err = float(np.abs(merged.astype(np.float64) - T_ref).max())
        assert err <= TOL_ABS, f"{g.name} Q={Q}: merged max|d| {err:.3e}"
        assert (np.linalg.norm(merged.astype(np.float64), axis=1) <= 1 + 1e-6).all()


def test_q1_is_the_unchunked_path(cl):
    g = gen.config("c1")
    outs = []
    for kw in ({}, dict(n_chunks=1, chunk=0, chunk_seed=9)):
        G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0, **kw)
        cl.cleora_init(G, 64, 1)
        cl.cleora_iterate(G, 3)
        outs.append(cl.cleora_merge_chunks([G]) if kw else cl.cleora_fetch(G))
        G.close()
    assert outs[0].tobytes() == outs[1].tobytes()


def test_merge_errors(cl):
    g = gen.config("c1")
    G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
    cl.cleora_init(G, 8, 0)
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_merge_chunks([G])                   # built without n_chunks: no occurrences
    assert e.value.code == cl.EUSAGE
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_build(g.src, g.dst, None, g.n, False, device=0, n_chunks=2, chunk=2)
    assert e.value.code == cl.EUSAGE
    G.close()


# ---------------------------------------------------------------- f2

def test_reconstruct_reproduces_the_last_step_bitwise(cl):
    for g in (gen.config("c1"), gen.chung_lu(20000, 60000, 2.1, 9.5388, 233115.5 * 20000 / 1134890, seed=2)):
        G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
        try:
            cl.cleora_init(G, 128, 0)
            cl.cleora_iterate(G, 2)
            T2 = cl.cleora_fetch(G)
            R = cl.cleora_reconstruct(G, np.concatenate([g.src, g.dst]), np.concatenate([g.dst, g.src]), None, g.n)
            cl.cleora_iterate(G, 1)
            T3 = cl.cleora_fetch(G)
        finally:
            G.close()
        assert R.tobytes() == T3.tobytes(), g.name
        close(R, oracle.reconstruct(np.concatenate([g.src, g.dst]), np.concatenate([g.dst, g.src]), None, g.n, T2),
              f"{g.name} reconstruct vs oracle")


@pytest.mark.parametrize("d", [5, 128, 1024, 1100])
def test_reconstruct_new_nodes(cl, d):
    rng = np.random.default_rng(d)
    g = gen.chung_lu(8000, 24000, 2.1, 9.5388, 233115.5 * 8000 / 1134890, seed=4)
    n_new = 700
    # new nodes: random neighbour sets (one with 5000 neighbours: the heavy path), some without edges
    new = np.concatenate([rng.integers(0, n_new - 20, 6000), np.full(5000, n_new - 21)]).astype(np.int32)
    known = rng.integers(0, g.n, new.size).astype(np.int32)
    w = rng.lognormal(0, 1, new.size).astype(np.float32)
    G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0)
    try:
        cl.cleora_init(G, d, 2)
        cl.cleora_iterate(G, 3)
        Tsrc = cl.cleora_fetch(G)
        for ww in (None, w):
            R = cl.cleora_reconstruct(G, new, known, ww, n_new)
            close(R, oracle.reconstruct(new, known, ww, n_new, Tsrc), f"d={d} weighted={ww is not None}")
            assert not R[n_new - 20:].any()              # no edges: zero rows (reading RZ)
        # more new nodes than known nodes
        big = np.arange(g.n + 50, dtype=np.int32)
        R = cl.cleora_reconstruct(G, big, big % g.n, None, g.n + 50)
        close(R, oracle.reconstruct(big, big % g.n, None, g.n + 50, Tsrc), "n_new > N")
        with pytest.raises(cl.CleoraError) as e:
            cl.cleora_reconstruct(G, np.array([0], np.int32), np.array([g.n], np.int32), None, 1)
        assert e.value.code == cl.EDATA
        with pytest.raises(cl.CleoraError) as e:
            cl.cleora_reconstruct(G, np.array([5], np.int32), np.array([0], np.int32), None, 3)
        assert e.value.code == cl.EDATA
    finally:
        G.close()


# ---------------------------------------------------------------- f3

def _hyper(seed, n=3000, n_he=2000, kmax=40):
    rng = np.random.default_rng(seed)
    k = rng.integers(1, kmax + 1, n_he)
    k[::97] = 300                                                      # some wide hyperedges
    ptr = np.concatenate([[0], np.cumsum(k)]).astype(np.int64)
    nodes = rng.integers(0, n, ptr[-1]).astype(np.int32)
    return ptr, nodes, rng.lognormal(0, 1, n_he).astype(np.float32), n


def test_expansion_bit_exact_and_embedding(cl):
    import torch
    for seed in range(3):
        ptr, nodes, w, n = _hyper(seed)
        for mode, ref in ((cl.EXPAND_CLIQUE, oracle.expand_clique(ptr, nodes, w)),
                          (cl.EXPAND_STAR, oracle.expand_star(ptr, nodes, n, w))):
            got = cl.cleora_expand(ptr, nodes, n, mode, w)
            for a, b in zip(got, ref):
                assert a.tobytes() == b.tobytes(), f"seed {seed} mode {mode}"
            # device in -> device out, same bytes
            dgot = cl.cleora_expand(torch.from_numpy(ptr).cuda(), torch.from_numpy(nodes).cuda(), n, mode,
                                    torch.from_numpy(w).cuda())
            for a, b in zip(dgot, ref):
                assert a.cpu().numpy().tobytes() == b.tobytes()
            # end to end: expand -> build -> embed, against the oracle on the oracle's expansion
            nn = n if mode == cl.EXPAND_CLIQUE else n + len(ptr) - 1
            G = cl.cleora_build(dgot[0], dgot[1], dgot[2], nn, False)
            cl.cleora_init(G, 64, 1)
            cl.cleora_iterate(G, 3)
            T = cl.cleora_fetch(G)
            G.close()
            R = oracle.embed(oracle.build_csr(ref[0], ref[1], ref[2], nn, False), 64, 1, 3)
            close(T, R, f"expanded seed {seed} mode {mode}")


def test_expansion_errors(cl):
    ptr = np.array([0, 2], np.int64)
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_expand(ptr, np.array([0, 5], np.int32), 5, cl.EXPAND_CLIQUE)
    assert e.value.code == cl.EDATA and "member 1" in str(e.value)
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_expand(ptr, np.array([0, 1], np.int32), 5, cl.EXPAND_STAR, np.array([-1.0], np.float32))
    assert e.value.code == cl.EDATA


def test_merge_after_trim(cl):
    """Chunk handles trimmed to their results (cleora_trim keeps T_I and the occurrence counts) merge
    to the same bytes as untrimmed ones: the memory-lean way to embed Q chunks one after another."""
    g = gen.config("c1")
    Q, cseed = 3, 21
    outs = []
    for trim in (False, True):
        hs = []
        try:
            for q in range(Q):
                G = cl.cleora_build(g.src, g.dst, None, g.n, False, device=0, n_chunks=Q, chunk=q, chunk_seed=cseed)
                hs.append(G)
                cl.cleora_init(G, 96, 2)
                cl.cleora_iterate(G, 3 if q != 1 else 4)    # odd and even counts: either buffer is kept
                if trim:
                    cl.cleora_trim(G)
            outs.append(cl.cleora_merge_chunks(hs))
        finally:
            for G in hs:
                G.close()
    assert outs[0].tobytes() == outs[1].tobytes()
