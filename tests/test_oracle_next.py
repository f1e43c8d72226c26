"""Pins of the oracle's SURVEY §8(f) rows (CPU only):

f1 -- Algorithm 1 with Q > 1 chunks: edge split (reading R13), per-chunk
      embedding, merge T_v = sum_q w_qv T^q_v with w_qv from endpoint occurrences (reading R14).
f2 -- inductive embedding of new nodes: normalised weighted
      average of the neighbours' rows of T_{I-1}.

Pinned against things other than the oracle itself: dense numpy brute force (per-chunk D^-1 A
and row normalisation), closed forms (Q = 1 identity, single-chunk nodes, SPEC.md's 2/3-1/3
example, leaf nodes, orthogonal neighbours), invariants (weights sum to 1, convexity of the
merge, the training-consistency identity reconstruct(v, T_{I-1}) = T_I[v]).
"""
import numpy as np
import pytest

import gen
import oracle


def dense_embed(src, dst, w, n, directed, d, seed, iters):
    """Brute force: dense D^-1 A in fp64, fp32 storage of every iterate (as the oracle)."""
    A = np.zeros((n, n))
    ww = np.ones(len(src)) if w is None else np.asarray(w, np.float64)
    for u, v, x in zip(src, dst, ww):
        A[u, v] += x
        if not directed and u != v:
            A[v, u] += x
    deg = A.sum(1)
    M = np.divide(A, deg[:, None], out=np.zeros_like(A), where=deg[:, None] > 0).astype(np.float32).astype(np.float64)
    T = oracle.hash_init(n, d, seed).astype(np.float64)
    for _ in range(iters):
        Y = M @ T
        nr = np.linalg.norm(Y, axis=1, keepdims=True)
        T = np.divide(Y, nr, out=np.zeros_like(Y), where=nr > 0).astype(np.float32).astype(np.float64)
    return T


# ---------------------------------------------------------------- f1: chunk assignment

def test_chunk_assignment_partitions_deterministically_and_uniformly():
    for Q in (1, 2, 3, 7, 16):
        c = oracle.chunk_assign(200_000, Q, 11)
        assert c.min() >= 0 and c.max() < Q                  # every edge in exactly one chunk
        assert np.array_equal(c, oracle.chunk_assign(200_000, Q, 11))
        cnt = np.bincount(c, minlength=Q)
        exp = 200_000 / Q
        chi2 = float(((cnt - exp) ** 2 / exp).sum())
        assert chi2 < Q + 6 * np.sqrt(2 * Q) + 10, (Q, cnt)  # uniform (loose chi^2 bound)
    assert not np.array_equal(oracle.chunk_assign(10_000, 4, 1), oracle.chunk_assign(10_000, 4, 2))
    assert (oracle.chunk_assign(1000, 1, 5) == 0).all()       # SPEC.md:305 Q=1: a single chunk
    # prefix-stable: the chunk of edge i does not depend on how many edges follow
    assert np.array_equal(oracle.chunk_assign(5000, 5, 3)[:1000], oracle.chunk_assign(1000, 5, 3))


def test_occurrences_are_endpoint_counts():
    src = np.array([0, 1, 2, 0, 3], np.int32)
    dst = np.array([1, 2, 0, 3, 3], np.int32)                # (3,3) a self-loop: two occurrences
    chunk = np.array([0, 0, 1, 1, 1], np.int32)
    occ = oracle.chunk_occurrences(src, dst, chunk, 2, 5)
    assert occ.tolist() == [[1, 2, 1, 0, 0], [2, 0, 1, 3, 0]]
    assert occ.sum() == 2 * src.size


# ---------------------------------------------------------------- f1: merge

def test_merge_worked_example_and_single_chunk_nodes():
    rng = np.random.default_rng(0)
    d = 6
    T1, T2, T3 = (rng.standard_normal((3, d)).astype(np.float32) for _ in range(3))
    occ = np.array([[2, 0, 0], [1, 0, 1], [0, 5, 0]], np.int64)   # node 0: chunks 1,2 (2:1)
    out = oracle.merge([T1, T2, T3], occ)
    # SPEC.md:318-319 [DERIVED]: (2/3) r1 + (1/3) r2
    np.testing.assert_allclose(out[0], (2 / 3) * T1[0].astype(np.float64) + (1 / 3) * T2[0], rtol=0, atol=1e-7)
    assert np.array_equal(out[1], T3[1])                    # only in chunk 3: weight 1.0, bit-exact
    assert np.array_equal(out[2], T2[2])                    # only in chunk 2
    # a node in no chunk merges to zeros
    assert not oracle.merge([T1, T2], np.zeros((2, 3), np.int64)).any()


def test_merge_is_convex():
    rng = np.random.default_rng(1)
    n, d, Q = 300, 16, 4
    Tq = []
    for _ in range(Q):
        t = rng.standard_normal((n, d))
        Tq.append((t / np.linalg.norm(t, axis=1, keepdims=True)).astype(np.float32))
    occ = rng.integers(0, 4, (Q, n)).astype(np.int64)
    out = oracle.merge(Tq, occ).astype(np.float64)
    tot = occ.sum(0)
    w = np.divide(occ, tot, out=np.zeros(occ.shape), where=tot > 0)
    assert np.allclose(w[:, tot > 0].sum(0), 1.0, atol=1e-12)
    ref = sum(w[q][:, None] * Tq[q].astype(np.float64) for q in range(Q))
    np.testing.assert_allclose(out, ref, rtol=0, atol=2e-7)
    assert (np.linalg.norm(out, axis=1) <= 1 + 1e-6).all()
    same = oracle.merge([Tq[0]] * Q, occ)                                # equal rows -> that row
    live = tot > 0
    np.testing.assert_allclose(same[live], Tq[0][live], rtol=0, atol=1e-7)


# ---------------------------------------------------------------- f1: the chunked pipeline

def test_q1_chunked_equals_unchunked_bitwise():
    """Q = 1 end to end is bit-identical to the unchunked pipeline (w = 1 exactly;
    nodes in no edge have the zero row in both after one step)."""
    for seed in range(20):
        g = gen.tiny_graph(seed)
        M = oracle.build_from(g)
        T = oracle.embed(M, 8, 4, 3)
        C = oracle.embed_chunked(g.src, g.dst, g.w, g.n, g.directed, 1, 99, 8, 4, 3)
        assert T.tobytes() == C.tobytes()


@pytest.mark.parametrize("seed", range(40))
def test_chunked_embedding_vs_dense_brute_force(seed):
    g = gen.tiny_graph(seed, n_max=30, e_max=120)
    Q, d, iters = 1 + seed % 4, 1 + seed % 7, 1 + seed % 4
    T, parts, occ, chunk = oracle.embed_chunked(g.src, g.dst, g.w, g.n, g.directed, Q, seed, d, 7, iters,
                                                return_parts=True)
    for q in range(Q):
        m = chunk == q
        if not m.any():
            continue
        ref = dense_embed(g.src[m], g.dst[m], None if g.w is None else g.w[m], g.n, g.directed, d, 7, iters)
        np.testing.assert_allclose(parts[q], ref, rtol=0, atol=2e-6)
    tot = occ.sum(0)
    w = np.divide(occ, tot, out=np.zeros(occ.shape), where=tot > 0)
    ref = sum(w[q][:, None] * parts[q].astype(np.float64) for q in range(Q))
    np.testing.assert_allclose(T, ref, rtol=0, atol=2e-7)


# ---------------------------------------------------------------- f2: inductive embedding

def test_reconstruct_reproduces_the_last_training_step():
    """SPEC.md:365 [DERIVED]: reconstructing every training node from its own edges and
    T_{I-1} gives T_I -- bitwise here (unit weights: identical sums in identical order)."""
    g = gen.config("c1")
    M = oracle.build_from(g)
    Ts = oracle.embed(M, 32, 0, 3, keep_all=True)
    # each undirected edge as two directed (new node -> known node) edges
    src = np.concatenate([g.src, g.dst])
    dst = np.concatenate([g.dst, g.src])
    R = oracle.reconstruct(src, dst, None, g.n, Ts[2])
    assert R.tobytes() == Ts[3].tobytes()


def test_reconstruct_closed_forms():
    rng = np.random.default_rng(2)
    d = 12
    T = rng.standard_normal((5, d)).astype(np.float32)
    # a new node with a single neighbour b gets T[b] / ||T[b]|| (leaf node)
    R = oracle.reconstruct(np.array([0], np.int32), np.array([3], np.int32), None, 1, T)
    np.testing.assert_allclose(R[0], T[3] / np.linalg.norm(T[3].astype(np.float64)), rtol=0, atol=1e-7)
    # two orthogonal unit neighbours with equal weights: cosine 1/sqrt(2) to each
    U = np.zeros((2, 4), np.float32)
    U[0, 0] = 1.0
    U[1, 2] = 1.0
    R = oracle.reconstruct(np.array([0, 0], np.int32), np.array([0, 1], np.int32), None, 1, U)
    assert np.allclose(R[0] @ U.T, [2 ** -0.5] * 2, atol=1e-7)
    # weights: 3:1 towards node 0
    R = oracle.reconstruct(np.array([0, 0], np.int32), np.array([0, 1], np.int32),
                           np.array([3.0, 1.0], np.float32), 1, U)
    np.testing.assert_allclose(R[0], np.array([3, 0, 1, 0]) / np.sqrt(10), rtol=0, atol=1e-7)
    # a new node without edges stays zero (reading RZ); unit norms otherwise; order-free
    R = oracle.reconstruct(np.array([1, 1, 1], np.int32), np.array([2, 4, 0], np.int32), None, 3, T)
    assert not R[0].any() and not R[2].any()
    assert abs(np.linalg.norm(R[1]) - 1) < 1e-6
    R2 = oracle.reconstruct(np.array([1, 1, 1], np.int32), np.array([4, 0, 2], np.int32), None, 3, T)
    assert R.tobytes() == R2.tobytes()


# ---------------------------------------------------------------- f3: hypergraph expansion

def _random_hypergraph(seed, n=40, n_he=30, kmax=7):
    rng = np.random.default_rng(seed)
    k = rng.integers(1, kmax + 1, n_he)
    ptr = np.concatenate([[0], np.cumsum(k)]).astype(np.int64)
    nodes = rng.integers(0, n, ptr[-1]).astype(np.int32)          # duplicates inside a hyperedge happen
    return ptr, nodes, rng.lognormal(0, 1, n_he).astype(np.float32)


def test_expansion_spec_examples():
    # SPEC.md:136 star {c,p,s} -> virtual h, edges (h,c),(h,p),(h,s); width 1 -> one edge
    s, d, w = oracle.expand_star([0, 3, 4], [5, 6, 7, 2], 10)
    assert list(zip(s.tolist(), d.tolist())) == [(10, 5), (10, 6), (10, 7), (11, 2)]
    # 1000 hyperedges of width 4 -> 1000 virtual nodes, 4000 edges
    ptr = np.arange(0, 4001, 4)
    s, d, _ = oracle.expand_star(ptr, np.arange(4000) % 97, 97)
    assert s.size == 4000 and np.unique(s).size == 1000 and s.min() == 97
    # clique of {u,v,w} -> (u,v),(u,w),(v,w); width 2 is the identity; no self-loops
    s, d, _ = oracle.expand_clique([0, 3], [1, 2, 3])
    assert list(zip(s.tolist(), d.tolist())) == [(1, 2), (1, 3), (2, 3)]
    s, d, _ = oracle.expand_clique([0, 2], [4, 9])
    assert list(zip(s.tolist(), d.tolist())) == [(4, 9)]
    s, d, _ = oracle.expand_clique([0, 3], [4, 4, 9])
    assert list(zip(s.tolist(), d.tolist())) == [(4, 9), (4, 9)]


@pytest.mark.parametrize("seed", range(10))
def test_expansion_counts_against_incidence_algebra(seed):
    """Clique: the unordered pair {u,v} (u != v) appears sum_e mult_e(u) mult_e(v) times, i.e. the
    off-diagonal of H^T H for the hyperedge-node multiplicity matrix H.  Star: the
    graph is bipartite original/virtual and node v is joined to hyperedge e mult_e(v) times."""
    ptr, nodes, w = _random_hypergraph(seed)
    n, n_he = 40, len(ptr) - 1
    H = np.zeros((n_he, n), np.int64)
    for e in range(n_he):
        np.add.at(H[e], nodes[ptr[e]:ptr[e + 1]], 1)
    s, d, ww = oracle.expand_clique(ptr, nodes, w)
    C = np.zeros((n, n), np.int64)
    np.add.at(C, (np.minimum(s, d), np.maximum(s, d)), 1)
    G = H.T @ H
    assert np.array_equal(C, np.triu(G, 1))
    assert not (s == d).any()
    s, d, ww = oracle.expand_star(ptr, nodes, n, w)
    assert (s >= n).all() and (d < n).all()                         # bipartite
    S = np.zeros((n_he, n), np.int64)
    np.add.at(S, (s - n, d), 1)
    assert np.array_equal(S, H)
    assert np.array_equal(ww, np.repeat(w, np.diff(ptr)))
