"""Pins for the CPU oracle (runs without a GPU).

Every test here checks oracle/ against something other than itself: a dense numpy
brute force (tests/_dense.py), worked examples (tests/golden/), closed forms and
invariants the paper states, or an independent pure-Python-integer hash.  Citations
are PAPER.md (arXiv 2102.02302) and SPEC.md lines.
"""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

import gen
import oracle
from tests._dense import dense_A, dense_M, dense_embed, normalize_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def f32_bits(x):
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


def csr_to_dense(M):
    D = np.zeros((M.n, M.n), np.float64)
    for a in range(M.n):
        for k in range(M.row_ptr[a], M.row_ptr[a + 1]):
            D[a, M.col[k]] = M.val[k]
    return D


# ----------------------------------------------------------------------------- I1 (init)

def _py_mix(z):
    M64 = (1 << 64) - 1
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 & M64
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB & M64
    return z ^ (z >> 31)


def test_hash_golden_values(golden_dir):
    """Oracle T_0 bit-equal to the survey's pure-Python-integer goldens (reading I1)."""
    rows = [l.split() for l in open(os.path.join(golden_dir, "hash_init_I1.tsv")) if l.strip() and not l.startswith("#")]
    assert len(rows) == 7
    for seed, v, j, h_hex, bits_hex in rows:
        seed, v, j = int(seed), int(v), int(j)
        x = oracle.hash_value(seed, v, j)
        assert f32_bits(x) == int(bits_hex, 16), (seed, v, j)
        # the stored hash word reproduces the stored value: (int(h>>40) - 2^23) * 2^-23
        h = int(h_hex, 16)
        assert x == ((h >> 40) - (1 << 23)) / float(1 << 23)


def test_hash_matches_python_integers_on_random_points():
    rng = np.random.default_rng(7)
    for _ in range(200):
        seed = int(rng.integers(0, 2**63)); v = int(rng.integers(0, 2**31 - 1)); j = int(rng.integers(0, 4096))
        s = _py_mix((seed + 0x9E3779B97F4A7C15) & ((1 << 64) - 1))
        h = _py_mix(s ^ ((v << 32) | j))
        assert oracle.hash_value(seed, v, j) == ((h >> 40) - (1 << 23)) / float(1 << 23)


def test_hash_init_is_uniform_minus1_1():
    """T_0 ~ U(-1,1): range, mean, variance, histogram flatness."""
    T = oracle.hash_init(4000, 256, seed=0).astype(np.float64)
    x = T.ravel()
    n = x.size
    assert x.min() >= -1.0 and x.max() < 1.0
    assert abs(x.mean()) < 5 * np.sqrt(1 / 3 / n)
    assert abs(x.var() - 1 / 3) < 5 * np.sqrt((1 / 5 - 1 / 9) / n) * 1.5
    hist, _ = np.histogram(x, bins=64, range=(-1, 1))
    expect = n / 64
    chi2 = ((hist - expect) ** 2 / expect).sum()
    assert chi2 < 63 + 6 * np.sqrt(2 * 63)   # ~6 sigma on a chi-square with 63 dof


def test_hash_init_rows_nearly_orthogonal():
    """rows 'different from each other' with 'similar pairwise distances':
    pairwise cosine of independent U(-1,1) rows has sd 1/sqrt(d) (SPEC.md:248 as a distribution)."""
    d = 1024
    T = oracle.hash_init(600, d, seed=3).astype(np.float64)
    U = normalize_rows(T)
    C = U @ U.T
    off = C[np.triu_indices(600, 1)]
    assert abs(off.mean()) < 0.01
    assert abs(off.std() - 1 / np.sqrt(d)) < 0.1 / np.sqrt(d)


def test_hash_init_id_keyed():
    """Row v depends only on (seed, v): any row window reproduces the same values."""
    a = oracle.hash_init(100, 33, seed=11)
    b = oracle.hash_init(40, 33, seed=11, row_begin=50)
    np.testing.assert_array_equal(a[50:90], b)
    c = oracle.hash_init(100, 33, seed=12)
    assert not np.array_equal(a, c)


# ----------------------------------------------------------------------------- B1-B4 (M)

def test_build_spec_examples(golden_dir):
    ex = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for case in ex["build_transition"]:
        e = np.array(case["edges"])
        M = oracle.build_csr(e[:, 0].astype(np.int32), e[:, 1].astype(np.int32), e[:, 2].astype(np.float32),
                             case["n"], case["directed"])
        got = {}
        gote = {}
        for a in range(M.n):
            for k in range(M.row_ptr[a], M.row_ptr[a + 1]):
                got[f"{a},{M.col[k]}"] = float(M.val[k])
                gote[f"{a},{M.col[k]}"] = float(M.e[k])
        assert got == case["M"], case["cite"]
        for key, val in case.get("e", {}).items():
            assert gote[key] == val, case["cite"]


@pytest.mark.parametrize("seed", range(200))
def test_build_matches_dense_bruteforce(seed):
    """CSR M equals the dense D^-1 A on random multigraphs with
    duplicates, self-loops, weights, both directions."""
    g = gen.tiny_graph(seed)
    M = oracle.build_csr(g.src, g.dst, g.w, g.n, g.directed)
    A = dense_A(g.src, g.dst, g.w, g.n, g.directed)
    Md, deg = dense_M(A)
    # structure: exactly the non-zero pattern of A, sorted by column within rows
    assert M.nnz == int((A != 0).sum())
    for a in range(g.n):
        cols = M.col[M.row_ptr[a]:M.row_ptr[a + 1]]
        assert np.array_equal(cols, np.nonzero(A[a])[0])
    np.testing.assert_allclose(M.deg, deg, rtol=1e-13, atol=0)
    # values: one fp32 rounding of the fp64 quotient (within 1 ulp of the dense quotient)
    D = csr_to_dense(M)
    np.testing.assert_allclose(D, Md, rtol=2 ** -23, atol=0)
    # e_ab
    E = np.zeros_like(A)
    for a in range(g.n):
        for k in range(M.row_ptr[a], M.row_ptr[a + 1]):
            E[a, M.col[k]] = M.e[k]
    np.testing.assert_allclose(E, A, rtol=1e-13, atol=0)


def test_build_row_stochastic_and_weight_scale_invariant():
    """Every non-empty row of M sums to 1 +- 1e-6; global weight scaling
    leaves M unchanged (M_ab = e_ab/deg(a) is homogeneous of degree 0)."""
    g = gen.config("c1")
    rng = np.random.default_rng(0)
    w = rng.lognormal(0, 1, size=g.n_edges).astype(np.float32)
    M1 = oracle.build_csr(g.src, g.dst, w, g.n, False)
    M2 = oracle.build_csr(g.src, g.dst, (w * np.float32(4.0)), g.n, False)   # exact power-of-2 scale
    sums = np.add.reduceat(M1.val.astype(np.float64), M1.row_ptr[:-1])
    assert np.all(np.abs(sums - 1) < 1e-6)
    np.testing.assert_array_equal(M1.val, M2.val)
    np.testing.assert_array_equal(M1.col, M2.col)


def test_build_rejects_bad_input():
    src = np.array([0, 1], np.int32); dst = np.array([1, 2], np.int32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_csr(src, dst, None, 2, False)      # id 2 >= n
    assert e.value.code == oracle.EDATA
    for bad in (0.0, -1.0, np.nan, np.inf):
        with pytest.raises(oracle.OracleError) as e:
            oracle.build_csr(src, np.array([1, 0], np.int32), np.array([1.0, bad], np.float32), 2, False)
        assert e.value.code == oracle.EDATA
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_csr(np.array([], np.int32), np.array([], np.int32), None, 2, False)
    assert e.value.code == oracle.EUSAGE


def test_build_undirected_mirror_and_selfloop_once():
    """Undirected edges are counted in both directions; a self-loop once (reading 5)."""
    M = oracle.build_csr(np.array([0, 0], np.int32), np.array([0, 1], np.int32), None, 2, False)
    # row 0: self-loop (e=1) + edge to 1 (e=1) -> 0.5, 0.5 ; row 1: edge to 0 -> 1.0
    assert list(M.col) == [0, 1, 0]
    assert list(M.val) == [0.5, 0.5, 1.0]
    assert list(M.deg) == [2.0, 1.0]


# ----------------------------------------------------------------------------- O1 (iteration)

@pytest.mark.parametrize("seed", range(200))
def test_embed_matches_dense_bruteforce(seed):
    """Oracle T_I equals dense normalize(M @ T) iterated (fp64 math, fp32 storage each
    iteration) on random graphs: |V|<=50, |E|<=200, d<=16, I<=6."""
    g = gen.tiny_graph(seed)
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.integers(1, 17)); iters = int(rng.integers(1, 7))
    M = oracle.build_csr(g.src, g.dst, g.w, g.n, g.directed)
    Ts = oracle.embed(M, d, seed, iters, keep_all=True)
    Md, _ = dense_M(dense_A(g.src, g.dst, g.w, g.n, g.directed))
    Ds, cond = dense_embed(Md, Ts[0], iters, return_cond=True)
    for i in range(iters + 1):
        if cond[i] < 1e-4:   # near-exact cancellation (e.g. d=1, rows of +-1): direction ill-defined
            break
        np.testing.assert_allclose(Ts[i], Ds[i], rtol=0, atol=1e-6, err_msg=f"iteration {i}")
        # zero-row sets identical, exactly (reading Z)
        assert np.array_equal(~Ts[i].any(axis=1), ~Ds[i].astype(np.float32).any(axis=1)) or i == 0


def test_step_spec_normalize_examples(golden_dir):
    """SPEC.md:201-203 via a graph whose M is the identity (one self-loop per node)."""
    ex = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for case in ex["l2_normalize_rows"]:
        row = np.array([case["row"]], np.float32)
        M = oracle.build_csr(np.array([0], np.int32), np.array([0], np.int32), None, 1, False)
        out = oracle.step(M, row)
        np.testing.assert_allclose(out[0], case["out"], rtol=0, atol=1e-7, err_msg=case["cite"])


def test_two_node_graph_swaps_rows():
    """a<->b, I=1: T_1[a] = normalize(T_0[b]), T_1[b] = normalize(T_0[a])."""
    M = oracle.build_csr(np.array([0], np.int32), np.array([1], np.int32), None, 2, False)
    T0 = oracle.hash_init(2, 64, seed=5).astype(np.float64)
    T1 = oracle.step(M, T0.astype(np.float32))
    np.testing.assert_allclose(T1[0], T0[1] / np.linalg.norm(T0[1]), atol=6e-8)
    np.testing.assert_allclose(T1[1], T0[0] / np.linalg.norm(T0[0]), atol=6e-8)


def test_star_graph_leaves_collapse():
    """Star with centre 0: after iteration 1 every leaf equals normalize(T_0[0]) exactly
    (each leaf has one neighbour; PAPER.md:515 'leaf nodes ... equal to the embedding of
    their single neighbor from the previous iteration')."""
    k = 30
    M = oracle.build_csr(np.zeros(k, np.int32), np.arange(1, k + 1, dtype=np.int32), None, k + 1, False)
    T = oracle.embed(M, 32, seed=1, iters=1)
    for leaf in range(1, k + 1):
        np.testing.assert_array_equal(T[leaf], T[1])
    T0 = oracle.hash_init(1, 32, seed=1)[0].astype(np.float64)
    np.testing.assert_allclose(T[1], T0 / np.linalg.norm(T0), atol=6e-8)
    # the centre is the normalised mean of the leaves
    L = oracle.hash_init(k + 1, 32, seed=1)[1:].astype(np.float64).mean(0)
    np.testing.assert_allclose(T[0], L / np.linalg.norm(L), atol=1e-7)


def test_complete_bipartite_period_two():
    """K_{m,n}: after iteration 1 all left rows are identical, likewise all right rows;
    from then on iteration i+2 equals iteration i (period 2)."""
    m, n = 4, 7
    src = np.repeat(np.arange(m), n).astype(np.int32)
    dst = (m + np.tile(np.arange(n), m)).astype(np.int32)
    M = oracle.build_csr(src, dst, None, m + n, False)
    Ts = oracle.embed(M, 48, seed=9, iters=5, keep_all=True)
    for T in Ts[1:]:
        for r in range(1, m):
            np.testing.assert_array_equal(T[r], T[0])
        for r in range(m + 1, m + n):
            np.testing.assert_array_equal(T[r], T[m])
    np.testing.assert_allclose(Ts[3], Ts[1], atol=1e-7)
    np.testing.assert_allclose(Ts[4], Ts[2], atol=1e-7)


def test_complete_graph_collapses():
    """'Too large iteration number will make all embeddings gradually more
    similar ... eventually collapsing to an exact same representation'.  On K_n,
    1 - min pairwise cosine decreases monotonically towards 0."""
    n = 10
    iu = np.triu_indices(n, 1)
    M = oracle.build_csr(iu[0].astype(np.int32), iu[1].astype(np.int32), None, n, False)
    Ts = oracle.embed(M, 64, seed=2, iters=6, keep_all=True)
    spread = []
    for T in Ts[1:]:
        U = normalize_rows(T.astype(np.float64))
        spread.append(1 - (U @ U.T).min())
    assert all(b < a for a, b in zip(spread, spread[1:])), spread
    assert spread[-1] < 1e-6


def test_iteration_collapse_connected_nonbipartite():
    """connected non-bipartite 20-node graph, I=64: mean pairwise cosine >= 0.99."""
    n = 20
    rng = np.random.default_rng(0)
    # a 20-cycle (connected) plus 40 random chords, including the triangle 0-1-2 (non-bipartite)
    cs, cd = rng.integers(0, n, 40), rng.integers(0, n, 40)
    keep = cs != cd
    src = np.concatenate([np.arange(n), [0], cs[keep]]).astype(np.int32)
    dst = np.concatenate([(np.arange(n) + 1) % n, [2], cd[keep]]).astype(np.int32)
    M = oracle.build_csr(src, dst, None, n, False)
    T = oracle.embed(M, 16, seed=4, iters=64).astype(np.float64)
    C = T @ T.T
    assert C[np.triu_indices(n, 1)].mean() >= 0.99


def test_leaf_equals_previous_neighbour_row():
    """PAPER.md:515 on a random graph: every node with exactly one neighbour b gets
    T_i[leaf] = T_{i-1}[b] / ||T_{i-1}[b]|| (exact up to the fp32 store)."""
    g = gen.er(300, 330, seed=3)
    M = oracle.build_csr(g.src, g.dst, None, g.n, False)
    Ts = oracle.embed(M, 24, seed=0, iters=4, keep_all=True)
    deg = np.diff(M.row_ptr)
    leaves = np.nonzero(deg == 1)[0]
    assert len(leaves) > 20
    for i in range(1, 5):
        for a in leaves:
            b = M.col[M.row_ptr[a]]
            prev = Ts[i - 1][b].astype(np.float64)
            nrm = np.linalg.norm(prev)
            exp = prev / nrm if nrm > 0 else prev
            np.testing.assert_allclose(Ts[i][a], exp, atol=6e-8)


def test_disjoint_components_independent():
    """Rows of component G1 inside G1 u G2 are bit-identical to G1 embedded alone (same ids)."""
    g1 = gen.er(80, 200, seed=1)
    g2 = gen.er(60, 150, seed=2)
    src = np.concatenate([g1.src, g2.src + 80]).astype(np.int32)
    dst = np.concatenate([g1.dst, g2.dst + 80]).astype(np.int32)
    Mu = oracle.build_csr(src, dst, None, 140, False)
    M1 = oracle.build_csr(g1.src, g1.dst, None, 80, False)
    Tu = oracle.embed(Mu, 40, seed=6, iters=4)
    T1 = oracle.embed(M1, 40, seed=6, iters=4)
    np.testing.assert_array_equal(Tu[:80], T1)


def test_scale_invariance_and_unit_norms():
    """normalize(M (cT)) = normalize(M T) for c > 0; every non-zero row has
    unit norm after each step (Alg. 1 line 7 'L2 normalize rows')."""
    g = gen.config("c1")
    M = oracle.build_from(g)
    T0 = oracle.hash_init(g.n, 32, seed=0)
    a = oracle.step(M, T0)
    b = oracle.step(M, (T0 * np.float32(8.0)))        # exact scaling by 2^3
    np.testing.assert_array_equal(a, b)
    c = oracle.step(M, (T0 * np.float32(0.3)))
    np.testing.assert_allclose(a, c, atol=2e-7)
    for T in oracle.embed(M, 32, seed=0, iters=4, keep_all=True)[1:]:
        nr = np.linalg.norm(T.astype(np.float64), axis=1)
        assert np.all(np.abs(nr - 1) < 1e-6)


def test_directed_sink_rows_zero_and_stay_zero():
    """Reading 3 / Z: directed rows average OUT-neighbours; a sink row is 0 and stays 0."""
    # 0 -> 1 -> 2, 2 is a sink; 3 -> 0
    src = np.array([0, 1, 3], np.int32); dst = np.array([1, 2, 0], np.int32)
    M = oracle.build_csr(src, dst, None, 4, True)
    Ts = oracle.embed(M, 16, seed=0, iters=3, keep_all=True)
    T0 = Ts[0].astype(np.float64)
    np.testing.assert_allclose(Ts[1][0], T0[1] / np.linalg.norm(T0[1]), atol=6e-8)
    np.testing.assert_allclose(Ts[1][1], T0[2] / np.linalg.norm(T0[2]), atol=6e-8)
    for T in Ts[1:]:
        assert not T[2].any()
    assert not Ts[2][1].any()     # 1's only neighbour became zero at iteration 1
    assert not Ts[3][0].any()


def test_oracle_independent_of_thread_count():
    """Rows are computed sequentially, so the output bytes do not depend on OMP threads."""
    code = ("import numpy as np, gen, oracle, sys;"
            "g=gen.config('c1'); M=oracle.build_from(g); T=oracle.embed(M,64,0,3);"
            "sys.stdout.write(__import__('hashlib').sha256(T.tobytes()+M.val.tobytes()).hexdigest())")
    outs = []
    for nt in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=nt, PYTHONPATH=ROOT)
        outs.append(subprocess.check_output([sys.executable, "-c", code], env=env, cwd=ROOT).decode())
    assert outs[0] == outs[1]
