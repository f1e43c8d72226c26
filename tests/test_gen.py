"""Generator checks (CPU): the synthetic stand-ins have the shapes SURVEY.md §8(d) specifies."""
import numpy as np

import gen


def test_rng_is_counter_based_and_uniform():
    a = [gen.unif(0, 1, c) for c in range(20000)]
    assert a == [gen.unif(0, 1, c) for c in range(20000)]
    x = np.array(a)
    assert 0 <= x.min() and x.max() < 1
    assert abs(x.mean() - 0.5) < 0.01
    assert gen.unif(0, 1, 5) != gen.unif(0, 2, 5) != gen.unif(1, 1, 5)


def test_permutation():
    p = gen.permutation(1000, 3)
    assert np.array_equal(np.sort(p), np.arange(1000))
    assert not np.array_equal(p, np.arange(1000))


def test_c1_erdos_renyi():
    g = gen.config("c1")
    assert g.n == 10_000 and g.n_edges == 50_000 and not g.directed and g.w is None
    assert np.all(g.src < g.dst)                                   # canonical u < v, no self-loops
    key = g.src.astype(np.int64) * g.n + g.dst
    assert np.unique(key).size == 50_000                          # distinct pairs
    deg = np.bincount(np.concatenate([g.src, g.dst]), minlength=g.n)
    assert deg.sum() == 100_000 and deg.max() < 40
    g2 = gen.config("c1")
    assert np.array_equal(g.src, g2.src) and np.array_equal(g.dst, g2.dst)


def test_c2_chung_lu_shape():
    g = gen.config("c2")
    assert g.n == 1_134_890
    assert 2_780_000 < g.n_edges < 2_900_000                      # ~2.84M after dedupe
    assert np.all(g.src != g.dst)
    deg = np.bincount(np.concatenate([g.src, g.dst]), minlength=g.n)
    assert 15_000 < deg.max() < 30_000                             # hub ~20k (w_0 = 30,000)
    assert 0.20 < (deg == 0).mean() < 0.27                         # ~23.7% isolated


def test_c3_lattice_shape():
    g = gen.config("c3")
    assert g.n == 1050 * 1050
    assert 1_540_000 < g.n_edges < 1_590_000
    assert np.abs(g.src - g.dst).max() <= 1051
    deg = np.bincount(np.concatenate([g.src, g.dst]), minlength=g.n)
    assert deg.max() <= 8


def test_rmat_small_directed_keeps_duplicates():
    g = gen.rmat_directed(5000, 13, 100_000, (0.57, 0.19, 0.19), 0.0, 1.0, seed=0)
    assert g.directed and g.w is not None and g.w.dtype == np.float32
    assert np.all(g.src < 5000) and np.all(g.dst < 5000) and np.all(g.src != g.dst)
    key = g.src.astype(np.int64) * g.n + g.dst
    assert np.unique(key).size < g.n_edges                        # duplicates present
    lw = np.log(g.w.astype(np.float64))
    assert abs(lw.mean()) < 0.02 and abs(lw.std() - 1) < 0.02      # lognormal(0,1)
    outd = np.bincount(g.src, minlength=g.n)
    assert outd.max() > 20 * outd.mean()                          # power-law skew


def test_rmat_small_undirected_dedupes():
    g = gen.rmat_undirected(5000, 13, 100_000, (0.57, 0.19, 0.19), seed=0)
    lo = np.minimum(g.src, g.dst).astype(np.int64); hi = np.maximum(g.src, g.dst)
    assert np.unique(lo * g.n + hi).size == g.n_edges
    assert np.all(g.src != g.dst)


def test_tiny_graphs_cover_cases():
    kinds = set()
    for s in range(200):
        g = gen.tiny_graph(s)
        kinds.add((g.directed, g.w is not None))
        assert g.src.dtype == np.int32 and np.all(g.src < g.n)
    assert len(kinds) == 4
