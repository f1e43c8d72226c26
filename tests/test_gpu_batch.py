"""many graphs in one handle (cleora_build_batch): block-diagonal M, one fused
SpMM launch per step for all of them.  Every graph's rows must be BITWISE the result of building
and embedding that graph alone (same entries, same per-row schedule, T_0 keyed on the local id),
and within the bars of the oracle run on that graph alone (one embedding per
relation pair, computed independently).
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


def _batch(graphs):
    ep = np.zeros(len(graphs) + 1, np.int64)
    ep[1:] = np.cumsum([g.n_edges for g in graphs])
    src = np.concatenate([g.src for g in graphs])
    dst = np.concatenate([g.dst for g in graphs])
    w = np.concatenate([g.w for g in graphs]) if graphs[0].w is not None else None
    return src, dst, w, ep, np.array([g.n for g in graphs], np.int32)


@pytest.mark.parametrize("directed,weighted", [(False, False), (True, True)])
@pytest.mark.parametrize("d", [3, 64, 256, 1024])
def test_batch_equals_separate_runs(cl, directed, weighted, d, monkeypatch):
    # bitwise against each graph run alone: every step normalised (a batch at d = 1024 may run half-row
    # passes where a graph alone does not; lazy steps, reading R21, are bitwise only against themselves
    # and are checked against the oracle in test_gpu_parity.py)
    monkeypatch.setenv("CLEORA_LAZY", "0")
    rng = np.random.default_rng(d + directed)
    graphs = []
    for i in range(40):
        g = gen.tiny_graph(1000 + i, n_max=300, e_max=2000, directed=directed, weighted=weighted)
        graphs.append(g)
    # a hub graph (heavy rows inside a batch) and a single-node graph with a self-loop
    hub_src = np.concatenate([np.zeros(3000, np.int32), rng.integers(0, 3500, 4000).astype(np.int32)])
    hub_dst = np.concatenate([np.arange(1, 3001, dtype=np.int32), rng.integers(0, 3500, 4000).astype(np.int32)])
    graphs.insert(7, gen.EdgeList("hub", 3500, hub_src, hub_dst,
                                  rng.lognormal(0, 1, 7000).astype(np.float32) if weighted else None, directed))
    graphs.append(gen.EdgeList("one", 1, np.zeros(1, np.int32), np.zeros(1, np.int32),
                               np.ones(1, np.float32) if weighted else None, directed))
    src, dst, w, ep, nc = _batch(graphs)
    iters = 3
    B = cl.cleora_build_batch(src, dst, w, ep, nc, directed, device=0)
    try:
        assert cl.cleora_info(B)["n_graphs"] == len(graphs)
        cl.cleora_init(B, d, 5)
        T0 = cl.cleora_fetch(B)
        cl.cleora_iterate(B, iters)
        T = cl.cleora_fetch(B)
    finally:
        B.close()
    base = np.concatenate([[0], np.cumsum(nc)])
    for i, g in enumerate(graphs):
        rows = slice(base[i], base[i + 1])
        assert np.array_equal(T0[rows].view(np.uint32), oracle.hash_init(g.n, d, 5).view(np.uint32)), g.name
        G = cl.cleora_build(g.src, g.dst, g.w, g.n, directed, device=0)
        cl.cleora_init(G, d, 5)
        cl.cleora_iterate(G, iters)
        alone = cl.cleora_fetch(G)
        G.close()
        assert T[rows].tobytes() == alone.tobytes(), f"graph {i} ({g.name}) differs from its own run"
        R = oracle.embed(oracle.build_from(g), d, 5, iters)
        Tg = T[rows].astype(np.float64)
        assert float(np.abs(Tg - R).max()) <= 1e-5, g.name
        assert np.array_equal(~T[rows].any(1), ~R.any(1)), g.name
        nz = R.any(1)                       # BASELINE north star: cosine >= 0.99999 per non-zero row
        if nz.any():
            cos = (Tg[nz] * R[nz]).sum(1) / (np.linalg.norm(Tg[nz], axis=1) * np.linalg.norm(R[nz], axis=1))
            assert float(cos.min()) >= 0.99999, f"{g.name}: min cosine {cos.min()}"


def test_batch_id_errors(cl):
    src = np.array([0, 1, 0], np.int32)
    dst = np.array([1, 2, 1], np.int32)
    with pytest.raises(cl.CleoraError) as e:       # graph 1 has 2 nodes: local id 2 is out of range
        cl.cleora_build_batch(src, dst, None, np.array([0, 1, 3], np.int64), np.array([2, 2], np.int32), device=0)
    assert e.value.code == cl.EDATA and "edge 1" in str(e.value)
