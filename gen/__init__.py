"""Seeded synthetic inputs shared by the oracle and the CUDA path (TEST / BENCH INFRASTRUCTURE).

This module draws graphs only.  It holds none of Cleora's arithmetic (no transition
matrix, degree, embedding or normalisation), so sharing it between ``oracle/`` and
the product path shares inputs, not computation (task rule ③).

The five configurations are BASELINE.json ``configs[0..4]``; they stand in for the
paper's Table 1 datasets (Table 1: Facebook, YouTube, RoadNet,
LiveJournal, Twitter), which are not available here.  Recipes: SURVEY.md §8(d) and
DESIGN.md "Input recipe".  The C generators live in ``cleora_gen.c`` (counter-based
SplitMix64 RNG, OpenMP, deterministic for any thread count).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cleora_gen.c")
_LIB = os.path.join(_HERE, "libcleora_gen.so")
_lib = None


def build_lib(force: bool = False) -> str:
    """Compile cleora_gen.c into libcleora_gen.so (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        build_lib()
        lib = ctypes.CDLL(_LIB)
        i32p = ctypes.POINTER(ctypes.c_int32)
        f32p = ctypes.POINTER(ctypes.c_float)
        u64, i64, i32, dbl = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        lib.gen_u64.restype = u64
        lib.gen_u64.argtypes = [u64, u64, u64]
        lib.gen_unif.restype = dbl
        lib.gen_unif.argtypes = [u64, u64, u64]
        lib.gen_permutation.restype = ctypes.c_int
        lib.gen_permutation.argtypes = [i32, u64, i32p]
        lib.gen_er.restype = i64
        lib.gen_er.argtypes = [i32, i64, u64, i32p, i32p]
        lib.gen_chung_lu.restype = i64
        lib.gen_chung_lu.argtypes = [i32, i64, dbl, dbl, dbl, u64, i32p, i32p]
        lib.gen_lattice.restype = i64
        lib.gen_lattice.argtypes = [i32, dbl, dbl, u64, i32p, i32p]
        lib.gen_rmat_directed.restype = i64
        lib.gen_rmat_directed.argtypes = [i32, i32, i64, dbl, dbl, dbl, dbl, dbl, u64, i32p, i32p, f32p]
        lib.gen_rmat_undirected.restype = i64
        lib.gen_rmat_undirected.argtypes = [i32, i32, i64, dbl, dbl, dbl, u64, i32p, i32p]
        _lib = lib
    return _lib


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


@dataclass
class EdgeList:
    """A COO edge list as the C-ABI takes it: ``src[E]``, ``dst[E]`` int32, optional fp32 ``w[E]``."""
    name: str
    n: int
    src: np.ndarray
    dst: np.ndarray
    w: np.ndarray | None
    directed: bool
    d: int = 0
    iters: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def n_edges(self) -> int:
        return int(self.src.shape[0])


# BASELINE.json configs[0..4]; SURVEY.md §8(d) generator specs.
CONFIGS = {
    "c1": dict(kind="er", n=10_000, m=50_000, d=128, iters=4, directed=False,
               desc="Erdos-Renyi undirected, N=10,000, 50,000 edges, unit weights, d=128, I=4"),
    "c2": dict(kind="chung_lu", n=1_134_890, pairs=2_987_624, gamma=2.1, i0=9.5388, c=233_115.5,
               d=1024, iters=4, directed=False,
               desc="Chung-Lu power law (gamma=2.1) undirected, N=1,134,890, ~2.84M edges, d=1024, I=4 (YouTube stand-in)"),
    "c3": dict(kind="lattice", side=1050, p_del=0.3, p_diag=0.02, d=1024, iters=5, directed=False,
               desc="damaged 1050x1050 lattice + 2% diagonals, ~1.56M undirected edges, d=1024, I=5 (RoadNet stand-in)"),
    "c4": dict(kind="rmat_dir", n=4_847_571, scale=23, m=68_993_773, abc=(0.57, 0.19, 0.19),
               mu=0.0, sigma=1.0, d=1024, iters=4, directed=True,
               desc="R-MAT directed, lognormal weights, N=4,847,571, 68,993,773 edges (dups kept), d=1024, I=4 (LiveJournal stand-in)"),
    "c5": dict(kind="rmat_und", n=41_652_230, scale=26, samples=1_468_365_182, abc=(0.57, 0.19, 0.19),
               d=256, iters=4, directed=False,
               desc="R-MAT undirected, N=41,652,230, 1.468B samples deduped, d=256, I=4 (Twitter stand-in)"),
}


def er(n: int, m: int, seed: int = 0) -> EdgeList:
    src = np.empty(m, np.int32); dst = np.empty(m, np.int32)
    got = _L().gen_er(n, m, seed, _p(src, ctypes.c_int32), _p(dst, ctypes.c_int32))
    if got < 0:
        raise MemoryError("gen_er")
    return EdgeList(f"er{n}_{m}", n, src[:got].copy(), dst[:got].copy(), None, False)


def chung_lu(n: int, pairs: int, gamma: float, i0: float, c: float, seed: int = 0) -> EdgeList:
    src = np.empty(pairs, np.int32); dst = np.empty(pairs, np.int32)
    got = _L().gen_chung_lu(n, pairs, gamma, i0, c, seed, _p(src, ctypes.c_int32), _p(dst, ctypes.c_int32))
    if got < 0:
        raise MemoryError("gen_chung_lu")
    return EdgeList(f"chung_lu{n}", n, src[:got].copy(), dst[:got].copy(), None, False)


def lattice(side: int, p_del: float, p_diag: float, seed: int = 0) -> EdgeList:
    cap = 2 * side * (side - 1) + (side - 1) ** 2
    src = np.empty(cap, np.int32); dst = np.empty(cap, np.int32)
    got = _L().gen_lattice(side, p_del, p_diag, seed, _p(src, ctypes.c_int32), _p(dst, ctypes.c_int32))
    return EdgeList(f"lattice{side}", side * side, src[:got].copy(), dst[:got].copy(), None, False)


def rmat_directed(n, scale, m, abc, mu, sigma, seed=0) -> EdgeList:
    src = np.empty(m, np.int32); dst = np.empty(m, np.int32); w = np.empty(m, np.float32)
    got = _L().gen_rmat_directed(n, scale, m, abc[0], abc[1], abc[2], mu, sigma, seed,
                                 _p(src, ctypes.c_int32), _p(dst, ctypes.c_int32), _p(w, ctypes.c_float))
    if got < 0:
        raise MemoryError("gen_rmat_directed")
    return EdgeList(f"rmat_dir{n}", n, src, dst, w, True)


def rmat_undirected(n, scale, samples, abc, seed=0) -> EdgeList:
    src = np.empty(samples, np.int32); dst = np.empty(samples, np.int32)
    got = _L().gen_rmat_undirected(n, scale, samples, abc[0], abc[1], abc[2], seed,
                                   _p(src, ctypes.c_int32), _p(dst, ctypes.c_int32))
    if got < 0:
        raise MemoryError("gen_rmat_undirected")
    # shrink without a second full copy when possible
    return EdgeList(f"rmat_und{n}", n, np.resize(src, got) if got != samples else src,
                    np.resize(dst, got) if got != samples else dst, None, False)


def _cache_path(name: str, seed: int):
    d = os.environ.get("CLEORA_GEN_CACHE")
    return os.path.join(d, f"{name}_s{seed}.npz") if d else None


def config(name: str, seed: int = 0) -> EdgeList:
    """Generate BASELINE.json config ``name`` (c1..c5) with generator seed ``seed``.

    With ``CLEORA_GEN_CACHE=<dir>`` the edge arrays are kept in ``<dir>`` after the first
    generation (c5 takes minutes of host time) and loaded from there afterwards."""
    c = CONFIGS[name]
    path = _cache_path(name, seed)
    if path and os.path.exists(path):
        z = np.load(path)
        w = z["w"] if "w" in z.files else None
        g = EdgeList(name, int(z["n"]), z["src"], z["dst"], w, bool(z["directed"]))
        g.d, g.iters = c["d"], c["iters"]
        g.meta = dict(desc=c["desc"], seed=seed)
        return g
    g = _generate(name, seed)
    if path:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        extra = {"w": g.w} if g.w is not None else {}
        tmp = path + f".tmp{os.getpid()}.npz"
        np.savez(tmp, n=g.n, src=g.src, dst=g.dst, directed=g.directed, **extra)
        os.replace(tmp, path)
    return g


def _generate(name: str, seed: int) -> EdgeList:
    c = CONFIGS[name]
    k = c["kind"]
    if k == "er":
        g = er(c["n"], c["m"], seed)
    elif k == "chung_lu":
        g = chung_lu(c["n"], c["pairs"], c["gamma"], c["i0"], c["c"], seed)
    elif k == "lattice":
        g = lattice(c["side"], c["p_del"], c["p_diag"], seed)
    elif k == "rmat_dir":
        g = rmat_directed(c["n"], c["scale"], c["m"], c["abc"], c["mu"], c["sigma"], seed)
    elif k == "rmat_und":
        g = rmat_undirected(c["n"], c["scale"], c["samples"], c["abc"], seed)
    else:  # pragma: no cover
        raise KeyError(k)
    g.name = name
    g.d = c["d"]
    g.iters = c["iters"]
    g.meta = dict(desc=c["desc"], seed=seed)
    return g


def tiny_graph(seed: int, n_max: int = 50, e_max: int = 200, directed: bool | None = None,
               weighted: bool | None = None, allow_dups: bool = True, allow_self: bool = True) -> EdgeList:
    """Small random multigraph for brute-force tests (numpy PCG64, seeded).

    Exercises duplicates, self-loops, isolated nodes, weights and direction.
    """
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, n_max + 1))
    e = int(rng.integers(1, e_max + 1))
    if directed is None:
        directed = bool(rng.integers(0, 2))
    if weighted is None:
        weighted = bool(rng.integers(0, 2))
    src = rng.integers(0, n, size=e).astype(np.int32)
    dst = rng.integers(0, n, size=e).astype(np.int32)
    if not allow_self and n > 1:
        same = src == dst
        dst[same] = (dst[same] + 1) % n
    if allow_dups and e > 4:
        k = int(rng.integers(0, e // 4 + 1))
        idx = rng.integers(0, e, size=k)
        at = rng.integers(0, e, size=k)
        src[at] = src[idx]; dst[at] = dst[idx]
    w = None
    if weighted:
        w = rng.lognormal(0.0, 1.0, size=e).astype(np.float32)
    return EdgeList(f"tiny{seed}", n, src, dst, w, directed)


def unif(seed: int, stream: int, counter: int) -> float:
    """The generator's counter-based uniform draw (exposed for tests of the generator itself)."""
    return float(_L().gen_unif(seed, stream, counter))


def permutation(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.int32)
    if _L().gen_permutation(n, seed, _p(out, ctypes.c_int32)):
        raise MemoryError("gen_permutation")
    return out
