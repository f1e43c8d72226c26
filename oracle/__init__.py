"""CPU ORACLE for Cleora's hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2102_02302_b200``) never imports it and shares no code with it.

The arithmetic lives in ``cleora_oracle.c`` (plain C + OpenMP over rows, fp64
accumulation, fp32 storage per iteration); this module only marshals arrays.
What each function computes, with the paper passage it follows
(PAPER.md = arXiv 2102.02302):

* :func:`build_csr` -- M = D^-1 A, ``M_ab = e_ab / deg(v_a)`` (PAPER.md:79-81,
  §3.2 "Embedding"; Algorithm 1 line 3), readings B1-B4.
* :func:`hash_init` -- ``T_0 ~ U(-1,1)`` (Alg. 1 line 4 PAPER.md:92)
  realised as the id-keyed hash of reading I1.  **Exact values: parity unpinned by
  the paper** (the paper fixes only the distribution, which the tests pin).
* :func:`step` -- one ``T_i = M T_{i-1}`` followed by row L2 normalisation
  (Alg. 1 lines 6-7).
* :func:`embed` -- Algorithm 1 with Q = 1 chunk.
* :func:`chunk_assign`, :func:`chunk_occurrences`, :func:`merge`, :func:`embed_chunked` --
  Algorithm 1 with Q > 1 chunks (lines 1-2 and 10-12), readings R13/R14.  The
  exact edge-to-chunk assignment (R13) is **parity unpinned by the paper**, which gives no rule;
  its properties (partition, determinism, uniformity) are pinned.
* :func:`reconstruct` -- a new node's embedding as the normalised weighted average of its
  neighbours' rows (§3.2): one row of normalize(M T) over the
  new nodes' own transition rows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cleora_oracle.c")
_LIB = os.path.join(_HERE, "libcleora_oracle.so")
_lib = None

OK, EUSAGE, EDATA, ENOMEM = 0, 2, 3, 4


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with code {code}")
        self.code = code


def build_lib(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -fopenmp; no -ffast-math: IEEE semantics matter)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        build_lib()
        lib = ctypes.CDLL(_LIB)
        vp = ctypes.c_void_p
        i32p, i64p = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)
        f32p, f64p = ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)
        lib.oracle_build.restype = ctypes.c_int
        lib.oracle_build.argtypes = [i32p, i32p, f32p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.POINTER(vp)]
        lib.oracle_csr_free.argtypes = [vp]
        lib.oracle_csr_nnz.restype = ctypes.c_int64
        lib.oracle_csr_nnz.argtypes = [vp]
        lib.oracle_csr_n.restype = ctypes.c_int32
        lib.oracle_csr_n.argtypes = [vp]
        lib.oracle_csr_copy.argtypes = [vp, i64p, i32p, f32p, f64p, f64p]
        lib.oracle_hash_value.restype = ctypes.c_float
        lib.oracle_hash_value.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64]
        lib.oracle_hash_init.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, f32p]
        lib.oracle_step_rows.argtypes = [vp, ctypes.c_int32, f32p, f32p, ctypes.c_int64, ctypes.c_int64]
        lib.oracle_embed.argtypes = [vp, ctypes.c_int32, ctypes.c_uint64, ctypes.c_int32, f32p, f32p]
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_chunk_of_edge.restype = ctypes.c_int32
        lib.oracle_chunk_of_edge.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32]
        lib.oracle_chunk_assign.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, i32p]
        lib.oracle_merge.argtypes = [ctypes.POINTER(f32p), i64p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, f32p]
        _lib = lib
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(t))


@dataclass
class Csr:
    """The oracle's M in CSR (original node labelling).  ``e`` is e_ab in fp64."""
    n: int
    nnz: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    e: np.ndarray
    deg: np.ndarray
    _h: ctypes.c_void_p = None

    def __del__(self):
        if self._h is not None and _lib is not None:
            _lib.oracle_csr_free(self._h)
            self._h = None


def build_csr(src, dst, w, n: int, directed: bool) -> Csr:
    """M = D^-1 A per readings B1-B4.  Raises OracleError(EDATA) on bad input."""
    src = np.ascontiguousarray(src, np.int32)
    dst = np.ascontiguousarray(dst, np.int32)
    if w is not None:
        w = np.ascontiguousarray(w, np.float32)
    h = ctypes.c_void_p()
    rc = _L().oracle_build(_p(src, ctypes.c_int32), _p(dst, ctypes.c_int32), _p(w, ctypes.c_float),
                           int(src.shape[0]), int(n), int(bool(directed)), ctypes.byref(h))
    if rc != OK:
        raise OracleError(rc, "build")
    nnz = int(_lib.oracle_csr_nnz(h))
    rp = np.empty(n + 1, np.int64); col = np.empty(nnz, np.int32); val = np.empty(nnz, np.float32)
    e = np.empty(nnz, np.float64); deg = np.empty(n, np.float64)
    _lib.oracle_csr_copy(h, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), _p(val, ctypes.c_float),
                         _p(e, ctypes.c_double), _p(deg, ctypes.c_double))
    return Csr(n, nnz, rp, col, val, e, deg, h)


def build_from(g) -> Csr:
    """build_csr for a ``gen.EdgeList``."""
    return build_csr(g.src, g.dst, g.w, g.n, g.directed)


def hash_value(seed: int, v: int, j: int) -> float:
    return float(_L().oracle_hash_value(seed, v, j))


def hash_init(n: int, d: int, seed: int, row_begin: int = 0) -> np.ndarray:
    """T_0 rows [row_begin, row_begin+n) (reading I1)."""
    out = np.empty((n, d), np.float32)
    _L().oracle_hash_init(seed, row_begin, row_begin + n, d, _p(out, ctypes.c_float))
    return out


def step(M: Csr, T_in: np.ndarray, r0: int = 0, r1: int | None = None) -> np.ndarray:
    """Rows [r0, r1) of normalize_rows(M . T_in) (Alg. 1 lines 6-7)."""
    r1 = M.n if r1 is None else r1
    T_in = np.ascontiguousarray(T_in, np.float32)
    assert T_in.shape[0] == M.n
    d = T_in.shape[1]
    out = np.empty((r1 - r0, d), np.float32)
    _L().oracle_step_rows(M._h, d, _p(T_in, ctypes.c_float), _p(out, ctypes.c_float), r0, r1)
    return out


def embed(M: Csr, d: int, seed: int, iters: int, keep_all: bool = False):
    """Algorithm 1 with Q = 1: T_iters (or the list [T_0 .. T_iters] when keep_all)."""
    T = hash_init(M.n, d, seed)
    if keep_all:
        out = [T]
        for _ in range(iters):
            T = step(M, T)
            out.append(T)
        return out
    for _ in range(iters):
        T = step(M, T)
    return T


def num_threads() -> int:
    return int(_L().oracle_num_threads())


# ---------------------------------------------------------------- f1: chunks (Algorithm 1, Q > 1)

def chunk_of_edge(chunk_seed: int, i: int, Q: int) -> int:
    return int(_L().oracle_chunk_of_edge(chunk_seed & 0xFFFFFFFFFFFFFFFF, int(i), int(Q)))


def chunk_assign(n_edges: int, Q: int, chunk_seed: int) -> np.ndarray:
    """Chunk index of every input edge (reading R13)."""
    out = np.empty(n_edges, np.int32)
    _L().oracle_chunk_assign(chunk_seed & 0xFFFFFFFFFFFFFFFF, int(n_edges), int(Q), _p(out, ctypes.c_int32))
    return out


def chunk_occurrences(src, dst, chunk, Q: int, n: int) -> np.ndarray:
    """occ[q, v] = occurrences of v as an endpoint of the edges of chunk q (reading R14)."""
    occ = np.zeros((Q, n), np.int64)
    np.add.at(occ, (chunk, src), 1)
    np.add.at(occ, (chunk, dst), 1)
    return occ


def merge(Tq: list, occ: np.ndarray) -> np.ndarray:
    """T_v = sum_q w_qv T^q_v (Algorithm 1 lines 10-12)."""
    Q, n = occ.shape
    d = Tq[0].shape[1]
    Tq = [np.ascontiguousarray(t, np.float32) for t in Tq]
    ptrs = (ctypes.POINTER(ctypes.c_float) * Q)(*[_p(t, ctypes.c_float) for t in Tq])
    occ = np.ascontiguousarray(occ, np.int64)
    out = np.empty((n, d), np.float32)
    _L().oracle_merge(ptrs, _p(occ, ctypes.c_int64), Q, n, d, _p(out, ctypes.c_float))
    return out


def embed_chunked(src, dst, w, n: int, directed: bool, Q: int, chunk_seed: int, d: int, seed: int, iters: int,
                  return_parts: bool = False):
    """Algorithm 1 with Q chunks: split the edges (R13), embed every chunk
    independently (its own M_q, T_0^q from the same id-keyed init, I steps), merge (R14)."""
    src = np.ascontiguousarray(src, np.int32)
    dst = np.ascontiguousarray(dst, np.int32)
    chunk = chunk_assign(src.shape[0], Q, chunk_seed)
    parts = []
    for q in range(Q):
        m = chunk == q
        if not m.any():
            parts.append(np.zeros((n, d), np.float32))     # an empty chunk: every row zero
            continue
        Mq = build_csr(src[m], dst[m], None if w is None else np.asarray(w)[m], n, directed)
        parts.append(embed(Mq, d, seed, iters))
    occ = chunk_occurrences(src, dst, chunk, Q, n)
    T = merge(parts, occ)
    return (T, parts, occ, chunk) if return_parts else T


# ---------------------------------------------------------------- f2: inductive embedding

def reconstruct(new_idx, known_idx, w, n_new: int, T_src: np.ndarray) -> np.ndarray:
    """Embeddings of n_new unseen nodes from edges (new node i, known node b, weight): row i =
    normalize(sum_b e_ib / sum e_i. * T_src[b]) -- "creation of new node embedding by weighted
    averaging of all neighbors' representations", the transition-row multiply the
    training loop performs; T_src should be T_{I-1}.  Built as
    one step of normalize(M T) over the directed graph new -> known (readings B1-B4, R6, RZ)."""
    T_src = np.ascontiguousarray(T_src, np.float32)
    n_src, d = T_src.shape
    n = max(n_new, n_src)
    M = build_csr(new_idx, known_idx, w, n, True)
    T_in = T_src if n == n_src else np.vstack([T_src, np.zeros((n - n_src, d), np.float32)])
    return step(M, T_in, 0, n_new)


# ---------------------------------------------------------------- f3: hypergraph expansion

def expand_clique(he_ptr, he_nodes, he_weight=None):
    """Clique expansion ("each hyperedge is transformed into a clique"), reading R16:
    hyperedge e with members m_0..m_{k-1} gives (m_i, m_j) for i < j, m_i != m_j, in the order
    (e, i, j), each with the hyperedge's weight.  Plain loops: small inputs only."""
    src, dst, w = [], [], []
    for e in range(len(he_ptr) - 1):
        m = [int(x) for x in he_nodes[he_ptr[e]:he_ptr[e + 1]]]
        we = 1.0 if he_weight is None else float(he_weight[e])
        for i in range(len(m)):
            for j in range(i + 1, len(m)):
                if m[i] != m[j]:
                    src.append(m[i])
                    dst.append(m[j])
                    w.append(we)
    return np.array(src, np.int32), np.array(dst, np.int32), np.array(w, np.float32)


def expand_star(he_ptr, he_nodes, n_nodes: int, he_weight=None):
    """Star expansion ("an extra node is introduced which links to the original
    nodes contained by a hyperedge"), reading R17: hyperedge e gets node n_nodes + e and the edges
    (n_nodes + e, m_i) for every listed member, in the order (e, i)."""
    he_ptr = np.asarray(he_ptr, np.int64)
    k = np.diff(he_ptr)
    src = (n_nodes + np.repeat(np.arange(len(k), dtype=np.int64), k)).astype(np.int32)
    dst = np.asarray(he_nodes, np.int32)[:he_ptr[-1]].copy()
    w = np.ones(len(dst), np.float32) if he_weight is None else np.repeat(np.asarray(he_weight, np.float32), k)
    return src, dst, w
