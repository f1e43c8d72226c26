"""Dense numpy brute force used to PIN the oracle (tests only).

It is the textbook formulation, independent of oracle/: an explicit |V| x |V|
matrix A with A[a,b] = e_ab, D = diag(row sums), M = D^-1 A as a
dense fp64 matrix, and T_i = normalize_rows(M @ T_{i-1}) with numpy's matmul and
numpy.linalg.norm (Alg. 1 lines 6-7).  Small graphs only.
"""
import numpy as np


def dense_A(src, dst, w, n, directed):
    A = np.zeros((n, n), np.float64)
    ww = np.ones(len(src)) if w is None else np.asarray(w, np.float64)
    for u, v, x in zip(src, dst, ww):
        A[u, v] += x
        if not directed and u != v:
            A[v, u] += x
    return A


def dense_M(A):
    deg = A.sum(axis=1)
    M = np.zeros_like(A)
    nz = deg > 0
    M[nz] = A[nz] / deg[nz, None]
    return M, deg


def normalize_rows(Y):
    nrm = np.linalg.norm(Y, axis=1)
    out = np.zeros_like(Y)
    nz = nrm > 0
    out[nz] = Y[nz] / nrm[nz, None]
    return out


def dense_embed(M, T0, iters, store_fp32=True, return_cond=False):
    """Iterate; with return_cond also return, per iteration, the smallest non-zero
    pre-normalisation row norm (normalising a near-zero vector is ill-conditioned:
    any rounding flips its direction, so comparisons past such a step are meaningless)."""
    T = np.asarray(T0, np.float64)
    outs = [T.copy()]
    cond = [np.inf]
    for _ in range(iters):
        Y = M @ T
        nr = np.linalg.norm(Y, axis=1)
        live = ((M != 0) & (np.linalg.norm(T, axis=1) > 0)[None, :]).any(axis=1)
        cond.append(nr[live].min() if live.any() else np.inf)
        T = normalize_rows(Y)
        if store_fp32:
            T = T.astype(np.float32).astype(np.float64)
        outs.append(T.copy())
    return (outs, cond) if return_cond else outs
