"""B200-native Cleora hot path: Python binding of libcleora.so (include/cleora.h).

Argument marshalling only.  Every step of the path -- CSR build (sort, merge, degree,
D^-1 scaling), hash initialisation, the fused SpMM + row-L2-normalise iteration, the
multi-GPU exchange -- runs in the library's CUDA kernels.  There is no CPU fallback:
importing this package without the built ``libcleora.so`` raises ImportError, and every
call without a usable B200 raises :class:`CleoraError` (code 4).

The functions carry the C names (``cleora_build`` ... ``cleora_fetch``).  Arrays may be
numpy arrays (host) or torch tensors (host or CUDA; CUDA tensors are passed as device
pointers, so nothing is copied through the host).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = [
    "CleoraError", "Graph", "LIB_PATH",
    "cleora_build", "cleora_init", "cleora_iterate", "cleora_fetch", "cleora_info", "cleora_stats",
    "cleora_sync", "cleora_destroy", "cleora_last_error", "cleora_fetch_csr", "cleora_set_rows", "cleora_fetch_replica",
    "cleora_fetch_async", "cleora_trim", "cleora_fetch_nonzero", "cleora_fetch_nonzero_async", "cleora_nonzero_count",
    "cleora_nccl_id_size", "cleora_nccl_get_unique_id", "cleora_plan_shards", "cleora_kernel_launches",
    "cleora_release_cached_memory", "cleora_merge_chunks", "cleora_reconstruct", "cleora_build_batch",
    "cleora_expand", "EXPAND_CLIQUE", "EXPAND_STAR", "cleora_probe_gather", "cleora_ipc_opens", "cleora_oom_fallbacks", "host_allgather_from",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcleora.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built (run `python -c 'import __graft_entry__ as g; g.build()'`); "
                      "the Cleora path has no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

OK, EUSAGE, EDATA, EINTERNAL = 0, 2, 3, 4
F_TIMING, F_LOOPBACK, F_EXCHANGE_NCCL = 1, 2, 4


# int (*cleora_allgather_fn)(void* ctx, const void* send, void* recv, int64_t bytes)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)


class _Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("input_on_device", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("flags", ctypes.c_int32), ("n_chunks", ctypes.c_int32), ("chunk", ctypes.c_int32),
                ("chunk_seed", ctypes.c_uint64), ("host_allgather", ALLGATHER_FN), ("host_ctx", ctypes.c_void_p)]


def host_allgather_from(group=None):
    """A cleora_allgather_fn over a torch.distributed process group (e.g. gloo on CPU): for world > 1
    without NCCL -- several processes sharing one GPU in a test, or a box without NCCL.  Keep the
    returned object alive as long as the handles built with it (cleora_build keeps a reference)."""
    import torch
    import torch.distributed as dist

    def fn(ctx, send, recv, nbytes):
        try:
            n = int(nbytes)
            mine = torch.frombuffer(bytearray(ctypes.string_at(send, n)), dtype=torch.uint8) if n else \
                torch.empty(0, dtype=torch.uint8)
            world = dist.get_world_size(group)
            out = [torch.empty(n, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(out, mine, group=group)
            buf = b"".join(bytes(t.numpy().tobytes()) for t in out)
            ctypes.memmove(recv, buf, len(buf))
            return 0
        except Exception:                # never raise through the C library
            return 1

    return ALLGATHER_FN(fn)


class _Info(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("nnz", ctypes.c_int64), ("n_edges_in", ctypes.c_int64),
                ("d", ctypes.c_int32), ("d_stride", ctypes.c_int32), ("iterations", ctypes.c_int64),
                ("zero_rows", ctypes.c_int64), ("max_degree", ctypes.c_int64), ("heavy_rows", ctypes.c_int64),
                ("heavy_items", ctypes.c_int64), ("shard_begin", ctypes.c_int64), ("shard_end", ctypes.c_int64),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device_bytes", ctypes.c_int64),
                ("hot_rows", ctypes.c_int64), ("referenced_rows", ctypes.c_int64), ("exchange", ctypes.c_int32),
                ("n_graphs", ctypes.c_int32), ("shard_nnz", ctypes.c_int64), ("launches_per_step", ctypes.c_int32)]


class _Stats(ctypes.Structure):
    _fields_ = [("spmm_launches", ctypes.c_int64), ("spmm_ms_total", ctypes.c_double),
                ("spmm_ms_min", ctypes.c_double), ("spmm_ms_max", ctypes.c_double),
                ("exchange_launches", ctypes.c_int64), ("exchange_ms_total", ctypes.c_double)]


_vp, _i32, _i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_SIGS = {
    "cleora_build": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i32, _i32, ctypes.POINTER(_Opts), ctypes.POINTER(_vp)]),
    "cleora_init": (ctypes.c_int, [_vp, _i32, ctypes.c_uint64]),
    "cleora_expand": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i64,
                                     ctypes.POINTER(_i64)]),
    "cleora_build_batch": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, ctypes.POINTER(_Opts), ctypes.POINTER(_vp)]),
    "cleora_iterate": (ctypes.c_int, [_vp, _i32]),
    "cleora_fetch": (ctypes.c_int, [_vp, _i64, _i64, _vp, _i32]),
    "cleora_fetch_async": (ctypes.c_int, [_vp, _i64, _i64, _vp, _i32]),
    "cleora_fetch_nonzero_async": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _i32]),
    "cleora_fetch_nonzero": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _i32]),
    "cleora_info": (ctypes.c_int, [_vp, ctypes.POINTER(_Info)]),
    "cleora_stats": (ctypes.c_int, [_vp, ctypes.POINTER(_Stats), _i32]),
    "cleora_sync": (ctypes.c_int, [_vp]),
    "cleora_trim": (ctypes.c_int, [_vp]),
    "cleora_destroy": (None, [_vp]),
    "cleora_last_error": (ctypes.c_char_p, []),
    "cleora_fetch_csr": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "cleora_set_rows": (ctypes.c_int, [_vp, _i64, _i64, _vp]),
    "cleora_fetch_replica": (ctypes.c_int, [_vp, _i32, _i64, _i64, _vp]),
    "cleora_merge_chunks": (ctypes.c_int, [_vp, _i32, _vp, _i32]),
    "cleora_reconstruct": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _i32]),
    "cleora_nccl_id_size": (ctypes.c_int, []),
    "cleora_nccl_get_unique_id": (ctypes.c_int, [_vp]),
    "cleora_plan_shards": (ctypes.c_int, [_vp, _i64, _i32, _vp]),
    "cleora_kernel_launches": (ctypes.c_int64, []),
    "cleora_release_cached_memory": (ctypes.c_int, []),
    "cleora_probe_gather": (ctypes.c_int, [_i32, _i32, _i64, _i64, ctypes.POINTER(ctypes.c_double)]),
    "cleora_ipc_opens": (ctypes.c_int64, []),
    "cleora_oom_fallbacks": (ctypes.c_int64, []),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class CleoraError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[cleora error {code}] {msg}")
        self.code = code


def cleora_last_error() -> str:
    m = _lib.cleora_last_error()
    return m.decode() if m else ""


def _check(rc: int):
    if rc != OK:
        raise CleoraError(rc, cleora_last_error())


def _ptr(a, dtype):
    """(pointer, on_device, keepalive) for a numpy array or torch tensor (or None)."""
    if a is None:
        return None, False, None
    if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):       # torch.Tensor
        import torch
        tdt = {np.int32: torch.int32, np.float32: torch.float32, np.int64: torch.int64,
               np.float64: torch.float64}[dtype]
        if a.dtype != tdt or not a.is_contiguous():
            a = a.to(tdt).contiguous()
        return a.data_ptr(), bool(a.is_cuda), a
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data, False, arr


def _torch_stream(device) -> int:
    """cudaStream_t of torch's current stream on `device` (an index or torch.device).  torch's default
    stream is the legacy NULL stream; it is passed as cudaStreamLegacy (0x1), because a NULL
    cleora_opts.stream means "a library-owned non-blocking stream", which would not be ordered."""
    import torch
    return int(torch.cuda.current_stream(device).cuda_stream) or 1


def _order_after_torch(tensors, lib_stream):
    """CUDA tensors handed to a call that runs on another stream than torch's current one: wait for
    torch's pending work on them first (a tensor just written by a torch kernel, or a block the
    caching allocator recycled while older kernels may still use it).  No-op for host arrays."""
    for t in tensors:
        if t is not None and getattr(t, "is_cuda", False):
            import torch
            cur = torch.cuda.current_stream(t.device)
            if lib_stream is None or (int(cur.cuda_stream) or 1) != int(lib_stream):
                cur.synchronize()
            return


class Graph:
    """Owning wrapper of a ``cleora_graph*`` (destroyed on close / garbage collection).  ``stream``
    is the cudaStream_t the handle enqueues on (None: a library-owned stream)."""

    def __init__(self, handle: int, stream: int | None = None, keep=None):
        self._h = handle
        self.stream = stream
        self._keep = keep            # objects the C handle points to (a host all-gather callback)

    @property
    def handle(self) -> int:
        if not self._h:
            raise CleoraError(EUSAGE, "graph already destroyed")
        return self._h

    def close(self):
        if self._h:
            _lib.cleora_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # convenience methods with the C semantics
    def init(self, d: int, seed: int = 0):
        cleora_init(self, d, seed)
        return self

    def iterate(self, k: int):
        cleora_iterate(self, k)
        return self

    def fetch(self, row_begin: int = 0, row_end: int | None = None, out=None):
        return cleora_fetch(self, row_begin, row_end, out)

    def info(self) -> dict:
        return cleora_info(self)


def cleora_build(src, dst, weight, n_nodes: int, directed: bool = False, *, device: int = -1, stream=None,
                 rank: int = 0, world: int = 1, nccl_id: bytes | None = None, timing: bool = False,
                 loopback: bool = False, exchange_nccl: bool = False, n_chunks: int = 0, chunk: int = 0,
                 chunk_seed: int = 0, host_allgather=None) -> Graph:
    """COO edge list -> device CSR of M = D^-1 A.  See include/cleora.h.
    world > 1: row-sharded, collectives over NCCL (nccl_id) or ``host_allgather`` (an ALLGATHER_FN,
    e.g. host_allgather_from(group))."""
    ps, ds, ks = _ptr(src, np.int32)
    pd, dd, kd = _ptr(dst, np.int32)
    pw, dw, kw = _ptr(weight, np.float32)
    if ps is None or pd is None:
        raise CleoraError(EUSAGE, "src/dst required")
    n = int(ks.shape[0])
    if int(kd.shape[0]) != n or (kw is not None and int(kw.shape[0]) != n):
        raise CleoraError(EUSAGE, "src, dst, weight must have the same length")
    on_dev = ds or dd or dw
    if on_dev and not (ds and dd and (kw is None or dw)):
        raise CleoraError(EUSAGE, "src/dst/weight must be all on the host or all on the device")
    if on_dev and device < 0:
        device = int(ks.device.index or 0)
    if stream is None and on_dev:
        # device inputs: enqueue on torch's current stream, so the build is ordered after the
        # kernels that produced them (and torch's later work after the build)
        stream = _torch_stream(ks.device)
    o = _Opts()
    o.device = device
    o.input_on_device = 1 if on_dev else 0
    if stream is not None:
        o.stream = stream if isinstance(stream, int) else int(getattr(stream, "cuda_stream", stream))
    o.rank, o.world = rank, world
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), len(nccl_id))
        o.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
    o.flags = (F_TIMING if timing else 0) | (F_LOOPBACK if loopback else 0) | \
        (F_EXCHANGE_NCCL if exchange_nccl else 0)
    o.n_chunks, o.chunk, o.chunk_seed = int(n_chunks), int(chunk), int(chunk_seed) & 0xFFFFFFFFFFFFFFFF
    if host_allgather is not None:
        o.host_allgather = host_allgather
    h = ctypes.c_void_p()
    _check(_lib.cleora_build(ps, pd, pw, n, int(n_nodes), 1 if directed else 0, ctypes.byref(o), ctypes.byref(h)))
    return Graph(h.value, o.stream, keep=host_allgather)


EXPAND_CLIQUE, EXPAND_STAR = 0, 1


def cleora_expand(he_ptr, he_nodes, n_nodes: int, mode: int, he_weight=None, *, device: int = -1, stream=None,
                  with_weight: bool = False):
    """Hypergraph -> undirected edge list on the device (clique or star expansion).
    Host arrays in -> numpy (src, dst[, w]) out; CUDA tensors in -> CUDA tensors out."""
    pp, dp_, kp = _ptr(he_ptr, np.int64)
    pn, dn, kn = _ptr(he_nodes, np.int32)
    pw, dw, kw = _ptr(he_weight, np.float32)
    on_dev = dp_ or dn or dw
    if on_dev and not (dp_ and dn and (kw is None or dw)):
        raise CleoraError(EUSAGE, "inputs must be all on the host or all on the device")
    n_he = int(kp.shape[0]) - 1
    if stream is None and on_dev:
        stream = _torch_stream(kp.device)        # ordered after the kernels that produced the inputs
    st = 0 if stream is None else (stream if isinstance(stream, int) else int(getattr(stream, "cuda_stream", stream)))
    if on_dev and device < 0:
        device = int(kp.device.index or 0)
    n = ctypes.c_int64()
    _check(_lib.cleora_expand(pp, pn, pw, n_he, int(n_nodes), int(mode), int(device), 1 if on_dev else 0, st,
                              None, None, None, 0, ctypes.byref(n)))
    m = int(n.value)
    want_w = with_weight or he_weight is not None
    if on_dev:
        import torch
        os_ = torch.empty(m, dtype=torch.int32, device=kp.device)
        od_ = torch.empty(m, dtype=torch.int32, device=kp.device)
        ow_ = torch.empty(m, dtype=torch.float32, device=kp.device) if want_w else None
        ptrs = (os_.data_ptr(), od_.data_ptr(), ow_.data_ptr() if want_w else None)
    else:
        os_, od_ = np.empty(m, np.int32), np.empty(m, np.int32)
        ow_ = np.empty(m, np.float32) if want_w else None
        ptrs = (os_.ctypes.data, od_.ctypes.data, ow_.ctypes.data if want_w else None)
    if m > 0:
        _check(_lib.cleora_expand(pp, pn, pw, n_he, int(n_nodes), int(mode), int(device), 1 if on_dev else 0, st,
                                  ptrs[0], ptrs[1], ptrs[2], m, ctypes.byref(n)))
    return (os_, od_, ow_) if want_w else (os_, od_)


def cleora_build_batch(src, dst, weight, edge_ptr, node_count, directed: bool = False, *, device: int = -1,
                       stream=None, timing: bool = False) -> Graph:
    """Several independent graphs in one handle (block-diagonal M, one launch per step; SURVEY
    §8(f) f4).  Graph g: edges [edge_ptr[g], edge_ptr[g+1]) with LOCAL ids; its rows are
    [sum(node_count[:g]), +node_count[g]).  See include/cleora.h."""
    ps, ds, ks = _ptr(src, np.int32)
    pd, dd, kd = _ptr(dst, np.int32)
    pw, dw, kw = _ptr(weight, np.float32)
    ep = np.ascontiguousarray(edge_ptr, np.int64)
    nc = np.ascontiguousarray(node_count, np.int32)
    if ps is None or pd is None:
        raise CleoraError(EUSAGE, "src/dst required")
    n = int(ks.shape[0])
    if int(kd.shape[0]) != n or (kw is not None and int(kw.shape[0]) != n) or int(ep[-1]) != n:
        raise CleoraError(EUSAGE, "src, dst, weight and edge_ptr[-1] must agree")
    on_dev = ds or dd or dw
    if on_dev and not (ds and dd and (kw is None or dw)):
        raise CleoraError(EUSAGE, "src/dst/weight must be all on the host or all on the device")
    if on_dev and device < 0:
        device = int(ks.device.index or 0)
    if stream is None and on_dev:
        stream = _torch_stream(ks.device)
    o = _Opts()
    o.device = device
    o.input_on_device = 1 if on_dev else 0
    if stream is not None:
        o.stream = stream if isinstance(stream, int) else int(getattr(stream, "cuda_stream", stream))
    o.world = 1
    o.flags = F_TIMING if timing else 0
    h = ctypes.c_void_p()
    _check(_lib.cleora_build_batch(ps, pd, pw, ep.ctypes.data, nc.ctypes.data, int(nc.shape[0]), 1 if directed else 0,
                                   ctypes.byref(o), ctypes.byref(h)))
    return Graph(h.value, o.stream)


def cleora_init(g: Graph, d: int, seed: int = 0):
    _check(_lib.cleora_init(g.handle, int(d), int(seed) & 0xFFFFFFFFFFFFFFFF))


def cleora_iterate(g: Graph, k: int):
    _check(_lib.cleora_iterate(g.handle, int(k)))


def cleora_fetch(g: Graph, row_begin: int = 0, row_end: int | None = None, out=None):
    """Rows [row_begin, row_end) of the current T as a (rows, d) fp32 array.  ``out`` may be a
    preallocated numpy array / host tensor (pinned for speed) or a CUDA tensor."""
    info = cleora_info(g, sync=False)
    if row_end is None:
        row_end = info["n_nodes"]
    rows = max(0, row_end - row_begin)
    if out is None:
        out = np.empty((rows, info["d"]), np.float32)
    p, on_dev, keep = _ptr(out, np.float32)
    if keep is not out:
        raise CleoraError(EUSAGE, "out must be a contiguous fp32 array")
    _order_after_torch([out], g.stream)
    _check(_lib.cleora_fetch(g.handle, int(row_begin), int(row_end), p, 1 if on_dev else 0))
    return out


def cleora_fetch_async(g: Graph, row_begin: int, row_end: int, out):
    """Enqueue the copy of rows [row_begin, row_end) into `out` (a preallocated pinned host or CUDA
    tensor / array) on the library's copy stream; returns at once.  Keep `out` alive until
    cleora_sync(g) or g.close()."""
    p, on_dev, keep = _ptr(out, np.float32)
    if keep is not out:
        raise CleoraError(EUSAGE, "out must be a contiguous fp32 array")
    _order_after_torch([out], None)
    _check(_lib.cleora_fetch_async(g.handle, int(row_begin), int(row_end), p, 1 if on_dev else 0))
    return out


def _fetch_nonzero(fn, g, out_rows, out_ids, sync):
    n = ctypes.c_int64(0)
    _check(fn(g.handle, None, None, 0, ctypes.byref(n), 0))
    rows = n.value
    if out_rows is None and out_ids is None:
        d = cleora_info(g, sync=False)["d"]
        out_rows = np.empty((rows, d), np.float32)
        out_ids = np.empty(rows, np.int32)
    pr, dev_r, kr = _ptr(out_rows, np.float32)
    pi, dev_i, ki = _ptr(out_ids, np.int32)
    if (out_rows is not None and kr is not out_rows) or (out_ids is not None and ki is not out_ids):
        raise CleoraError(EUSAGE, "out_rows / out_ids must be contiguous fp32 / int32 arrays")
    if out_rows is not None and out_ids is not None and dev_r != dev_i:
        raise CleoraError(EUSAGE, "out_rows and out_ids must both be host or both be device memory")
    cap = min(len(out_rows) if out_rows is not None else rows, len(out_ids) if out_ids is not None else rows)
    _order_after_torch([out_rows, out_ids], None)
    _check(fn(g.handle, pr, pi, int(cap), ctypes.byref(n), 1 if (dev_r or dev_i) else 0))
    k = n.value
    return (out_rows[:k] if out_rows is not None else None), (out_ids[:k] if out_ids is not None else None)


def cleora_fetch_nonzero(g: Graph, out_rows=None, out_ids=None):
    """(rows, ids): the rows of this handle's shard with entries in M (ascending ids) and their rows of
    the current T; every other row is exactly 0 (see include/cleora.h).  Outputs are allocated as numpy
    arrays when both are None, else written into the given host / CUDA arrays (views of the first n
    rows are returned)."""
    return _fetch_nonzero(_lib.cleora_fetch_nonzero, g, out_rows, out_ids, True)


def cleora_fetch_nonzero_async(g: Graph, out_rows, out_ids):
    """Enqueue cleora_fetch_nonzero into preallocated outputs (pinned host or CUDA); returns the views
    at once.  Keep the outputs alive until cleora_sync(g) or g.close()."""
    return _fetch_nonzero(_lib.cleora_fetch_nonzero_async, g, out_rows, out_ids, False)


def cleora_nonzero_count(g: Graph) -> int:
    """Rows cleora_fetch_nonzero would return now."""
    n = ctypes.c_int64(0)
    _check(_lib.cleora_fetch_nonzero(g.handle, None, None, 0, ctypes.byref(n), 0))
    return n.value


def cleora_info(g: Graph, sync: bool = True) -> dict:
    i = _Info()
    _check(_lib.cleora_info(g.handle, ctypes.byref(i)))
    return {f: getattr(i, f) for f, _ in _Info._fields_}


def cleora_stats(g: Graph, reset: bool = False) -> dict:
    s = _Stats()
    _check(_lib.cleora_stats(g.handle, ctypes.byref(s), 1 if reset else 0))
    return {f: getattr(s, f) for f, _ in _Stats._fields_}


def cleora_sync(g: Graph):
    _check(_lib.cleora_sync(g.handle))


def cleora_trim(g: Graph):
    """Keep only the current embedding on the device (see include/cleora.h): afterwards the
    handle can still be fetched (also asynchronously), merged, queried and closed."""
    _check(_lib.cleora_trim(g.handle))


def cleora_destroy(g: Graph):
    g.close()


def cleora_fetch_csr(g: Graph) -> dict:
    """This rank's rows of M (the whole M on one GPU; see include/cleora.h for shards)."""
    info = cleora_info(g)
    n, nnz = info["n_nodes"], info["shard_nnz"]
    rp = np.empty(n + 1, np.int64); col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float32); deg = np.empty(n, np.float64)
    _check(_lib.cleora_fetch_csr(g.handle, rp.ctypes.data, col.ctypes.data, val.ctypes.data, deg.ctypes.data))
    return dict(row_ptr=rp, col=col, val=val, deg=deg)


def cleora_fetch_replica(g: Graph, rank: int, row_begin: int = 0, row_end: int | None = None) -> np.ndarray:
    """Rows of rank ``rank``'s replica (every replica is local with ``loopback=True``)."""
    info = cleora_info(g)
    if row_end is None:
        row_end = info["n_nodes"]
    out = np.empty((max(0, row_end - row_begin), info["d"]), np.float32)
    _check(_lib.cleora_fetch_replica(g.handle, int(rank), int(row_begin), int(row_end), out.ctypes.data))
    return out


def cleora_merge_chunks(chunks, out=None):
    """Algorithm 1 lines 10-12: the occurrence-weighted average of the chunks' current T
    (handles built with n_chunks / chunk / chunk_seed).  Returns an N x d fp32 array (or `out`)."""
    chunks = list(chunks)
    info = cleora_info(chunks[0])
    if out is None:
        out = np.empty((info["n_nodes"], info["d"]), np.float32)
    p, on_dev, keep = _ptr(out, np.float32)
    if keep is not out:
        raise CleoraError(EUSAGE, "out must be a contiguous fp32 array")
    _order_after_torch([out], chunks[0].stream)
    arr = (ctypes.c_void_p * len(chunks))(*[c.handle for c in chunks])
    _check(_lib.cleora_merge_chunks(ctypes.cast(arr, ctypes.c_void_p), len(chunks), p, 1 if on_dev else 0))
    return out


def cleora_reconstruct(g: Graph, new_idx, known_idx, weight, n_new: int, out=None):
    """Embeddings of n_new unseen nodes from edges (new_idx[i] -> known_idx[i], weight) against
    g's current T (use T_{I-1}).  Returns an n_new x d fp32 array (or `out`)."""
    pn, dn, kn = _ptr(new_idx, np.int32)
    pk, dk, kk = _ptr(known_idx, np.int32)
    pw, dw, kw = _ptr(weight, np.float32)
    if pn is None or pk is None:
        raise CleoraError(EUSAGE, "new_idx/known_idx required")
    n_e = int(kn.shape[0])
    if int(kk.shape[0]) != n_e or (kw is not None and int(kw.shape[0]) != n_e):
        raise CleoraError(EUSAGE, "new_idx, known_idx, weight must have the same length")
    on_dev = dn or dk or dw
    if on_dev and not (dn and dk and (kw is None or dw)):
        raise CleoraError(EUSAGE, "inputs must be all on the host or all on the device")
    info = cleora_info(g)
    if out is None:
        out = np.empty((int(n_new), info["d"]), np.float32)
    po, od, ko = _ptr(out, np.float32)
    if ko is not out:
        raise CleoraError(EUSAGE, "out must be a contiguous fp32 array")
    _order_after_torch([kn, kk, kw, out], g.stream)
    _check(_lib.cleora_reconstruct(g.handle, pn, pk, pw, n_e, int(n_new), 1 if on_dev else 0, po, 1 if od else 0))
    return out


def cleora_set_rows(g: Graph, row_begin: int, rows):
    arr = np.ascontiguousarray(rows, np.float32)
    _check(_lib.cleora_set_rows(g.handle, int(row_begin), int(row_begin) + int(arr.shape[0]), arr.ctypes.data))


def cleora_nccl_id_size() -> int:
    return int(_lib.cleora_nccl_id_size())


def cleora_nccl_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(cleora_nccl_id_size())
    _check(_lib.cleora_nccl_get_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def cleora_plan_shards(row_ptr, world: int) -> np.ndarray:
    """Host-side nnz-balanced contiguous row cuts (no GPU needed)."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cuts = np.empty(world + 1, np.int64)
    _check(_lib.cleora_plan_shards(rp.ctypes.data, int(rp.shape[0] - 1), int(world), cuts.ctypes.data))
    return cuts


def cleora_kernel_launches() -> int:
    """Process-wide count of kernels libcleora has launched (its own + CUB's)."""
    return int(_lib.cleora_kernel_launches())


def cleora_release_cached_memory():
    """Return the library's cached device blocks (freed T replicas, CSR, sort buffers) to the driver."""
    _check(_lib.cleora_release_cached_memory())


def cleora_probe_gather(row_bytes: int, table_bytes: int = 64 << 20, n_gathers: int = 1 << 22, device: int = -1) -> float:
    """Random-row gather rate (GB/s) from an L2-resident table (diagnostic; see include/cleora.h)."""
    r = ctypes.c_double()
    _check(_lib.cleora_probe_gather(int(device), int(row_bytes), int(table_bytes), int(n_gathers), ctypes.byref(r)))
    return float(r.value)


def cleora_ipc_opens() -> int:
    """Process-wide count of CUDA IPC mappings opened (peer T buffers; cached across handles)."""
    return int(_lib.cleora_ipc_opens())


def cleora_oom_fallbacks() -> int:
    """Process-wide count of allocations that had to return cached segments to the driver first."""
    return int(_lib.cleora_oom_fallbacks())
