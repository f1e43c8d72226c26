"""C-ABI checks that need no GPU: the library loads, exports every symbol include/cleora.h
declares, host-side shard planning, and the loud failure without a device."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "cleora.h")).read()
    return sorted(set(re.findall(r"CLEORA_API\s+[\w\s\*]+?\b(cleora_\w+)\s*\(", txt)))


def test_header_declares_the_path_calls():
    names = header_functions()
    for must in ("cleora_build", "cleora_init", "cleora_iterate", "cleora_fetch", "cleora_destroy",
                 "cleora_last_error", "cleora_info"):
        assert must in names


def test_library_exports_every_header_symbol():
    import ctypes
    import paper_2102_02302_b200 as cl
    lib = ctypes.CDLL(cl.LIB_PATH)
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding exposes the same names
    for n in header_functions():
        assert hasattr(cl, n), n


def test_library_is_sm100a():
    import subprocess
    import paper_2102_02302_b200 as cl
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", cl.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2102_02302_b200 as cl
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_build(np.array([0], np.int32), np.array([1], np.int32), None, 2)
    assert e.value.code == cl.EINTERNAL and "no CUDA device" in str(e.value)


def test_usage_errors_are_host_side():
    import paper_2102_02302_b200 as cl
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_build(np.array([], np.int32), np.array([], np.int32), None, 2)
    assert e.value.code == cl.EUSAGE
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_build(np.array([0], np.int32), np.array([1], np.int32), None, 2, world=2, rank=0)
    assert e.value.code == cl.EUSAGE and "nccl_id" in str(e.value)
    one = np.array([0], np.int32)
    for ep, nc, why in (([0, 1], [0], "node_count"), ([1, 1], [2], "edge_ptr[0]"), ([0, 2, 1], [2, 2], "non-decreasing")):
        with pytest.raises(cl.CleoraError) as e:
            cl.cleora_build_batch(one, one, None, np.array(ep, np.int64), np.array(nc, np.int32))
        assert e.value.code == cl.EUSAGE and why in str(e.value), why
    with pytest.raises(cl.CleoraError) as e:
        cl.cleora_build(one, one, None, 2, n_chunks=2, chunk=3)
    assert e.value.code == cl.EUSAGE and "chunk" in str(e.value)


def test_plan_shards_balances_nnz():
    import gen
    import oracle
    import paper_2102_02302_b200 as cl
    g = gen.config("c1")
    M = oracle.build_from(g)
    for world in (1, 2, 3, 4, 8):
        cuts = cl.cleora_plan_shards(M.row_ptr, world)
        assert cuts[0] == 0 and cuts[-1] == g.n and np.all(np.diff(cuts) >= 0)
        per = np.diff(M.row_ptr[cuts])
        assert per.sum() == M.nnz
        assert per.max() - per.min() <= 2 * np.diff(M.row_ptr).max() + 1
        # cut p is the first row whose nnz prefix reaches p * nnz / world
        for p in range(1, world):
            r = cuts[p]
            assert M.row_ptr[r] * world >= p * M.nnz
            assert r == 0 or M.row_ptr[r - 1] * world < p * M.nnz
