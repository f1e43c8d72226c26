"""Compile libcleora.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libcleora.so")
SOURCES = ["api.cu", "build.cu", "chunks.cu", "expand.cu", "fetch.cu", "init.cu", "probe.cu", "spmm_norm.cu", "spmm_tma.cu"]
HEADERS = ["common.cuh", "spmm_common.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared", "-cudart", "static",
    # IEEE division / sqrt everywhere: the CSR build must be bit-exact (B4)
    "-prec-div=true", "-prec-sqrt=true", "-fmad=true",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "cleora.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """One object per translation unit, compiled in parallel, then one shared-library link."""
    if not force and not _stale():
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    tmp = LIB + f".tmp{os.getpid()}"
    extra = os.environ.get("CLEORA_NVCC_EXTRA", "").split()   # measurement builds (-D switches)
    compile_flags = [f for f in FLAGS if f not in ("-shared", "-cudart", "static")]
    with tempfile.TemporaryDirectory(prefix="cleora_build_") as td:
        def one(src):
            obj = os.path.join(td, src.replace(".cu", ".o"))
            cmd = [NVCC, *compile_flags, *extra, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj,
                   os.path.join(CSRC, src)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd, cwd=CSRC)
            return obj
        with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
            objs = list(ex.map(one, SOURCES))
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                               "-o", tmp, *objs, "-ldl"], cwd=CSRC)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
