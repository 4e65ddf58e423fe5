"""Build libgicp_b200.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgicp_b200.so")
SOURCES = ["api.cu", "index.cu", "knn.cu", "cov.cu", "linearize.cu", "prep.cu", "vgicp.cu", "ground.cu", "cluster.cu", "submap.cu", "shard.cu"]
HEADERS = ["gicp_internal.cuh", "cov_device.cuh", "lin_device.cuh", "sortnet.cuh", "knn_tile.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "--extended-lambda",
    # IEEE fp32: no fast math, no flush-to-zero; the spec'd d2 uses __fmaf_rn etc.
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-Xcompiler", "-ffp-contract=off",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "gicp.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra=(), out: str | None = None) -> str:
    """Compile every .cu to an object in parallel (no cross-file device code: no
    -rdc), then link the shared library."""
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    with tempfile.TemporaryDirectory(prefix="gicp_build_") as tmp:
        def compile_one(f):
            obj = os.path.join(tmp, f.replace(".cu", ".o"))
            cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", "-o", obj, os.path.join(CSRC, f)]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
            return obj
        with ThreadPoolExecutor(max_workers=min(len(SOURCES), max(1, os.cpu_count() or 1))) as ex:
            objs = list(ex.map(compile_one, SOURCES))
        link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", target + ".tmp", *objs]
        if verbose:
            print(" ".join(link), file=sys.stderr)
        subprocess.run(link, check=True)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else [])
