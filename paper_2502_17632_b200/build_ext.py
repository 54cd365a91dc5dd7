"""Compile the CUDA library libgiftb200.so in-tree for sm_100a (nvcc).

Run `python -m paper_2502_17632_b200.build_ext` or call `build()`; the
__graft_entry__.build() hook does the same.  Rebuilds only when a source is
newer than the library.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libgiftb200.so")
SOURCES = ["csrc/abi.cu", "csrc/build.cu", "csrc/filter.cu", "csrc/bmt.cu", "csrc/metrics.cu", "csrc/plio.cu", "csrc/bookshelf.cu", "csrc/shard.cu", "csrc/hf.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xcompiler", "-Wno-deprecated-declarations",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(HERE, s) for s in SOURCES]
    deps += glob.glob(os.path.join(HERE, "csrc", "*.cuh"))
    deps.append(os.path.join(ROOT, "include", "gift_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", LIB + ".tmp", *[os.path.join(HERE, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
