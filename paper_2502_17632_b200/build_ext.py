"""Compile the CUDA library libgiftb200.so in-tree for sm_100a (nvcc).

Run `python -m paper_2502_17632_b200.build_ext` or call `build()`; the
__graft_entry__.build() hook does the same.  Every source is compiled to its
own object (in parallel, under the git-ignored `_obj/`) and only when it or a
header is newer than that object; the objects are then linked in-tree.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libgiftb200.so")
SOURCES = ["csrc/abi.cu", "csrc/build.cu", "csrc/filter.cu", "csrc/bmt.cu", "csrc/metrics.cu", "csrc/plio.cu", "csrc/bookshelf.cu", "csrc/shard.cu", "csrc/hf.cu", "csrc/peer.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-Wno-deprecated-declarations",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


OBJ_DIR = os.path.join(HERE, "_obj")


def _headers() -> list[str]:
    return glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "gift_b200.h")]


def _obj(src: str) -> str:
    return os.path.join(OBJ_DIR, os.path.splitext(os.path.basename(src))[0] + ".o")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def needs_build() -> bool:
    return _stale(LIB, [os.path.join(HERE, s) for s in SOURCES] + _headers())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(OBJ_DIR, exist_ok=True)
    hdrs = _headers()

    def compile_one(src: str) -> None:
        path = os.path.join(HERE, src)
        if not force and not _stale(_obj(src), [path] + hdrs):
            return
        cmd = [_nvcc(), *NVCC_FLAGS, "-c", path, "-o", _obj(src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True, cwd=HERE)

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as pool:
        list(pool.map(compile_one, SOURCES))
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp",
           *[_obj(s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
