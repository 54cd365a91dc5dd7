"""ctypes wrapper around oracle/gift_oracle.c -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker (or as the
timed CPU baseline). The product path never touches it.

Each function names the reference code it restates (see gift_oracle.c for the
file:line map). Arrays are numpy; index arrays are int64; values fp64.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libgift_oracle.so")
_PROBE_PATH = os.path.join(_HERE, "_build", "libstdsort_probe.so")

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i32p = ctypes.POINTER(ctypes.c_int)

_lib = None
_probe = None


def build() -> None:
    """Compile the oracle (gcc) into oracle/_build/, and stage the reference."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    stage_reference()


REF_SRC = "/root/reference/pkg/src/giftplace"
REF_DIR = os.path.join(_HERE, "_ref")


def stage_reference(src: str = REF_SRC) -> bool:
    """Copy the reference package (pure Python) into oracle/_ref/ -- git-ignored,
    it travels to the GPU box with the built libraries -- so bench.py's
    cpu_baseline leg can time the reference's own gift_filter (gift.py:73-95)
    where /root/reference does not exist.  No-op when the source is absent
    (the GPU box uses the staged copy)."""
    import shutil

    if not os.path.isdir(src):
        return os.path.isdir(os.path.join(REF_DIR, "giftplace"))
    dst = os.path.join(REF_DIR, "giftplace")
    if os.path.isdir(dst):
        shutil.rmtree(dst)
    shutil.copytree(src, dst, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    return True


def reference_module():
    """The staged reference package (`giftplace`), or None."""
    import importlib
    import sys

    if not os.path.isdir(os.path.join(REF_DIR, "giftplace")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    return importlib.import_module("giftplace")


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.orc_count_clique_pairs.restype = ctypes.c_int64
        lib.orc_count_clique_pairs.argtypes = [ctypes.c_int64, _i64p, ctypes.c_int64]
        lib.orc_build_clique_graph.restype = ctypes.c_int64
        lib.orc_build_clique_graph.argtypes = [
            ctypes.c_int64, ctypes.c_int64, _i64p, _i64p, ctypes.c_int64,
            _i64p, _i64p, _f64p, _i64p, _i32p,
        ]
        lib.orc_emit_clique_pairs.restype = ctypes.c_int64
        lib.orc_emit_clique_pairs.argtypes = [
            ctypes.c_int64, _i64p, _i64p, ctypes.c_int64, _i64p, _i64p, _f64p, _i64p,
        ]
        lib.orc_coo_to_csr.restype = ctypes.c_int64
        lib.orc_coo_to_csr.argtypes = [
            ctypes.c_int64, ctypes.c_int64, _i64p, _i64p, _f64p, ctypes.c_int,
            _i64p, _i64p, _f64p, _i32p,
        ]
        lib.orc_degrees.restype = None
        lib.orc_degrees.argtypes = [ctypes.c_int64, _i64p, _f64p, _f64p]
        lib.orc_inv_sqrt_scale.restype = ctypes.c_int64
        lib.orc_inv_sqrt_scale.argtypes = [ctypes.c_int64, _f64p, ctypes.c_double, _f64p]
        lib.orc_normalized.restype = ctypes.c_int64
        lib.orc_normalized.argtypes = [
            ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, ctypes.c_double, _i64p, _i64p, _f64p,
        ]
        lib.orc_matvecs.restype = None
        lib.orc_matvecs.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p]
        lib.orc_gift_filter.restype = ctypes.c_int64
        lib.orc_gift_filter.argtypes = [
            ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, ctypes.c_int, _f64p, _i64p, _f64p,
            ctypes.c_int64, _f64p, _f64p,
        ]
        lib.orc_place_epilogue.restype = None
        lib.orc_place_epilogue.argtypes = [ctypes.c_int64, _f64p, _u8p, _f64p, _f64p]
        lib.orc_std_sort_perm.restype = None
        lib.orc_std_sort_perm.argtypes = [ctypes.c_int64, _i64p, _i64p]
        lib.orc_heapsort_calls.restype = ctypes.c_int64
        lib.orc_num_threads.restype = ctypes.c_int
        lib.orc_set_num_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return int(_load().orc_num_threads())


def set_num_threads(t: int) -> None:
    _load().orc_set_num_threads(int(t))


@dataclass
class CSR:
    n: int
    indptr: np.ndarray   # int64 [n+1]
    indices: np.ndarray  # int64 [nnz]
    data: np.ndarray     # fp64 [nnz]
    input_rows_sorted: bool = True  # scipy skipped std::sort (A.3)

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])


def build_clique_graph(n: int, net_start, pin_cell, max_clique_pins: int | None = None) -> CSR:
    """graph.py:120-158 on flat pin arrays (Design.pin_table, netlist.py:142-166)."""
    lib = _load()
    net_start = _i64(net_start)
    pin_cell = _i64(pin_cell)
    n_nets = len(net_start) - 1
    # None = no cap; any cap < 2 skips every net with >= 2 pins (m > cap), as the reference
    cap = max(int(max_clique_pins), 0) if max_clique_pins is not None else -1
    T = int(lib.orc_count_clique_pairs(n_nets, _p(net_start, _i64p), cap))
    indptr = np.zeros(n + 1, dtype=np.int64)
    indices = np.empty(max(2 * T, 1), dtype=np.int64)
    data = np.empty(max(2 * T, 1), dtype=np.float64)
    skipped = ctypes.c_int64(0)
    srt = ctypes.c_int(1)
    nnz = int(lib.orc_build_clique_graph(
        n, n_nets, _p(net_start, _i64p), _p(pin_cell, _i64p), cap,
        _p(indptr, _i64p), _p(indices, _i64p), _p(data, _f64p),
        ctypes.byref(skipped), ctypes.byref(srt),
    ))
    return CSR(n, indptr, indices[:nnz].copy(), data[:nnz].copy(), bool(srt.value))


def coo_to_csr(n: int, rows, cols, vals, drop_zeros: bool = True) -> CSR:
    """scipy coo_matrix((vals,(rows,cols))).tocsr() + eliminate_zeros (graph.py:114-117, :57-58)."""
    lib = _load()
    rows, cols, vals = _i64(rows), _i64(cols), _f64(vals)
    k = len(rows)
    indptr = np.zeros(n + 1, dtype=np.int64)
    indices = np.empty(max(k, 1), dtype=np.int64)
    data = np.empty(max(k, 1), dtype=np.float64)
    srt = ctypes.c_int(1)
    nnz = int(lib.orc_coo_to_csr(
        n, k, _p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p), int(drop_zeros),
        _p(indptr, _i64p), _p(indices, _i64p), _p(data, _f64p), ctypes.byref(srt),
    ))
    return CSR(n, indptr, indices[:nnz].copy(), data[:nnz].copy(), bool(srt.value))


def degrees(csr: CSR) -> np.ndarray:
    """graph.py:89-94 (np.add.reduceat pairwise order)."""
    out = np.empty(csr.n, dtype=np.float64)
    _load().orc_degrees(csr.n, _p(csr.indptr, _i64p), _p(csr.data, _f64p), _p(out, _f64p))
    return out


def inv_sqrt_scale(deg: np.ndarray, sigma: float) -> np.ndarray:
    """graph.py:176-184; raises LookupError(node) for an isolated node at sigma == 0."""
    deg = _f64(deg)
    s = np.empty_like(deg)
    iso = int(_load().orc_inv_sqrt_scale(len(deg), _p(deg, _f64p), float(sigma), _p(s, _f64p)))
    if iso >= 0:
        raise LookupError(iso)
    return s


def normalized(csr: CSR, sigma: float, deg: np.ndarray | None = None) -> CSR:
    """graph.py:167-188, materialised."""
    deg = degrees(csr) if deg is None else _f64(deg)
    s = inv_sqrt_scale(deg, sigma)
    n = csr.n
    o_ptr = np.zeros(n + 1, dtype=np.int64)
    o_idx = np.empty(csr.nnz + n + 1, dtype=np.int64)
    o_val = np.empty(csr.nnz + n + 1, dtype=np.float64)
    k = int(_load().orc_normalized(
        n, _p(csr.indptr, _i64p), _p(csr.indices, _i64p), _p(csr.data, _f64p),
        _p(s, _f64p), float(sigma), _p(o_ptr, _i64p), _p(o_idx, _i64p), _p(o_val, _f64p),
    ))
    return CSR(n, o_ptr, o_idx[:k].copy(), o_val[:k].copy())


def matmul(csr: CSR, x) -> np.ndarray:
    """graph.py:96-100 -> scipy csr_matvecs (sequential fp64 per row)."""
    x = _f64(x)
    one_d = x.ndim == 1
    x2 = x.reshape(csr.n, -1)
    y = np.empty_like(x2)
    _load().orc_matvecs(csr.n, x2.shape[1], _p(csr.indptr, _i64p), _p(csr.indices, _i64p),
                        _p(csr.data, _f64p), _p(x2, _f64p), _p(y, _f64p))
    return y.ravel() if one_d else y


def gift_filter(csr: CSR, g, terms, deg: np.ndarray | None = None) -> np.ndarray:
    """gift.py:73-95. terms: iterable of (sigma, k, alpha)."""
    terms = list(terms)
    g = _f64(g)
    one_d = g.ndim == 1
    g2 = g.reshape(csr.n, -1)
    out = np.empty_like(g2)
    sig = _f64([t[0] for t in terms])
    kk = _i64([t[1] for t in terms])
    al = _f64([t[2] for t in terms])
    deg_arr = None if deg is None else _f64(deg)
    st = int(_load().orc_gift_filter(
        csr.n, _p(csr.indptr, _i64p), _p(csr.indices, _i64p), _p(csr.data, _f64p),
        _p(deg_arr, _f64p) if deg_arr is not None else None,
        len(terms), _p(sig, _f64p), _p(kk, _i64p), _p(al, _f64p), g2.shape[1],
        _p(g2, _f64p), _p(out, _f64p),
    ))
    if st >= 0:
        raise LookupError(st)
    return out.ravel() if one_d else out


def place_epilogue(out: np.ndarray, fixed_mask, fixed_pos, region) -> np.ndarray:
    """gift.py:112-118 (in place on a copy)."""
    out = _f64(out).copy()
    n = out.shape[0]
    mask = np.ascontiguousarray(fixed_mask, dtype=np.uint8)
    fpos = _f64(np.nan_to_num(np.asarray(fixed_pos, dtype=float), nan=0.0))
    reg = _f64(region)
    _load().orc_place_epilogue(n, _p(out, _f64p), _p(mask, _u8p), _p(fpos, _f64p), _p(reg, _f64p))
    return out


def gift_place(csr: CSR, g0, terms, fixed_mask, fixed_pos, region, deg=None) -> np.ndarray:
    """gift.py:98-119 without the host RNG (g0 = initial_signal output)."""
    out = gift_filter(csr, g0, terms, deg)
    return place_epilogue(out, fixed_mask, fixed_pos, region)


def heapsort_calls() -> int:
    """Times the introsort restatement fell back to heapsort (coverage probe)."""
    return int(_load().orc_heapsort_calls())


def std_sort_perm_emulated(keys) -> np.ndarray:
    keys = _i64(keys)
    perm = np.empty(len(keys), dtype=np.int64)
    _load().orc_std_sort_perm(len(keys), _p(keys, _i64p), _p(perm, _i64p))
    return perm


def std_sort_perm_libstdcxx(keys) -> np.ndarray:
    """The real libstdc++ std::sort (stdsort_probe.cpp) for cross-checking."""
    global _probe
    if _probe is None:
        if not os.path.exists(_PROBE_PATH):
            build()
        _probe = ctypes.CDLL(_PROBE_PATH)
        _probe.probe_std_sort_perm.argtypes = [ctypes.c_int64, _i64p, _i64p]
    keys = _i64(keys)
    perm = np.empty(len(keys), dtype=np.int64)
    _probe.probe_std_sort_perm(len(keys), _p(keys, _i64p), _p(perm, _i64p))
    return perm


def antiqsort_keys(n: int) -> np.ndarray:
    """Adversarial keys (McIlroy) that push libstdc++ introsort to heapsort."""
    std_sort_perm_libstdcxx(np.zeros(0, dtype=np.int64))  # loads the probe
    _probe.probe_antiqsort.argtypes = [ctypes.c_int64, _i64p]
    out = np.empty(n, dtype=np.int64)
    _probe.probe_antiqsort(n, _p(out, _i64p))
    return out
