"""ctypes binding of libgiftb200.so (the C ABI declared in include/gift_b200.h).

The library is the product: there is no CPU fallback.  Loading fails loudly
(`DeviceError`) when the shared object is missing or no CUDA device is
visible.  Device buffers handed to the library are torch CUDA tensors
(PyTorch is plumbing here: allocation, streams, host<->device copies).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    DeviceError,
    DimensionMismatchError,
    GiftPlaceError,
    IsolatedNodeError,
    NonSymmetricError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
# GIFT_LIB: an alternative build of the same library (A/B of compile-time variants, tools/)
LIB_PATH = os.environ.get("GIFT_LIB") or os.path.join(HERE, "libgiftb200.so")

GIFT_OK = 0
GIFT_ERR_VALUE = 1
GIFT_ERR_DIMENSION = 2
GIFT_ERR_ISOLATED_NODE = 3
GIFT_ERR_NON_SYMMETRIC = 4
GIFT_ERR_TOO_LARGE = 5
GIFT_ERR_CUDA = 6
GIFT_ERR_OOM = 7
GIFT_ERR_INTERNAL = 8

GIFT_PREC_FP32 = 0
GIFT_PREC_FP64_EXACT = 1
GIFT_DTYPE_F32 = 0
GIFT_DTYPE_F64 = 1

GIFT_TILED_NEVER = 0
GIFT_TILED_ON_REUSE = 1
GIFT_TILED_ALWAYS = 2

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_vp = ctypes.c_void_p
c_dp = ctypes.POINTER(ctypes.c_double)
c_i64p = ctypes.POINTER(ctypes.c_int64)

# (name, restype, argtypes) -- every symbol include/gift_b200.h declares
SIGNATURES = [
    ("gift_ctx_create", c_int, [c_int, ctypes.POINTER(c_vp)]),
    ("gift_ctx_destroy", c_int, [c_vp]),
    ("gift_ctx_set_stream", c_int, [c_vp, c_vp]),
    ("gift_last_error", ctypes.c_char_p, []),
    ("gift_last_error_arg", c_i64, []),
    ("gift_version", ctypes.c_char_p, []),
    ("gift_ctx_set_tiled_policy", c_int, [c_vp, c_int]),
    ("gift_ctx_set_option", c_int, [c_vp, ctypes.c_char_p, c_i64]),
    ("gift_csr_tiled_info", c_int, [c_vp, c_int, c_i64p]),
    ("gift_ctx_launch_count", c_i64, [c_vp]),
    ("gift_ctx_set_profiling", c_int, [c_vp, c_int]),
    ("gift_ctx_profile_drain", c_int, [c_vp, c_int, c_vp, c_vp, c_vp, ctypes.POINTER(c_int)]),
    ("gift_build_clique_graph", c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, ctypes.POINTER(c_vp), c_i64p]),
    ("gift_csr_from_coo", c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, ctypes.POINTER(c_vp)]),
    ("gift_csr_destroy", c_int, [c_vp]),
    ("gift_csr_shape", c_int, [c_vp, c_i64p, c_i64p]),
    ("gift_csr_arrays", c_int, [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)]),
    ("gift_csr_download", c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    ("gift_csr_degrees", c_int, [c_vp, c_vp, ctypes.POINTER(c_vp)]),
    ("gift_normalized_augmented_adjacency", c_int, [c_vp, c_vp, ctypes.c_double, ctypes.POINTER(c_vp)]),
    ("gift_csr_matmul", c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    ("gift_filter", c_int, [c_vp, c_vp, c_int, c_dp, c_i64p, c_dp, c_i64, c_int, c_vp, c_int, c_vp, c_vp, c_vp,
                            c_dp, c_int]),
    ("gift_filter_host", c_int, [c_vp, c_vp, c_int, c_dp, c_i64p, c_dp, c_i64, c_int, c_vp, c_int, c_vp, c_vp,
                                 c_vp, c_dp, c_int]),
    ("gift_place_host", c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_int, c_dp, c_i64p, c_dp, c_vp, c_vp, c_vp,
                                c_dp, c_int, c_vp, c_int, c_i64p]),
    # stepped bank (shard.py)
    ("gift_csr_scale", c_int, [c_vp, c_vp, ctypes.c_double, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)]),
    ("gift_csr_weights32", c_int, [c_vp, c_vp, ctypes.POINTER(c_vp)]),
    ("gift_csr_from_arrays", c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, ctypes.POINTER(c_vp)]),
    ("gift_hop_fp32", c_int, [c_vp, c_vp, c_vp]),
    ("gift_pack_fp32", c_int, [c_vp, c_i64, c_int, c_int, c_vp, c_int, c_vp, c_i64, c_i64, c_int, c_vp]),
    ("gift_gather_rows_f32", c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_vp]),
    ("gift_peer_alloc", c_int, [c_vp, c_i64, ctypes.POINTER(c_vp), c_vp]),
    ("gift_peer_open", c_int, [c_vp, c_vp, ctypes.POINTER(c_vp)]),
    ("gift_peer_close", c_int, [c_vp, c_vp]),
    ("gift_peer_free", c_int, [c_vp, c_vp]),
    ("gift_pull_rows_f32", c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_vp]),
    ("gift_pull_join", c_int, [c_vp]),
    ("gift_csr_row_bounds", c_int, [c_vp, c_vp, c_int, c_i64p]),
    ("gift_csr_attach_high_fanout", c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64p]),
    ("gift_csr_attach_implicit_nets", c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64p]),
    ("gift_csr_split_rows", c_int, [c_vp, c_vp, c_i64, c_i64, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)]),
    ("gift_csr_ext_ids", c_int, [c_vp, ctypes.POINTER(c_vp), c_i64p]),
    # placement metrics (metrics.py)
    ("gift_quadratic_wirelength", c_int, [c_vp, c_vp, c_vp, c_dp]),
    ("gift_laplacian", c_int, [c_vp, c_vp, ctypes.POINTER(c_vp)]),
    ("gift_rayleigh_parts", c_int, [c_vp, c_vp, c_vp, c_int, c_dp, c_dp]),
    ("gift_hpwl", c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_dp]),
    ("gift_format_placement", c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_char_p, c_vp,
                                      c_i64, c_i64p]),
    ("gift_bookshelf_parse", c_int, [c_vp, ctypes.c_char_p, c_i64, ctypes.c_char_p, c_i64, ctypes.c_char_p, c_i64,
                                     ctypes.POINTER(c_vp)]),
    ("gift_bookshelf_info", c_int, [c_vp, c_i64p, c_dp]),
    ("gift_bookshelf_device", c_int, [c_vp] + [ctypes.POINTER(c_vp)] * 8),
    ("gift_bookshelf_copy", c_int, [c_vp, c_vp] + [c_vp] * 12),
    ("gift_bookshelf_destroy", c_int, [c_vp, c_vp]),
]

_lib = None
_lock = threading.Lock()
_ctxs: dict[tuple[int, int], int] = {}  # (thread id, device) -> gift_ctx*
_policy = GIFT_TILED_ON_REUSE
_options: dict[str, int] = {}


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """dlopen the library and bind every symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DeviceError(
                    f"CUDA library {path} is missing; build it with "
                    "`python -m paper_2502_17632_b200.build_ext` (there is no CPU fallback)")
            lib = ctypes.CDLL(path)
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int) -> None:
    """Map a C ABI status to the reference's exception classes."""
    if status == GIFT_OK:
        return
    lib = load_library()
    msg = (lib.gift_last_error() or b"").decode(errors="replace")
    if status == GIFT_ERR_VALUE:
        raise ValueError(msg)
    if status == GIFT_ERR_DIMENSION:
        raise DimensionMismatchError(msg)
    if status == GIFT_ERR_ISOLATED_NODE:
        raise IsolatedNodeError(int(lib.gift_last_error_arg()))
    if status == GIFT_ERR_NON_SYMMETRIC:
        raise NonSymmetricError(msg)
    if status in (GIFT_ERR_CUDA, GIFT_ERR_OOM):
        raise DeviceError(msg)
    raise GiftPlaceError(msg)


def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the GiFt B200 path has no CPU fallback")
    return torch


def context(device: int | None = None) -> int:
    """Library context of (this thread, device), bound to torch's current
    stream.  A gift_ctx holds per-call scratch and a stream, so threads get
    their own (the library also serialises entry points on a context)."""
    torch = torch_cuda()
    lib = load_library()
    dev = torch.cuda.current_device() if device is None else int(device)
    key = (threading.get_ident(), dev)
    ctx = _ctxs.get(key)
    if ctx is None:
        h = c_vp()
        check(lib.gift_ctx_create(dev, ctypes.byref(h)))
        ctx = h.value
        check(lib.gift_ctx_set_tiled_policy(ctx, _policy))
        for name, value in _options.items():
            check(lib.gift_ctx_set_option(ctx, name.encode(), int(value)))
        with _lock:
            _ctxs[key] = ctx
    stream = torch.cuda.current_stream(dev).cuda_stream
    check(lib.gift_ctx_set_stream(ctx, c_vp(stream)))
    return ctx


def set_tiled_policy(policy: str) -> None:
    """When the fp32 bank builds a graph's tiled copy: "on_reuse" (default:
    the first bank on a graph runs the row kernel, later ones build and use
    the copy), "always" (first hop) or "never"."""
    global _policy
    codes = {"never": GIFT_TILED_NEVER, "on_reuse": GIFT_TILED_ON_REUSE, "always": GIFT_TILED_ALWAYS}
    if policy not in codes:
        raise ValueError(f"tiled policy must be one of {sorted(codes)}, got {policy!r}")
    _policy = codes[policy]
    lib = load_library()
    with _lock:
        ctxs = list(_ctxs.values())
    for ctx in ctxs:
        check(lib.gift_ctx_set_tiled_policy(ctx, _policy))


DEFAULT_OPTIONS = {"tiled": 1, "tiled_min_rows": 98304, "tiled_min_mean": 32, "tile_rows": 0, "col_bits": 0,
                   "barrier_free": 1, "graphs": 1, "fused": 1, "zero_copy": 1, "schedule": 2, "row_lanes": 0,
                   "codes": 0, "prefetch": 0, "stream": 0, "balance": 1, "implicit_above": 0}


def set_option(name: str, value: int) -> None:
    """Kernel-selection option (gift_ctx_set_option) for every context, present
    and future: tiled, tiled_min_rows, tiled_min_mean, tile_rows, col_bits,
    barrier_free, graphs, zero_copy, schedule, row_lanes, balance."""
    if name not in DEFAULT_OPTIONS:
        raise ValueError(f"unknown option {name!r}")
    lib = load_library()
    with _lock:
        ctxs = list(_ctxs.values())
    for ctx in ctxs:
        check(lib.gift_ctx_set_option(ctx, name.encode(), int(value)))
    if value == DEFAULT_OPTIONS[name]:
        _options.pop(name, None)
    else:
        _options[name] = int(value)


class options:
    """Context manager: `with options(tiled_min_rows=1): ...` sets kernel
    options and restores the previous values on exit (tests, sweeps)."""

    def __init__(self, **kw):
        self.kw = kw
        self.prev = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.prev[k] = _options.get(k, DEFAULT_OPTIONS.get(k))
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.prev.items():
            set_option(k, v)
        return False


def launch_count(device: int | None = None) -> int:
    torch = torch_cuda()
    dev = torch.cuda.current_device() if device is None else int(device)
    ctx = _ctxs.get((threading.get_ident(), dev))
    return int(load_library().gift_ctx_launch_count(ctx)) if ctx else 0


def set_profiling(on: bool, device: int | None = None) -> None:
    check(load_library().gift_ctx_set_profiling(context(device), 1 if on else 0))


def drain_profile(device: int | None = None, max_records: int = 1 << 16):
    """[(kind, units, ms)] for the launches recorded since the last drain."""
    import numpy as np

    kind = np.zeros(max_records, dtype=np.int32)
    units = np.zeros(max_records, dtype=np.int32)
    ms = np.zeros(max_records, dtype=np.float32)
    n = c_int(0)
    check(load_library().gift_ctx_profile_drain(
        context(device), max_records, kind.ctypes.data_as(c_vp), units.ctypes.data_as(c_vp),
        ms.ctypes.data_as(c_vp), ctypes.byref(n)))
    k = n.value
    return list(zip(kind[:k].tolist(), units[:k].tolist(), ms[:k].tolist()))


def dptr(t) -> c_vp:
    return c_vp(t.data_ptr())
