"""GiFt multi-frequency filter and placement initialisation on the B200.

Drop-in for `giftplace/gift.py`:

    DEFAULT_TERMS, JITTER_REGION_FRACTION, GiftConfig   gift.py:26-45
    initial_signal                                      gift.py:54-70
    gift_filter                                         gift.py:73-95
    gift_place                                          gift.py:98-119

    g' = 0.1 * A_2^2 g + 0.7 * A_4^2 g + 0.2 * A_4^4 g,
    A_sigma = (D + sigma I)^(-1/2) (A + sigma I) (D + sigma I)^(-1/2)

`initial_signal` stays on the host: it is numpy's PCG64 + ziggurat normal
stream, which is inherently sequential, and keeping it there makes the seed
signal bit-identical to the reference's.  Everything after it runs in
libgiftb200.so.

`GiftConfig.precision` selects the device path:
  "fp32"  (default) fused pre-scaled bank, sigma chains packed per pass,
          <= 1e-5 relative L2 against the reference (north star);
  "fp64"  reference operation order in fp64 -- bit-identical output.
Outputs are float64 numpy arrays like the reference's (fixed rows copied
exactly from the fp64 fixed positions in either mode);
`GiftConfig.output_dtype="float32"` returns float32 instead (the configs'
"N x 2 fp32 output", half the device-to-host bytes).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatchError
from .graph import FilterTerm, SparseSymMatrix, as_device_matrix

DEFAULT_TERMS: tuple[FilterTerm, ...] = (
    FilterTerm(sigma=2.0, k=2, alpha=0.1),
    FilterTerm(sigma=4.0, k=2, alpha=0.7),
    FilterTerm(sigma=4.0, k=4, alpha=0.2),
)

JITTER_REGION_FRACTION = 0.25  # auto jitter_scale as a fraction of min region dimension

_PRECISIONS = {"fp32": _lib.GIFT_PREC_FP32, "fp64": _lib.GIFT_PREC_FP64_EXACT}


@dataclass
class GiftConfig:
    terms: tuple[FilterTerm, ...] = DEFAULT_TERMS
    seed: int = 0
    jitter_scale: float | None = None  # None = JITTER_REGION_FRACTION * min region dim
    precision: str = "fp32"            # extension: "fp32" (fast, fused) | "fp64" (bit-exact)
    output_dtype: str = "float64"      # extension: "float64" (reference) | "float32" (half the D2H bytes)

    def __post_init__(self) -> None:
        self.terms = tuple(self.terms)
        if not self.terms:
            raise ValueError("filter needs at least one term")
        if self.precision not in _PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(_PRECISIONS)}, got {self.precision!r}")
        if self.output_dtype not in ("float64", "float32"):
            raise ValueError(f"output_dtype must be 'float64' or 'float32', got {self.output_dtype!r}")


def _jitter_scale(design, config: GiftConfig) -> float:
    if config.jitter_scale is not None:
        return config.jitter_scale
    return JITTER_REGION_FRACTION * min(design.region.width, design.region.height)


def initial_signal(design, config: GiftConfig) -> np.ndarray:
    """Movable cells at region centre + N(0,1) * jitter_scale; fixed cells pinned.

    Noise is drawn for every cell id in order from default_rng(seed), then
    fixed rows are overwritten (so movable jitter does not depend on which
    cells are fixed) -- the reference's exact stream (gift.py:54-70)."""
    rng = np.random.default_rng(config.seed)
    g = np.tile(design.region.center, (design.num_cells, 1))
    g += rng.standard_normal((design.num_cells, 2)) * _jitter_scale(design, config)
    mask = design.fixed_mask()
    if mask.any():
        g[mask] = design.fixed_positions()[mask]
    return g


def _term_arrays(terms):
    sig = np.ascontiguousarray([t.sigma for t in terms], dtype=np.float64)
    kk = np.ascontiguousarray([t.k for t in terms], dtype=np.int64)
    al = np.ascontiguousarray([t.alpha for t in terms], dtype=np.float64)
    return sig, kk, al


def _run_bank(adj: SparseSymMatrix, g: np.ndarray, config: GiftConfig, design=None) -> np.ndarray:
    torch = _lib.torch_cuda()
    lib = _lib.load_library()
    g = np.asarray(g)
    if g.dtype not in (np.float32, np.float64):
        g = g.astype(np.float64)
    ncols = 1 if g.ndim == 1 else int(np.prod(g.shape[1:]))
    ctx = _lib.context()
    dg = torch.from_numpy(np.ascontiguousarray(g).reshape(adj.n, ncols)).cuda()
    f32_out = config.output_dtype == "float32"
    out = torch.empty((adj.n, ncols), dtype=torch.float32 if f32_out else torch.float64, device=dg.device)
    sig, kk, al = _term_arrays(config.terms)
    in_dtype = _lib.GIFT_DTYPE_F32 if g.dtype == np.float32 else _lib.GIFT_DTYPE_F64
    mask_p = pos_p = None
    region = None
    keep = []
    if design is not None:
        mask = np.ascontiguousarray(design.fixed_mask(), dtype=np.uint8)
        pos = np.nan_to_num(np.asarray(design.fixed_positions(), dtype=np.float64), nan=0.0)
        dm = torch.from_numpy(mask).cuda()
        dp = torch.from_numpy(np.ascontiguousarray(pos)).cuda()
        keep += [dm, dp]
        mask_p, pos_p = _lib.dptr(dm), _lib.dptr(dp)
        r = design.region
        region = np.array([r.xmin, r.ymin, r.xmax, r.ymax], dtype=np.float64)
    st = lib.gift_filter(
        ctx, adj.handle, len(sig), sig.ctypes.data_as(_lib.c_dp), kk.ctypes.data_as(_lib.c_i64p),
        al.ctypes.data_as(_lib.c_dp), ncols, in_dtype, _lib.dptr(dg),
        _lib.GIFT_DTYPE_F32 if f32_out else _lib.GIFT_DTYPE_F64, _lib.dptr(out),
        mask_p, pos_p, region.ctypes.data_as(_lib.c_dp) if region is not None else None,
        _PRECISIONS[config.precision])
    _lib.check(st)
    res = out.cpu().numpy()
    return res.reshape(g.shape)


def gift_filter(adj, g: np.ndarray, config: GiftConfig | None = None) -> np.ndarray:
    """Apply sum(alpha * A_sigma^k) to each column of g (linear; no clamping or pinning)."""
    config = config or GiftConfig()
    adj = as_device_matrix(adj)
    g = np.asarray(g)
    if g.shape[0] != adj.n:
        raise DimensionMismatchError(f"signal has {g.shape[0]} rows, graph has {adj.n} nodes")
    return _run_bank(adj, g, config)


def gift_place(design, adj, config: GiftConfig | None = None) -> tuple[np.ndarray, dict[str, float]]:
    """Seed signal, filter, re-pin fixed cells, clamp movable cells to the region.

    Returns (placement float64 [N, 2], {"filter": seconds}); the re-pin/clamp
    epilogue is fused into the bank's final hop on the device."""
    config = config or GiftConfig()
    adj = as_device_matrix(adj)
    g = initial_signal(design, config)
    if g.shape[0] != adj.n:
        raise DimensionMismatchError(f"signal has {g.shape[0]} rows, graph has {adj.n} nodes")
    torch = _lib.torch_cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = _run_bank(adj, g, config, design=design)
    filter_seconds = time.perf_counter() - t0
    return out, {"filter": filter_seconds}


def gift_place_arrays(net_start, pin_cell, g0, fixed_mask, fixed_pos, region, terms=DEFAULT_TERMS,
                      max_clique_pins: int | None = None, precision: str = "fp32",
                      out_dtype=np.float64, implicit_above: int | None = None) -> tuple[np.ndarray, int]:
    """Netlist in, positions out, through the single host-buffer C ABI call
    `gift_place_host` (H2D, clique build, bank, epilogue, D2H).
    Returns (positions [N, 2], nnz of the clique graph).  implicit_above=T:
    the factored clique model (see build_clique_graph) -- nets above T pins
    applied as the O(pins) implicit term; nnz then counts the stored part."""
    if implicit_above is not None:
        if int(implicit_above) < 2:
            raise ValueError(f"implicit_above must be >= 2, got {implicit_above}")
        with _lib.options(implicit_above=int(implicit_above)):
            return gift_place_arrays(net_start, pin_cell, g0, fixed_mask, fixed_pos, region, terms, max_clique_pins,
                                     precision, out_dtype)
    lib = _lib.load_library()
    ctx = _lib.context()
    net_start = np.ascontiguousarray(net_start, dtype=np.int64)
    pin_cell = np.ascontiguousarray(pin_cell, dtype=np.int32)
    g0 = np.ascontiguousarray(g0, dtype=np.float32)
    n = g0.shape[0]
    mask = np.ascontiguousarray(fixed_mask, dtype=np.uint8)
    pos = np.ascontiguousarray(np.nan_to_num(np.asarray(fixed_pos, dtype=np.float64), nan=0.0))
    reg = np.ascontiguousarray(region, dtype=np.float64)
    sig, kk, al = _term_arrays(terms)
    out = np.empty((n, 2), dtype=out_dtype)
    nnz = ctypes.c_int64(0)
    cap = max(int(max_clique_pins), 0) if max_clique_pins is not None else -1  # -1 = None
    _lib.check(lib.gift_place_host(
        ctx, n, len(net_start) - 1, net_start.ctypes.data_as(ctypes.c_void_p),
        pin_cell.ctypes.data_as(ctypes.c_void_p), cap, len(sig), sig.ctypes.data_as(_lib.c_dp),
        kk.ctypes.data_as(_lib.c_i64p), al.ctypes.data_as(_lib.c_dp), g0.ctypes.data_as(ctypes.c_void_p),
        mask.ctypes.data_as(ctypes.c_void_p), pos.ctypes.data_as(ctypes.c_void_p), reg.ctypes.data_as(_lib.c_dp),
        _lib.GIFT_DTYPE_F64 if out_dtype == np.float64 else _lib.GIFT_DTYPE_F32,
        out.ctypes.data_as(ctypes.c_void_p), _PRECISIONS[precision], ctypes.byref(nnz)))
    return out, int(nnz.value)
