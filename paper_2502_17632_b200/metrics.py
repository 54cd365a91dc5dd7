"""Placement-quality measures on the device.

Consumers of the filter output, reusing the resident CSR / pin table:

    quadratic_wirelength(adj, g)        metrics.py:63-74
    laplacian(adj)                      graph.py:161-164 (bit-exact)
    rayleigh_smoothness(lap, col, ...)  metrics.py:77-92
    hpwl(design, g)                     metrics.py:95-112

fp64 with fixed reduction trees: deterministic, and equal to the reference up
to summation order (~1e-15 relative).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DimensionMismatchError, ZeroSignalError
from .graph import SparseSymMatrix, as_device_matrix
from .netlist import FlatDesign


def _dev(a):
    torch = _lib.torch_cuda()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def quadratic_wirelength(adj, g: np.ndarray) -> float:
    """S(g) = sum_ij w_ij * ((x_i-x_j)^2 + (y_i-y_j)^2) over unordered pairs."""
    adj = as_device_matrix(adj)
    g = np.asarray(g, dtype=np.float64)
    if g.shape[0] != adj.n:
        raise DimensionMismatchError(f"placement has {g.shape[0]} rows, graph has {adj.n} nodes")
    if adj.nnz == 0:
        return 0.0
    out = ctypes.c_double()
    dg = _dev(g.reshape(adj.n, 2))
    _lib.check(_lib.load_library().gift_quadratic_wirelength(_lib.context(), adj.handle, _lib.dptr(dg),
                                                            ctypes.byref(out)))
    return float(out.value)


def laplacian(adj) -> SparseSymMatrix:
    """Combinatorial Laplacian L = D - A, built on the device."""
    adj = as_device_matrix(adj)
    h = ctypes.c_void_p()
    _lib.check(_lib.load_library().gift_laplacian(_lib.context(), adj.handle, ctypes.byref(h)))
    return SparseSymMatrix._from_handle(h.value)


def rayleigh_smoothness(laplacian_op, column: np.ndarray, center: bool = True) -> float:
    """R(g) = g^T L g / g^T g, after mean-centering by default."""
    lap = as_device_matrix(laplacian_op)
    col = np.asarray(column, dtype=np.float64).ravel()
    if col.shape[0] != lap.n:
        raise DimensionMismatchError(f"signal has {col.shape[0]} rows, Laplacian has {lap.n}")
    num, den = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.load_library().gift_rayleigh_parts(_lib.context(), lap.handle, _lib.dptr(_dev(col)),
                                                      1 if center else 0, ctypes.byref(num), ctypes.byref(den)))
    if den.value <= 1e-30:
        raise ZeroSignalError("signal is zero (or constant, after centering)")
    return float(num.value) / float(den.value)


def hpwl(design, g: np.ndarray) -> float:
    """Half-perimeter wirelength over pin positions (cell centre + pin offset)."""
    g = np.asarray(g, dtype=np.float64)
    if isinstance(design, FlatDesign):
        net_start, pin_cell = design.net_start, design.pin_cell
        pdx = pdy = None
    else:
        net_start, pin_cell, pdx, pdy = design.pin_table()
        if not (np.any(pdx) or np.any(pdy)):
            pdx = pdy = None
    if len(pin_cell) == 0:
        return 0.0
    keep = [_dev(np.asarray(net_start, dtype=np.int64)), _dev(np.asarray(pin_cell, dtype=np.int32)),
            _dev(g.reshape(-1, 2))]
    ddx = _dev(np.asarray(pdx, dtype=np.float64)) if pdx is not None else None
    ddy = _dev(np.asarray(pdy, dtype=np.float64)) if pdy is not None else None
    out = ctypes.c_double()
    _lib.check(_lib.load_library().gift_hpwl(
        _lib.context(), len(net_start) - 1, _lib.dptr(keep[0]), _lib.dptr(keep[1]),
        _lib.dptr(ddx) if ddx is not None else None, _lib.dptr(ddy) if ddy is not None else None,
        _lib.dptr(keep[2]), ctypes.byref(out)))
    return float(out.value)
