"""Bookshelf .pl writer on the device.

    write_placement(design, placement, path)   netlist.py:503-522
    format_placement(design, placement) -> bytes

Same name, arguments, error and bytes as the reference's `write_placement`:
"UCLA pl 1.0", a blank line, then `name<TAB>llx<TAB>lly<TAB>: N[ /FIXED]` per
cell in `design.cells` order, lower-left corners in fixed 6-decimal format
(`PL_PRECISION`, netlist.py:29).  The text is produced by
`gift_format_placement` (csrc/plio.cu): exact %.6f formatting in 128-bit
integer arithmetic, one thread per cell.  A `FlatDesign` has no name strings;
its cells are "c<i>" (the names `FlatDesign.to_design` and the reference's
benchgen give them), generated on the device.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import GiftPlaceError
from .netlist import FlatDesign

PL_PRECISION = 6  # netlist.py:29 -- the device formatter is fixed at 6 decimals


def _columns(design):
    """(widths, heights, fixed uint8, names bytes | None, name offsets | None, prefix, rows)."""
    if isinstance(design, FlatDesign):
        n = design.num_cells
        return (np.ascontiguousarray(design.widths, dtype=np.float64),
                np.ascontiguousarray(design.heights, dtype=np.float64),
                design.fixed_mask().astype(np.uint8), None, None, b"c", None)
    cells = design.cells
    n = len(cells)
    w = np.fromiter((c.width for c in cells), dtype=np.float64, count=n)
    h = np.fromiter((c.height for c in cells), dtype=np.float64, count=n)
    fx = np.fromiter((bool(c.fixed) for c in cells), dtype=np.uint8, count=n)
    ids = np.fromiter((c.id for c in cells), dtype=np.int64, count=n)
    encoded = [c.name.encode() for c in cells]
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.fromiter((len(b) for b in encoded), dtype=np.int64, count=n), out=off[1:])
    names = np.frombuffer(b"".join(encoded), dtype=np.uint8) if n else np.zeros(0, np.uint8)
    rows = None if np.array_equal(ids, np.arange(n)) else ids
    return w, h, fx, names, off, b"", rows


def format_placement(design, placement: np.ndarray) -> bytes:
    """The exact bytes `write_placement` would write."""
    placement = np.asarray(placement, dtype=float)
    if placement.shape != (design.num_cells, 2):
        raise GiftPlaceError(
            f"placement shape {placement.shape} does not match design with {design.num_cells} cells"
        )
    torch = _lib.torch_cuda()
    lib = _lib.load_library()
    w, h, fx, names, off, prefix, rows = _columns(design)
    pos = placement if rows is None else placement[rows]  # cell order, rows by cell.id (netlist.py:515)
    n = pos.shape[0]

    def dev(a):
        return torch.from_numpy(np.require(a, requirements=["C", "W"])).cuda()

    keep = [dev(pos), dev(w), dev(h), dev(fx)]
    d_names = d_off = None
    if names is not None:
        keep += [dev(names if len(names) else np.zeros(1, np.uint8)), dev(off)]
        d_names, d_off = _lib.dptr(keep[4]), _lib.dptr(keep[5])
    args = [_lib.context(), n, _lib.dptr(keep[0]), _lib.dptr(keep[1]), _lib.dptr(keep[2]), _lib.dptr(keep[3]),
            d_names, d_off, prefix]
    size = ctypes.c_int64()
    _lib.check(lib.gift_format_placement(*args, None, 0, ctypes.byref(size)))
    out = torch.empty(size.value, dtype=torch.uint8, device="cuda")
    _lib.check(lib.gift_format_placement(*args, _lib.dptr(out), size.value, ctypes.byref(size)))
    return out.cpu().numpy().tobytes()


def write_placement(design, placement: np.ndarray, path: str) -> None:
    """Write a .pl file; coordinates are converted to lower-left corners.

    Fixed cells carry the /FIXED marker; the output is deterministic (no
    timestamps, fixed 6-decimal coordinates) and byte-identical to the
    reference writer (netlist.py:503-522).
    """
    data = format_placement(design, placement)
    with open(path, "wb") as f:
        f.write(data)
