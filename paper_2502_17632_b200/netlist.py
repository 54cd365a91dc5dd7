"""Design model: the input contract of the GiFt hot path.

Two interchangeable front doors feed `build_clique_graph` / `gift_place`:

* the object model (`Cell`, `Pin`, `Net`, `Row`, `Region`, `Design`) with the
  same field names and accessor semantics as the reference
  (`giftplace/netlist.py:32-189`), so code written against the reference
  builds designs unchanged;
* `FlatDesign`, an array-native design (CSR-like pin table + fixed arrays)
  for multi-million-cell netlists where ten million Python `Cell` objects
  would dominate end-to-end time.

Both expose the accessors the path reads: `num_cells`, `fixed_mask()`,
`fixed_positions()`, `pin_table()` and `region` (netlist.py:104-166).
Bookshelf text I/O is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import GiftPlaceError


@dataclass
class Cell:
    """A placeable object; `fixed_pos` (centre) is set iff `fixed` (netlist.py:32-41)."""

    id: int
    name: str
    width: float
    height: float
    fixed: bool = False
    fixed_pos: tuple[float, float] | None = None


@dataclass
class Pin:
    """A net pin on cell `cell` with an offset from its centre (netlist.py:44-50)."""

    cell: int
    dx: float = 0.0
    dy: float = 0.0


@dataclass
class Net:
    """A hyperedge; `degree` counts every pin, duplicates included (netlist.py:53-61)."""

    id: int
    name: str
    pins: list[Pin] = field(default_factory=list)

    @property
    def degree(self) -> int:
        return len(self.pins)


@dataclass
class Row:
    y: float
    height: float
    x: float
    num_sites: int
    site_width: float = 1.0


@dataclass
class Region:
    """Placement region; `center` seeds the initial signal (netlist.py:74-93)."""

    xmin: float
    ymin: float
    xmax: float
    ymax: float
    rows: list[Row] = field(default_factory=list)

    @property
    def width(self) -> float:
        return self.xmax - self.xmin

    @property
    def height(self) -> float:
        return self.ymax - self.ymin

    @property
    def center(self) -> tuple[float, float]:
        return (0.5 * (self.xmin + self.xmax), 0.5 * (self.ymin + self.ymax))

    def bounds(self) -> np.ndarray:
        """[xmin, ymin, xmax, ymax] as fp64 (the clamp box of gift.py:115-118)."""
        return np.array([self.xmin, self.ymin, self.xmax, self.ymax], dtype=np.float64)


class Design:
    """Object-model design; derived arrays are computed once and cached."""

    def __init__(self, cells: list[Cell], nets: list[Net], region: Region) -> None:
        self.cells = cells
        self.nets = nets
        self.region = region

    @property
    def num_cells(self) -> int:
        return len(self.cells)

    @property
    def num_movable(self) -> int:
        return int(np.count_nonzero(~self.fixed_mask()))

    @property
    def num_fixed(self) -> int:
        return int(np.count_nonzero(self.fixed_mask()))

    def fixed_mask(self) -> np.ndarray:
        mask = getattr(self, "_fixed_mask", None)
        if mask is None:
            mask = np.fromiter((c.fixed for c in self.cells), dtype=bool, count=len(self.cells))
            self._fixed_mask = mask
        return mask

    def fixed_positions(self) -> np.ndarray:
        """N x 2 fp64: fixed centres, NaN on movable rows."""
        pos = getattr(self, "_fixed_pos", None)
        if pos is None:
            pos = np.full((self.num_cells, 2), np.nan)
            for c in self.cells:
                if c.fixed:
                    pos[c.id] = c.fixed_pos
            self._fixed_pos = pos
        return pos.copy()

    def pin_table(self):
        """(net_start int64[E+1], pin_cell int64[P], pin_dx, pin_dy)."""
        tbl = getattr(self, "_pin_table", None)
        if tbl is None:
            counts = np.fromiter((len(n.pins) for n in self.nets), dtype=np.int64, count=len(self.nets))
            net_start = np.zeros(len(self.nets) + 1, dtype=np.int64)
            np.cumsum(counts, out=net_start[1:])
            total = int(net_start[-1])
            pin_cell = np.fromiter((p.cell for n in self.nets for p in n.pins), dtype=np.int64, count=total)
            pin_dx = np.fromiter((p.dx for n in self.nets for p in n.pins), dtype=float, count=total)
            pin_dy = np.fromiter((p.dy for n in self.nets for p in n.pins), dtype=float, count=total)
            tbl = (net_start, pin_cell, pin_dx, pin_dy)
            self._pin_table = tbl
        return tbl

    def validate(self) -> None:
        names = set()
        for i, c in enumerate(self.cells):
            if c.id != i:
                raise GiftPlaceError(f"cell ids not contiguous: cell {c.name!r} has id {c.id} at index {i}")
            if c.name in names:
                raise GiftPlaceError(f"duplicate cell name {c.name!r}")
            names.add(c.name)
            if not (c.width > 0 and c.height > 0):
                raise GiftPlaceError(f"cell {c.name!r} has non-positive dimensions")
            if c.fixed != (c.fixed_pos is not None):
                raise GiftPlaceError(f"cell {c.name!r}: fixed_pos must be present exactly when fixed")
        n = len(self.cells)
        for j, net in enumerate(self.nets):
            if net.id != j:
                raise GiftPlaceError(f"net ids not contiguous at index {j}")
            for p in net.pins:
                if not (0 <= p.cell < n):
                    raise GiftPlaceError(f"net {net.name!r} pin references cell id {p.cell} out of range")
        if not (self.region.xmax > self.region.xmin and self.region.ymax > self.region.ymin):
            raise GiftPlaceError("region must have positive extent")


class FlatDesign:
    """Array-native design with the accessors the hot path reads.

    net_start : int64[E+1]  net e owns pins [net_start[e], net_start[e+1])
    pin_cell  : int32/int64[P] cell id of every pin, in net order
    fixed_mask: bool[N]
    fixed_pos : fp64[N, 2]   fixed centres, NaN on movable rows
    """

    def __init__(self, net_start, pin_cell, fixed_mask, fixed_pos, region: Region,
                 widths=None, heights=None, meta: dict | None = None, pin_dx=None, pin_dy=None,
                 cell_names=None, net_names=None) -> None:
        self.net_start = np.ascontiguousarray(net_start, dtype=np.int64)
        self.pin_cell = np.ascontiguousarray(pin_cell)
        self._mask = np.ascontiguousarray(fixed_mask, dtype=bool)
        self._fixed_pos = np.ascontiguousarray(fixed_pos, dtype=np.float64)
        self.region = region
        n = len(self._mask)
        self.widths = np.ones(n) if widths is None else np.asarray(widths, dtype=float)
        self.heights = np.ones(n) if heights is None else np.asarray(heights, dtype=float)
        self.meta = dict(meta or {})
        # optional (a parsed Bookshelf design has them; synthetic designs do not):
        # pin offsets from the cell centre, and names as (uint8 bytes, int64 offsets)
        self.pin_dx = None if pin_dx is None else np.ascontiguousarray(pin_dx, dtype=np.float64)
        self.pin_dy = None if pin_dy is None else np.ascontiguousarray(pin_dy, dtype=np.float64)
        self.cell_names = cell_names
        self.net_names = net_names

    @property
    def num_cells(self) -> int:
        return len(self._mask)

    @property
    def num_nets(self) -> int:
        return len(self.net_start) - 1

    @property
    def num_pins(self) -> int:
        return int(self.net_start[-1])

    @property
    def num_fixed(self) -> int:
        return int(np.count_nonzero(self._mask))

    @property
    def num_movable(self) -> int:
        return self.num_cells - self.num_fixed

    def fixed_mask(self) -> np.ndarray:
        return self._mask

    def fixed_positions(self) -> np.ndarray:
        return self._fixed_pos.copy()

    def pin_table(self):
        if self.pin_dx is not None:
            return (self.net_start, self.pin_cell, self.pin_dx, self.pin_dy)
        z = np.zeros(self.num_pins)
        return (self.net_start, self.pin_cell, z, z)

    @staticmethod
    def _names(packed, count: int, default: str) -> list[str]:
        if packed is None:
            return [f"{default}{i}" for i in range(count)]
        data, off = packed
        raw = bytes(np.asarray(data, dtype=np.uint8))
        return [raw[off[i]:off[i + 1]].decode() for i in range(count)]

    def cell_name_list(self) -> list[str]:
        """Cell names: parsed ones, else "c<i>" (FlatDesign.to_design / benchgen convention)."""
        return self._names(self.cell_names, self.num_cells, "c")

    def net_name_list(self) -> list[str]:
        return self._names(self.net_names, self.num_nets, "n")

    def to_design(self, module=None) -> Design:
        """Materialise the object model (this package's, or `module`'s classes --
        e.g. the reference's -- when given). O(N+P) Python objects."""
        mod = module
        C = getattr(mod, "Cell", Cell)
        P = getattr(mod, "Pin", Pin)
        Nt = getattr(mod, "Net", Net)
        R = getattr(mod, "Region", Region)
        D = getattr(mod, "Design", Design)
        cells = []
        cnames = self.cell_name_list()
        for i in range(self.num_cells):
            if self._mask[i]:
                cells.append(C(id=i, name=cnames[i], width=float(self.widths[i]), height=float(self.heights[i]),
                               fixed=True, fixed_pos=(float(self._fixed_pos[i, 0]), float(self._fixed_pos[i, 1]))))
            else:
                cells.append(C(id=i, name=cnames[i], width=float(self.widths[i]), height=float(self.heights[i])))
        pc = self.pin_cell.tolist()
        ns = self.net_start.tolist()
        nnames = self.net_name_list()
        if self.pin_dx is not None:
            dx, dy = self.pin_dx.tolist(), self.pin_dy.tolist()
            nets = [Nt(id=e, name=nnames[e], pins=[P(cell=pc[k], dx=dx[k], dy=dy[k]) for k in range(ns[e], ns[e + 1])])
                    for e in range(self.num_nets)]
        else:
            nets = [Nt(id=e, name=nnames[e], pins=[P(cell=c) for c in pc[ns[e]:ns[e + 1]]])
                    for e in range(self.num_nets)]
        r = self.region
        RowC = getattr(mod, "Row", Row)
        rows = [RowC(y=w.y, height=w.height, x=w.x, num_sites=w.num_sites, site_width=w.site_width)
                for w in getattr(r, "rows", [])]
        return D(cells=cells, nets=nets, region=R(r.xmin, r.ymin, r.xmax, r.ymax, rows=rows))


def pin_arrays(design) -> tuple[np.ndarray, np.ndarray]:
    """(net_start int64, pin_cell) from either front door."""
    if isinstance(design, FlatDesign):
        return design.net_start, design.pin_cell
    net_start, pin_cell = design.pin_table()[:2]
    return np.asarray(net_start, dtype=np.int64), np.asarray(pin_cell)
