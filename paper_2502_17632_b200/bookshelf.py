"""Bookshelf reader: parse_design on the device.

    read_design(aux_path)  -> FlatDesign   array-native, names + pin offsets kept
    parse_design(aux_path) -> Design       the reference's object model (netlist.py:418-458)
    aux_files(aux_path)                    netlist.py:389-415

The .nodes / .nets / .pl texts are parsed by `gift_bookshelf_parse`
(csrc/bookshelf.cu, one thread per line, scans for the sequential parts) with
the reference's semantics and its first-error-in-line-order behaviour; the
.aux manifest and the .scl rows (a few thousand lines at most) are read here
on the host.  Errors are the reference's classes with its messages
(errors.py:14-47).
"""

from __future__ import annotations

import ctypes
import logging
import os

import numpy as np

from . import _lib
from .errors import (
    DanglingPinError,
    DuplicateCellError,
    GiftPlaceError,
    MalformedLineError,
    MissingFileError,
)
from .netlist import Design, FlatDesign, Region, Row

log = logging.getLogger(__name__)

GIFT_ERR_PARSE = 9

# device error codes (csrc/bookshelf.cu enum) -> reference reason strings
_REASON = {
    1: "header missing ':'",                                   # netlist.py:224
    2: "header count is not an integer",                       # :228
    3: "expected 'name width height [terminal]'",              # :236
    4: "width/height are not numbers",                         # :242
    5: "width/height must be positive",                        # :244
    20: "header missing ':'",                                  # :263
    21: "header count is not an integer",                      # :267
    23: "NetDegree missing ':'",                               # :277
    24: "NetDegree count is not an integer",                   # :282
    25: "pin line outside a NetDegree block",                  # :288
    27: "pin offsets are not numbers",                         # :301
    40: "expected 'name x y [: orient] [/FIXED]'",             # :319
    41: "coordinates are not numbers",                         # :325
}


class _Record:
    """One data line of a Bookshelf text: comment cut at '#', stripped; blank
    lines and UCLA banners never become records (netlist.py:193-203)."""

    __slots__ = ("lineno", "text", "tokens")

    def __init__(self, lineno: int, text: str):
        self.lineno = lineno
        self.text = text
        self.tokens = text.split()

    @property
    def value(self) -> str | None:
        """Text after the first ':' of a 'Key : value' header, stripped (None: no colon)."""
        head, colon, tail = self.text.partition(":")
        return tail.strip() if colon else None


def _records(path: str):
    with open(path, "r") as f:
        for lineno, raw in enumerate(f, start=1):
            text = raw.partition("#")[0].strip()
            if text and not text.startswith("UCLA"):
                yield _Record(lineno, text)


# .aux entries by extension: required ones, and the optional placement rows
_AUX_REQUIRED = (".nodes", ".nets", ".pl")
_AUX_KNOWN = frozenset(_AUX_REQUIRED + (".scl",))


def aux_files(aux_path: str) -> dict[str, str]:
    """{extension: path} from the .aux manifest (netlist.py:389-415 semantics):
    every record is 'Tag : file ...'; .nodes/.nets/.pl are required, .scl is
    optional, other files are skipped with a warning, listed files must exist."""
    if not os.path.isfile(aux_path):
        raise MissingFileError(aux_path)
    base = os.path.dirname(os.path.abspath(aux_path))
    listed: list[str] = []
    for rec in _records(aux_path):
        if rec.value is None:
            raise MalformedLineError(aux_path, rec.lineno, rec.text, "expected 'Tag : file ...'")
        listed += rec.value.split()
    found: dict[str, str] = {}
    for fname in listed:
        ext = os.path.splitext(fname)[1]
        if ext not in _AUX_KNOWN:
            log.warning("%s: unsupported file %s skipped", aux_path, fname)
            continue
        path = os.path.join(base, fname)
        if not os.path.isfile(path):
            raise MissingFileError(path)
        found[ext] = path
    missing = [ext for ext in _AUX_REQUIRED if ext not in found]
    if missing:
        raise MissingFileError(os.path.join(base, f"<{missing[0]} entry in {os.path.basename(aux_path)}>"))
    return found


def _subrow_origin(rec: _Record) -> dict[str, float]:
    """'SubrowOrigin : x [NumSites : s]' -> {"x": .., "num_sites": ..}."""
    words = rec.text.replace(":", " ").split()
    got = {"x": float(words[1])}
    if "NumSites" in words:
        got["num_sites"] = float(words[words.index("NumSites") + 1])
    return got


# attributes of a CoreRow block: keyword -> fields it sets (netlist.py:330-370 semantics)
_ROW_ATTRS = {
    "Coordinate": lambda rec: {"y": float(rec.value)},
    "Height": lambda rec: {"height": float(rec.value)},
    "Sitewidth": lambda rec: {"site_width": float(rec.value)},
    "SubrowOrigin": _subrow_origin,
}
_ROW_NEEDS = frozenset(("y", "height", "x", "num_sites"))


def _parse_scl(path: str) -> list[Row]:
    """CoreRow ... End blocks of a .scl file -> Rows.  Lines outside a block
    are ignored; inside, 'Key : value' attributes from _ROW_ATTRS are read
    (others and colon-less lines ignored, a bad number is a
    MalformedLineError); a block missing any of y / height / x / num_sites is
    skipped with a warning; site width defaults to 1."""
    rows: list[Row] = []
    block: dict[str, float] | None = None
    for rec in _records(path):
        key = rec.tokens[0]
        if key == "CoreRow":
            block = {"site_width": 1.0}
        elif block is None:
            continue
        elif key == "End":
            if _ROW_NEEDS <= block.keys():
                rows.append(Row(y=block["y"], height=block["height"], x=block["x"],
                                num_sites=int(block["num_sites"]), site_width=block["site_width"]))
            else:
                log.warning("%s:%d: incomplete CoreRow block skipped", path, rec.lineno)
            block = None
        elif rec.value is not None and key in _ROW_ATTRS:
            try:
                block.update(_ROW_ATTRS[key](rec))
            except (ValueError, IndexError):
                raise MalformedLineError(path, rec.lineno, rec.text, "malformed row attribute") from None
    return rows


def _region_from_rows(rows: list[Row]) -> Region:
    """Bounding box of the rows (netlist.py:373-378)."""
    xs = [(r.x, r.x + r.num_sites * r.site_width) for r in rows]
    ys = [(r.y, r.y + r.height) for r in rows]
    return Region(xmin=min(x0 for x0, _ in xs), ymin=min(y0 for y0, _ in ys),
                  xmax=max(x1 for _, x1 in xs), ymax=max(y1 for _, y1 in ys), rows=rows)


def _raise_parse_error(msg: str, paths: list[str]) -> None:
    file_s, lineno_s, code_s, value_s, text = msg.split("\t", 4)
    path = paths[int(file_s)]
    lineno, code, value = int(lineno_s), int(code_s), int(value_s)
    if code == 6:
        raise DuplicateCellError(path, lineno, text)
    if code == 26:
        raise DanglingPinError(path, lineno, text)
    if code == 7:
        raise MalformedLineError(path, 0, f"NumNodes : {value}", f"header declares {value} nodes, body has {text}")
    if code == 29:
        raise MalformedLineError(path, 0, f"NumNets : {value}", f"header declares {value} nets, body has {text}")
    if code == 22:
        raise MalformedLineError(path, lineno, text, f"previous net is missing {value} pin line(s)")
    if code == 28:
        raise MalformedLineError(path, 0, "", f"last net is missing {value} pin line(s)")
    if code == 42:
        raise MalformedLineError(path, 0, text, "fixed cell has no placement")
    if code == 61:
        raise MalformedLineError(path, lineno, text, "integer outside the int64 range of the device reader")
    if code in _REASON:
        raise MalformedLineError(path, lineno, text, _REASON[code])
    raise GiftPlaceError(f"{path}:{lineno}: Bookshelf parse error {code}: {text!r}")


def _read(path: str) -> bytes:
    with open(path, "rb") as f:
        return f.read()


def read_design(aux_path: str) -> FlatDesign:
    """Parse a .aux manifest and its files into an array-native FlatDesign.

    Same classification, positions, region and errors as the reference's
    parse_design (netlist.py:418-458); the cell / net names and pin offsets
    are kept, so `to_design()` rebuilds the reference's object model.
    """
    by_ext = aux_files(aux_path)
    paths = [by_ext[".nodes"], by_ext[".nets"], by_ext[".pl"]]
    texts = [_read(p) for p in paths]
    lib = _lib.load_library()
    ctx = _lib.context()
    handle = ctypes.c_void_p()
    status = lib.gift_bookshelf_parse(ctx, texts[0], len(texts[0]), texts[1], len(texts[1]), texts[2],
                                      len(texts[2]), ctypes.byref(handle))
    if status == GIFT_ERR_PARSE:
        _raise_parse_error((lib.gift_last_error() or b"").decode(errors="replace"), paths)
    _lib.check(status)
    try:
        sizes = (ctypes.c_int64 * 10)()
        bbox = (ctypes.c_double * 4)()
        _lib.check(lib.gift_bookshelf_info(handle, sizes, bbox))
        n, e, p, n_fixed, n_term, cnb, nnb, unknown, n_placed = list(sizes)[:9]
        net_start = np.empty(e + 1, np.int64)
        pin_cell = np.empty(p, np.int32)
        pin_dx = np.empty(p)
        pin_dy = np.empty(p)
        w = np.empty(n)
        h = np.empty(n)
        fixed = np.empty(n, np.uint8)
        fixed_pos = np.empty((n, 2))
        cnames = np.empty(max(cnb, 1), np.uint8)
        coff = np.empty(n + 1, np.int64)
        nnames = np.empty(max(nnb, 1), np.uint8)
        noff = np.empty(e + 1, np.int64)

        def ptr(a):
            return a.ctypes.data_as(ctypes.c_void_p)

        _lib.check(lib.gift_bookshelf_copy(ctx, handle, ptr(net_start), ptr(pin_cell), ptr(pin_dx), ptr(pin_dy),
                                           ptr(w), ptr(h), ptr(fixed), ptr(fixed_pos), ptr(cnames), ptr(coff),
                                           ptr(nnames), ptr(noff)))
    finally:
        lib.gift_bookshelf_destroy(ctx, handle)
    if unknown:
        log.warning("%s: placement for %d undeclared cell(s) skipped", by_ext[".pl"], unknown)
    if n_term >= 0 and n_term != n_fixed:
        log.warning("%s: NumTerminals declares %d but %d cells are fixed", by_ext[".nodes"], n_term, n_fixed)
    rows = _parse_scl(by_ext[".scl"]) if ".scl" in by_ext else []
    bad = np.flatnonzero(~((w > 0) & (h > 0)))  # NaN sizes pass the parser, not validate() (netlist.py:177-178)
    if rows:
        region = _region_from_rows(rows)
    else:
        xmin, ymin, xmax, ymax = list(bbox)
        if n_placed == 0 or xmax <= xmin or ymax <= ymin:  # netlist.py:461-476
            log.warning("degenerate placement bounding box; using unit region")
            region = Region(0.0, 0.0, 1.0, 1.0)
        else:
            region = Region(xmin, ymin, xmax, ymax)
        log.warning("%s: no usable .scl; region set to placement bounding box", aux_path)
    if bad.size:
        name = bytes(cnames[coff[bad[0]]:coff[bad[0] + 1]]).decode()
        raise GiftPlaceError(f"cell {name!r} has non-positive dimensions")
    if not (region.xmax > region.xmin and region.ymax > region.ymin):  # Design.validate, netlist.py:189-190
        raise GiftPlaceError("region must have positive extent")
    return FlatDesign(net_start, pin_cell, fixed.astype(bool), fixed_pos, region, widths=w, heights=h,
                      meta={"source": os.path.abspath(aux_path)}, pin_dx=pin_dx, pin_dy=pin_dy,
                      cell_names=(cnames[:cnb], coff), net_names=(nnames[:nnb], noff))


def parse_design(aux_path: str, module=None) -> Design:
    """The reference's object model (or `module`'s classes) from the device parse."""
    return read_design(aux_path).to_design(module)
