"""CPU restatement of the reference .pl writer -- TEST INFRASTRUCTURE ONLY.

Restates giftplace/netlist.py:503-522 (`write_placement`, PL_PRECISION = 6 at
:29) on flat arrays: one line per cell in cell order,
name, lower-left x, lower-left y with Python's correctly rounded "%.6f", and
the /FIXED marker.  Python's own float formatting is the arithmetic here (it
is what the reference calls), so this oracle is exact by construction; it is
pinned against the reference's bytes in tests/golden (pl_edge, pl_c0).

Only tests/ and __graft_entry__.smoke() import this module, as the checker.
"""

from __future__ import annotations

import numpy as np

PL_PRECISION = 6


def format_placement(names, widths, heights, fixed, pos) -> bytes:
    """names: list[str]; widths/heights fp64 [n]; fixed bool [n]; pos fp64 [n, 2] centres."""
    out = ["UCLA pl 1.0", ""]
    pos = np.asarray(pos, dtype=np.float64)
    with np.errstate(invalid="ignore"):  # inf - w/2 etc. print as the reference prints them
        for i, name in enumerate(names):
            llx = pos[i, 0] - float(widths[i]) / 2.0   # netlist.py:516-517
            lly = pos[i, 1] - float(heights[i]) / 2.0
            tail = " /FIXED" if fixed[i] else ""       # netlist.py:518
            out.append(f"{name}\t{llx:.{PL_PRECISION}f}\t{lly:.{PL_PRECISION}f}\t: N{tail}")
    return ("\n".join(out) + "\n").encode()


def fmt6(values) -> list[str]:
    """Python's "%.6f" of each fp64 value (the per-number contract)."""
    return [f"{v:.{PL_PRECISION}f}" for v in np.asarray(values, dtype=np.float64).tolist()]
