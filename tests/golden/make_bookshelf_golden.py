"""Bookshelf reader fixtures: design files + what the REFERENCE parser makes of them.

Run in the build container (the reference is importable there):
    python tests/golden/make_bookshelf_golden.py [/root/reference/pkg/src]
Writes tests/golden/bookshelf/<case>/{d.aux,d.nodes,d.nets,d.pl[,d.scl]} and
tests/golden/bookshelf/expected.json (+ expected.npz for the arrays): for every
case either the parsed design (arrays, names, region) or the exception class
and message giftplace.parse_design raises.  The texts are written by this
script (seeded generator + hand-made edge cases); nothing is copied from the
reference's tests.
"""

from __future__ import annotations

import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, ROOT)

import giftplace as gp  # noqa: E402  (the reference)

OUT = os.path.join(HERE, "bookshelf")

NODES = """UCLA nodes 1.0
# generated fixture
NumNodes : 6
NumTerminals : 1

alpha\t2 1
beta 1.5 1   # trailing comment
gamma 1 2.25
delta 3e0 +1
eps .5 5.
io_0 1 1 terminal
"""

NETS = """UCLA nets 1.0
NumNets : 3
NumPins : 8
NetDegree : 3 sig_a
  alpha I : 0.5 -0.25
  beta O
  gamma B : -1 0
NetDegree : 2
  delta I : 1_0.5 2
  io_0 I
NetDegree : 3 sig_c
  eps I : 0 0
  alpha I
  delta I : 0.1 0.2 extra
"""

PL = """UCLA pl 1.0

alpha 0 0 : N
beta 4 0 : N
gamma 0 4 : N
delta 5 5 : N
eps 1 7 : N
io_0 9 9 : N /FIXED
ghost 3 3 : N
beta 4.5 0.5 : N
"""

SCL = """UCLA scl 1.0
NumRows : 2
CoreRow Horizontal
  Coordinate : 0
  Height : 5
  Sitewidth : 1
  SubrowOrigin : 0 NumSites : 10
End
CoreRow Horizontal
  Coordinate : 5
  Height : 5
  Sitewidth : 1
  SubrowOrigin : 0 NumSites : 10
End
"""


def _num(rng, v: float) -> str:
    """A float literal in one of several spellings float() accepts."""
    k = int(rng.integers(0, 8))
    if k == 0:
        return repr(float(v))
    if k == 1:
        return f"{v:.3f}"
    if k == 2:
        return f"{v:e}"
    if k == 3:
        return f"{v:+.6g}"
    if k == 4:
        return f"{v:.25f}"  # > 19 significant digits: host path
    if k == 5:  # PEP 515 separator: float() accepts it, the device defers to the host
        t = f"{v:.4f}"
        i = 1 if t[0] in "+-" else 0
        return t[: i + 1] + "_" + t[i + 1:] if t[i + 1].isdigit() else t
    if k == 6:
        return f"{v:.17g}"
    return f"{v:.1E}"


def synthetic(rng, n_cells: int, n_nets: int, crlf: bool) -> dict[str, str]:
    names = [f"o{i}" if i % 7 else f"cell/{i}[0]" for i in range(n_cells)]
    term = rng.random(n_cells) < 0.03
    w = rng.choice([1.0, 2.0, 0.5, 3.25, 1.125], size=n_cells)
    h = rng.choice([1.0, 2.0, 0.75], size=n_cells)
    nodes = ["UCLA nodes 1.0", f"NumNodes : {n_cells}", f"NumTerminals : {int(term.sum())}"]
    for i in range(n_cells):
        t = " terminal" if term[i] else ""
        nodes.append(f"\t{names[i]}  {_num(rng, w[i])} {_num(rng, h[i])}{t}")
    nets = ["UCLA nets 1.0", f"NumNets : {n_nets}", "NumPins : 0"]
    for e in range(n_nets):
        m = int(rng.integers(0, 7))
        label = f" net_{e}" if rng.random() < 0.7 else ""
        nets.append(f"NetDegree : {m}{label}")
        c = int(rng.integers(0, n_cells))
        for _ in range(m):
            cell = int(np.clip(c + rng.integers(-40, 41), 0, n_cells - 1))
            if rng.random() < 0.5:
                nets.append(f"  {names[cell]} I : {_num(rng, rng.normal())} {_num(rng, rng.normal())}")
            else:
                nets.append(f"  {names[cell]} O")
        if rng.random() < 0.05:
            nets.append("# interleaved comment")
            nets.append("")
    pl = ["UCLA pl 1.0", ""]
    order = rng.permutation(n_cells)
    for i in order:
        fx = " /FIXED" if (term[i] or rng.random() < 0.01) else ""
        pl.append(f"{names[i]} {_num(rng, rng.uniform(0, 900))} {_num(rng, rng.uniform(0, 900))} : N{fx}")
    for i in rng.choice(n_cells, size=n_cells // 20, replace=False):  # re-placed cells: the last line wins
        pl.append(f"{names[i]}\t{_num(rng, rng.uniform(0, 900))}\t{_num(rng, rng.uniform(0, 900))}\t: N")
    nl = "\r\n" if crlf else "\n"
    return {"nodes": nl.join(nodes) + nl, "nets": nl.join(nets) + nl, "pl": nl.join(pl) + nl}


def write_case(name: str, files: dict[str, str]) -> str:
    d = os.path.join(OUT, name)
    os.makedirs(d, exist_ok=True)
    listed = []
    for ext in ("nodes", "nets", "pl", "scl"):
        if ext in files:
            with open(os.path.join(d, f"d.{ext}"), "w", newline="") as f:
                f.write(files[ext])
            listed.append(f"d.{ext}")
    with open(os.path.join(d, "d.aux"), "w") as f:
        f.write("RowBasedPlacement : " + " ".join(listed) + "\n")
    return os.path.join(d, "d.aux")


def variants() -> dict[str, dict[str, str]]:
    base = {"nodes": NODES, "nets": NETS, "pl": PL, "scl": SCL}

    def v(**kw):
        out = dict(base)
        for k, val in kw.items():
            if val is None:
                out.pop(k, None)
            else:
                out[k] = val
        return out

    return {
        "basic": v(),
        "bbox_region": v(scl=None),
        "cr_only_newlines": {k: t.replace("\n", "\r") for k, t in base.items()},
        "nodes_hdr_colon": v(nodes=NODES.replace("NumNodes : 6", "NumNodes 6")),
        "nodes_hdr_int": v(nodes=NODES.replace("NumNodes : 6", "NumNodes : six")),
        "nodes_hdr_underscore": v(nodes=NODES.replace("NumNodes : 6", "NumNodes : 0_6")),
        "nodes_few": v(nodes=NODES.replace("gamma 1 2.25", "gamma 1")),
        "nodes_num": v(nodes=NODES.replace("gamma 1 2.25", "gamma 1 2.2.5")),
        "nodes_pos": v(nodes=NODES.replace("gamma 1 2.25", "gamma 0 2.25")),
        "nodes_nan": v(nodes=NODES.replace("gamma 1 2.25", "gamma nan 2.25")),
        "nodes_dup": v(nodes=NODES.replace("eps .5 5.", "beta .5 5.")),
        "nodes_dup_then_num": v(nodes=NODES.replace("eps .5 5.", "beta .5 5.").replace("io_0 1 1", "io_0 x 1")),
        "nodes_num_then_dup": v(nodes=NODES.replace("beta 1.5 1", "beta 1.5 q").replace("eps .5 5.", "alpha .5 5.")),
        "nodes_count": v(nodes=NODES.replace("NumNodes : 6", "NumNodes : 9")),
        "nodes_header_as_cell": v(nodes=NODES.replace("NumNodes : 6", "NumNodes: 6")),
        "nets_hdr_int": v(nets=NETS.replace("NumPins : 8", "NumPins : eight")),
        "nets_deg_colon": v(nets=NETS.replace("NetDegree : 2\n", "NetDegree 2\n")),
        "nets_deg_int": v(nets=NETS.replace("NetDegree : 2\n", "NetDegree : two\n")),
        "nets_outside": v(nets=NETS.replace("NumPins : 8\n", "NumPins : 8\n  alpha I\n")),
        "nets_too_many": v(nets=NETS.replace("  io_0 I\n", "  io_0 I\n  beta I\n")),
        "nets_prev_missing": v(nets=NETS.replace("  io_0 I\n", "")),
        "nets_last_missing": v(nets=NETS.replace("  delta I : 0.1 0.2 extra\n", "")),
        "nets_negative": v(nets=NETS.replace("NetDegree : 2\n", "NetDegree : -1\n")),
        "nets_zero": v(nets=NETS.replace("NetDegree : 2\n  delta I : 1_0.5 2\n  io_0 I\n", "NetDegree : 0 empty\n")
                       .replace("NumNets : 3", "NumNets : 3")),
        "nets_dangling": v(nets=NETS.replace("  beta O\n", "  nobody O\n")),
        "nets_offsets": v(nets=NETS.replace("gamma B : -1 0", "gamma B : -1 zero")),
        "nets_count": v(nets=NETS.replace("NumNets : 3", "NumNets : 4")),
        "nets_dangling_before_offsets": v(nets=NETS.replace("gamma B : -1 0", "ghost B : -1 zero")),
        "pl_few": v(pl=PL.replace("gamma 0 4 : N", "gamma 0")),
        "pl_num": v(pl=PL.replace("gamma 0 4 : N", "gamma 0 four : N")),
        "pl_fixed_ni": v(pl=PL.replace("gamma 0 4 : N", "gamma 0 4 : N /FIXED_NI")),
        "pl_no_place": v(pl=PL.replace("io_0 9 9 : N /FIXED\n", "")),
        "pl_refix_last_wins": v(pl=PL + "io_0 2 2 : N\nalpha 1 1 : N /FIXED\n"),
        "numbers_slow": v(nodes=NODES.replace("gamma 1 2.25", "gamma 1.0000000000000000000001 2.2500000000000000000000001")
                          .replace("delta 3e0 +1", "delta 3e-30 1e25")),
        "numbers_specials": v(nodes=NODES.replace("gamma 1 2.25", "gamma inf Infinity"),
                              pl=PL.replace("gamma 0 4 : N", "gamma -0 1e-320 : N")),
    }


def expected_of(aux: str):
    try:
        d = gp.parse_design(aux)
    except gp.GiftPlaceError as exc:
        msg = str(exc).replace(OUT, "<DIR>")
        return {"error": type(exc).__name__, "message": msg}, None
    net_start, pin_cell, pin_dx, pin_dy = d.pin_table()
    arrays = {
        "net_start": np.asarray(net_start, np.int64), "pin_cell": np.asarray(pin_cell, np.int64),
        "pin_dx": np.asarray(pin_dx, np.float64), "pin_dy": np.asarray(pin_dy, np.float64),
        "width": np.array([c.width for c in d.cells]), "height": np.array([c.height for c in d.cells]),
        "fixed": d.fixed_mask().astype(np.uint8), "fixed_pos": d.fixed_positions(),
    }
    r = d.region
    meta = {
        "cell_names": [c.name for c in d.cells], "net_names": [n.name for n in d.nets],
        "region": [r.xmin, r.ymin, r.xmax, r.ymax],
        "rows": [[w.y, w.height, w.x, w.num_sites, w.site_width] for w in r.rows],
    }
    return meta, arrays


def main() -> None:
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    cases = variants()
    rng = np.random.default_rng(20261020)
    cases["synth_lf"] = synthetic(rng, 3000, 3200, crlf=False)
    cases["synth_crlf"] = synthetic(rng, 1200, 1000, crlf=True)
    expected, npz = {}, {}
    for name, files in cases.items():
        aux = write_case(name, files)
        meta, arrays = expected_of(aux)
        expected[name] = meta
        if arrays is not None:
            for k, a in arrays.items():
                npz[f"{name}__{k}"] = a
    with open(os.path.join(OUT, "expected.json"), "w") as f:
        json.dump(expected, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(OUT, "expected.npz"), **npz)
    print(f"{len(cases)} cases; errors: {sum('error' in e for e in expected.values())}")


if __name__ == "__main__":
    main()
