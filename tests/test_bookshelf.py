"""Bookshelf reader: parse_design, netlist.py:418-458.

Fixtures in tests/golden/bookshelf/ were parsed by the REFERENCE
(make_bookshelf_golden.py): for each case the design it builds or the exact
exception it raises.  GPU tests run the device reader on the same files.
CPU tests cover the host side (manifest, .scl rows, error mapping).
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BS = os.path.join(HERE, "golden", "bookshelf")


@pytest.fixture(scope="module")
def expected():
    with open(os.path.join(BS, "expected.json")) as f:
        meta = json.load(f)
    return meta, dict(np.load(os.path.join(BS, "expected.npz")))


def _aux(case):
    return os.path.join(BS, case, "d.aux")


def _cases():
    with open(os.path.join(BS, "expected.json")) as f:
        return sorted(json.load(f))


# ------------------------------------------------------------------ CPU --
def test_aux_manifest_errors(tmp_path):
    import paper_2502_17632_b200 as gb

    with pytest.raises(gb.MissingFileError):
        gb.aux_files(str(tmp_path / "none.aux"))
    (tmp_path / "a.nodes").write_text("")
    (tmp_path / "a.nets").write_text("")
    aux = tmp_path / "a.aux"
    aux.write_text("RowBasedPlacement : a.nodes a.nets\n")
    with pytest.raises(gb.MissingFileError, match=r"<\.pl entry in a\.aux>"):
        gb.aux_files(str(aux))
    aux.write_text("RowBasedPlacement : a.nodes a.nets a.pl\n")
    with pytest.raises(gb.MissingFileError, match="a.pl"):
        gb.aux_files(str(aux))
    aux.write_text("just words\n")
    with pytest.raises(gb.MalformedLineError):
        gb.aux_files(str(aux))
    files = gb.aux_files(_aux("basic"))
    assert sorted(files) == [".nets", ".nodes", ".pl", ".scl"]


def test_scl_rows_and_region(expected):
    from paper_2502_17632_b200 import bookshelf

    meta, _ = expected
    rows = bookshelf._parse_scl(os.path.join(BS, "basic", "d.scl"))
    assert [[r.y, r.height, r.x, r.num_sites, r.site_width] for r in rows] == meta["basic"]["rows"]
    r = bookshelf._region_from_rows(rows)
    assert [r.xmin, r.ymin, r.xmax, r.ymax] == meta["basic"]["region"]


# (case, file, lineno, device code, value, text): what the device reports for
# each reference error; the host must raise the reference's class and message
DEVICE_REPORTS = [
    ("nodes_few", 0, 8, 3, 0, "gamma 1"),
    ("nodes_dup", 0, 10, 6, 0, "beta"),
    ("nodes_count", 0, 0, 7, 9, "6"),
    ("nodes_header_as_cell", 0, 3, 3, 0, "NumNodes: 6"),
    ("nodes_hdr_colon", 0, 3, 1, 0, "NumNodes 6"),
    ("nets_prev_missing", 1, 10, 22, 1, "NetDegree : 3 sig_c"),
    ("nets_negative", 1, 11, 22, -3, "NetDegree : 3 sig_c"),
    ("nets_last_missing", 1, 0, 28, 1, ""),
    ("nets_dangling", 1, 6, 26, 0, "nobody"),
    ("nets_count", 1, 0, 29, 4, "3"),
    ("nets_offsets", 1, 7, 27, 0, "gamma B : -1 zero"),
    ("nets_outside", 1, 4, 25, 0, "alpha I"),
    ("pl_no_place", 2, 0, 42, 0, "io_0"),
    ("pl_num", 2, 5, 41, 0, "gamma 0 four : N"),
    ("pl_few", 2, 5, 40, 0, "gamma 0"),
]


@pytest.mark.parametrize("case,file,lineno,code,value,text", DEVICE_REPORTS)
def test_error_messages_map_like_the_reference(expected, case, file, lineno, code, value, text):
    import paper_2502_17632_b200 as gb
    from paper_2502_17632_b200 import bookshelf

    meta, _ = expected
    exp = meta[case]
    d = os.path.join(BS, case)
    paths = [os.path.join(d, "d.nodes"), os.path.join(d, "d.nets"), os.path.join(d, "d.pl")]
    with pytest.raises(getattr(gb, exp["error"])) as exc:
        bookshelf._raise_parse_error(f"{file}\t{lineno}\t{code}\t{value}\t{text}", paths)
    assert str(exc.value).replace(BS, "<DIR>") == exp["message"]


# ------------------------------------------------------------------ GPU --
@pytest.mark.gpu
@pytest.mark.parametrize("case", _cases())
def test_device_reader_matches_reference(expected, case):
    import paper_2502_17632_b200 as gb

    meta, arrays = expected
    exp = meta[case]
    if "error" in exp:
        with pytest.raises(getattr(gb, exp["error"])) as exc:
            gb.read_design(_aux(case))
        assert str(exc.value).replace(BS, "<DIR>") == exp["message"]
        return
    fd = gb.read_design(_aux(case))
    net_start, pin_cell, pin_dx, pin_dy = fd.pin_table()

    def eq(name, got):
        ref = arrays[f"{case}__{name}"]
        got = np.asarray(got, dtype=ref.dtype)
        assert got.shape == ref.shape, name
        if ref.dtype.kind == "f":
            assert np.array_equal(got.view(np.int64), ref.view(np.int64)), name  # bit-exact, NaN payloads too
        else:
            assert np.array_equal(got, ref), name

    eq("net_start", net_start)
    eq("pin_cell", pin_cell)
    eq("pin_dx", pin_dx)
    eq("pin_dy", pin_dy)
    eq("width", fd.widths)
    eq("height", fd.heights)
    eq("fixed", fd.fixed_mask().astype(np.uint8))
    fp = fd.fixed_positions()
    ref_fp = arrays[f"{case}__fixed_pos"]
    assert np.array_equal(np.isnan(fp), np.isnan(ref_fp))
    assert np.array_equal(fp[~np.isnan(fp)], ref_fp[~np.isnan(ref_fp)])
    assert fd.cell_name_list() == exp["cell_names"]
    assert fd.net_name_list() == exp["net_names"]
    r = fd.region
    assert [r.xmin, r.ymin, r.xmax, r.ymax] == exp["region"]
    assert [[w.y, w.height, w.x, w.num_sites, w.site_width] for w in r.rows] == exp["rows"]


@pytest.mark.gpu
def test_parse_design_object_model(expected):
    import paper_2502_17632_b200 as gb

    meta, _ = expected
    d = gb.parse_design(_aux("basic"))
    assert [c.name for c in d.cells] == meta["basic"]["cell_names"]
    assert [n.name for n in d.nets] == meta["basic"]["net_names"]
    assert d.nets[0].pins[0].dx == 0.5 and d.nets[0].pins[0].dy == -0.25
    io = d.cells[meta["basic"]["cell_names"].index("io_0")]
    assert io.fixed and io.fixed_pos == (9.5, 9.5)
    d.validate()


@pytest.mark.gpu
def test_read_then_place_and_write_round_trip(tmp_path):
    """Bookshelf text of a synthetic c1-scale design -> device reader -> the
    same pin table; the parsed design places and writes a .pl that parses back."""
    import paper_2502_17632_b200 as gb
    from paper_2502_17632_b200 import synth

    fd = synth.generate("c1", seed=3, scale=0.25)
    n = fd.num_cells
    names = [f"c{i}" for i in range(n)]
    lines = ["UCLA nodes 1.0", f"NumNodes : {n}"]
    fixed = fd.fixed_mask()
    w, h = fd.widths.tolist(), fd.heights.tolist()
    lines += [f"{names[i]} {w[i]!r} {h[i]!r}{' terminal' if fixed[i] else ''}" for i in range(n)]
    (tmp_path / "d.nodes").write_text("\n".join(lines) + "\n")
    ns, pc = fd.net_start, fd.pin_cell
    out = ["UCLA nets 1.0", f"NumNets : {fd.num_nets}"]
    for e in range(fd.num_nets):
        out.append(f"NetDegree : {ns[e + 1] - ns[e]}")
        out += [f"  {names[c]} I" for c in pc[ns[e]:ns[e + 1]]]
    (tmp_path / "d.nets").write_text("\n".join(out) + "\n")
    fp = fd.fixed_positions()
    fpl = fp.tolist()
    pl = ["UCLA pl 1.0"]
    for i in range(n):
        if fixed[i]:
            pl.append(f"{names[i]} {fpl[i][0] - w[i] / 2!r} {fpl[i][1] - h[i] / 2!r} : N /FIXED")
        else:
            pl.append(f"{names[i]} 0 0 : N")
    (tmp_path / "d.pl").write_text("\n".join(pl) + "\n")
    (tmp_path / "d.aux").write_text("RowBasedPlacement : d.nodes d.nets d.pl\n")
    got = gb.read_design(str(tmp_path / "d.aux"))
    assert np.array_equal(got.net_start, fd.net_start)
    assert np.array_equal(got.pin_cell, fd.pin_cell)
    assert np.array_equal(got.fixed_mask(), fixed)
    half = np.stack([fd.widths / 2.0, fd.heights / 2.0], 1)
    assert np.array_equal(got.fixed_positions()[fixed], ((fp - half) + half)[fixed])  # lower-left + size/2
    adj = gb.build_clique_graph(got)
    placed, _ = gb.gift_place(got, adj, gb.GiftConfig(seed=0, jitter_scale=10.0))
    gb.write_placement(got, placed, str(tmp_path / "out.pl"))
    (tmp_path / "d2.aux").write_text("RowBasedPlacement : d.nodes d.nets out.pl\n")
    again = gb.read_design(str(tmp_path / "d2.aux"))
    # the .pl keeps 6 decimals (PL_PRECISION): fixed centres come back to within 1e-6
    assert np.allclose(again.fixed_positions()[fixed], got.fixed_positions()[fixed], rtol=0, atol=1.0000001e-6)
