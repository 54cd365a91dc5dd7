"""Bookshelf .pl writer: write_placement, netlist.py:503-522.

CPU: the oracle restatement reproduces the reference's bytes (golden pl_edge)
and the host-side column staging.  GPU: gift_format_placement is
byte-identical to the reference on the edge-case design, on config c0's
placement (sha of the reference's file), and to the oracle on random bit
patterns.
"""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest


def _edge_design(gb, golden):
    names = bytes(golden["pl_edge__names"]).decode().split("\n")
    cells = []
    for i, name in enumerate(names):
        fixed = bool(golden["pl_edge__fixed"][i])
        cells.append(gb.Cell(id=i, name=name, width=float(golden["pl_edge__width"][i]),
                             height=float(golden["pl_edge__height"][i]), fixed=fixed,
                             fixed_pos=(0.0, 0.0) if fixed else None))
    return gb.Design(cells=cells, nets=[], region=gb.Region(0.0, 0.0, 10.0, 10.0)), names


def test_oracle_matches_reference_bytes(golden):
    from oracle import pl_oracle

    names = bytes(golden["pl_edge__names"]).decode().split("\n")
    text = pl_oracle.format_placement(names, golden["pl_edge__width"], golden["pl_edge__height"],
                                      golden["pl_edge__fixed"].astype(bool), golden["pl_edge__pos"])
    assert text == bytes(golden["pl_edge__text"])


def test_host_columns(golden):
    import paper_2502_17632_b200 as gb
    from paper_2502_17632_b200 import plio, synth

    d, names = _edge_design(gb, golden)
    w, h, fx, nb, off, prefix, rows = plio._columns(d)
    assert rows is None and prefix == b""
    assert bytes(nb) == "".join(names).encode()
    assert off[-1] == len(bytes(nb)) and np.all(np.diff(off) >= 0)
    assert np.array_equal(fx, golden["pl_edge__fixed"])
    # cells listed out of id order: rows follow cell.id (netlist.py:515)
    d.cells = d.cells[::-1]
    assert np.array_equal(plio._columns(d)[6], np.arange(len(names))[::-1])
    fd = synth.generate("c0", seed=1, scale=0.05)
    w, h, fx, nb, off, prefix, rows = plio._columns(fd)
    assert nb is None and prefix == b"c" and fx.sum() == fd.num_fixed


def test_shape_mismatch_raises_before_device(golden):
    import paper_2502_17632_b200 as gb

    d, _ = _edge_design(gb, golden)
    with pytest.raises(gb.GiftPlaceError):
        gb.format_placement(d, np.zeros((3, 2)))


@pytest.mark.gpu
def test_edge_cases_byte_identical(golden, tmp_path):
    import paper_2502_17632_b200 as gb

    d, _ = _edge_design(gb, golden)
    ref = bytes(golden["pl_edge__text"])
    assert gb.format_placement(d, golden["pl_edge__pos"]) == ref
    path = os.path.join(tmp_path, "edge.pl")
    gb.write_placement(d, golden["pl_edge__pos"], path)
    assert open(path, "rb").read() == ref
    # out-of-order cell list: same rows by id, lines in list order
    d.cells = d.cells[::-1]
    from oracle import pl_oracle

    pos = golden["pl_edge__pos"]
    exp = pl_oracle.format_placement([c.name for c in d.cells], [c.width for c in d.cells],
                                     [c.height for c in d.cells], [c.fixed for c in d.cells],
                                     pos[[c.id for c in d.cells]])
    assert gb.format_placement(d, pos) == exp


@pytest.mark.gpu
def test_c0_placement_file_matches_reference(golden_meta):
    import paper_2502_17632_b200 as gb
    from paper_2502_17632_b200 import synth

    meta = golden_meta["cases"]["pl_c0"]
    fd = synth.generate("c0", seed=1)
    adj = gb.build_clique_graph(fd, max_clique_pins=fd.meta["max_clique_pins"])
    placed, _ = gb.gift_place(fd, adj, gb.GiftConfig(seed=0, jitter_scale=10.0, precision="fp64"))
    text = gb.format_placement(fd, placed)  # generated "c<i>" names
    assert len(text) == meta["bytes"]
    assert hashlib.sha256(text).hexdigest() == meta["sha"]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1])
def test_random_bit_patterns_match_python_formatting(seed):
    import paper_2502_17632_b200 as gb
    from oracle import pl_oracle

    rng = np.random.default_rng(seed)
    n = 60000
    raw = rng.integers(0, 2**63, size=n, dtype=np.uint64) | (rng.integers(0, 2, size=n, dtype=np.uint64) << 63)
    v = raw.view(np.float64).copy()
    v[~(np.abs(v) < 2.0 ** 100) & np.isfinite(v)] = 1.0  # keep the exact range
    mags = rng.normal(size=n) * 10.0 ** rng.integers(-8, 16, size=n)
    ties = (rng.integers(-10**9, 10**9, size=n) + 0.5) / 2.0 ** rng.integers(0, 20, size=n)
    pos = np.stack([np.concatenate([v, mags, ties])[: 3 * n], np.roll(np.concatenate([v, mags, ties]), 7)], 1)
    pos = pos.reshape(-1, 2)
    m = pos.shape[0]
    w = rng.choice([0.0, 1.0, 2.0, 0.5, 3.0], size=m)
    h = rng.choice([0.0, 1.0, 0.25], size=m)
    fixed = rng.random(m) < 0.1
    fd = gb.FlatDesign(np.zeros(1, np.int64), np.zeros(0, np.int64), fixed, np.zeros((m, 2)),
                       gb.Region(0.0, 0.0, 1.0, 1.0), widths=w, heights=h)
    got = gb.format_placement(fd, pos)
    exp = pl_oracle.format_placement([f"c{i}" for i in range(m)], w, h, fixed, pos)
    if got != exp:
        gl, el = got.split(b"\n"), exp.split(b"\n")
        bad = [i for i in range(min(len(gl), len(el))) if gl[i] != el[i]][:3]
        pytest.fail(f"{len(bad)}+ lines differ, e.g. {[(gl[i], el[i]) for i in bad]}")


@pytest.mark.gpu
def test_empty_and_range_errors():
    import paper_2502_17632_b200 as gb

    d = gb.Design(cells=[], nets=[], region=gb.Region(0.0, 0.0, 1.0, 1.0))
    assert gb.format_placement(d, np.zeros((0, 2))) == b"UCLA pl 1.0\n\n"
    d = gb.Design(cells=[gb.Cell(id=0, name="a", width=1.0, height=1.0)], nets=[],
                  region=gb.Region(0.0, 0.0, 1.0, 1.0))
    with pytest.raises(ValueError):
        gb.format_placement(d, np.array([[1e40, 0.0]]))
    assert gb.format_placement(d, np.array([[0.5, 0.5]])) == b"UCLA pl 1.0\n\na\t0.000000\t0.000000\t: N\n"
