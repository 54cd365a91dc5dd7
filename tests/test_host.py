"""CPU: host-side logic -- the synthetic generator's contract, the config and
term validation, the seed signal (numpy stream identical to the reference's
gift.py:54-70), and the design front doors."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2502_17632_b200 as gb
from paper_2502_17632_b200 import synth


@pytest.mark.parametrize("config", ["c0", "c1"])
def test_generator_contract(config):
    cfg = synth.CONFIGS[config]
    fd = synth.generate(config, seed=3)
    assert fd.num_cells == cfg["n_mov"] + cfg["n_pads"] + cfg["n_macros"]
    assert fd.num_nets == cfg["n_nets"]
    ns, pc = fd.net_start, fd.pin_cell
    m = np.diff(ns)
    n_mov = cfg["n_mov"]
    mov = pc < n_mov
    e = np.repeat(np.arange(len(m)), m)
    mov_cnt = np.bincount(e[mov], minlength=len(m))
    lo, hi = min(b[0] for b in cfg["bins"]), max(b[1] for b in cfg["bins"])
    assert mov_cnt.min() >= lo and mov_cnt.max() <= hi
    # distinct movable cells per net
    key = e[mov].astype(np.int64) * (fd.num_cells + 1) + pc[mov]
    assert len(np.unique(key)) == len(key)
    # locality window: movable cells of a net span <= 2W
    span = np.zeros(len(m), dtype=np.int64)
    np.maximum.at(span, e[mov], pc[mov])
    mn = np.full(len(m), n_mov, dtype=np.int64)
    np.minimum.at(mn, e[mov], pc[mov])
    assert (span - mn).max() <= 2 * cfg["window"]
    # ~5% of nets carry one pad, as their last pin
    has_pad = (pc[ns[1:] - 1] >= n_mov)
    assert abs(has_pad.mean() - 0.05) < 0.01
    assert (pc[~mov] >= n_mov).all() and (pc < fd.num_cells).all()
    # bin mix
    probs = np.array([b[2] for b in cfg["bins"]])
    counts = [np.count_nonzero((mov_cnt >= b[0]) & (mov_cnt <= b[1])) for b in cfg["bins"]]
    assert np.allclose(np.array(counts) / len(m), probs, atol=0.01)
    # pads fixed on the die boundary ring
    pos = fd.fixed_positions()
    assert np.isnan(pos[:n_mov]).all() and not np.isnan(pos[n_mov:]).any()
    die = fd.meta["die"]
    p = pos[n_mov:]
    on_edge = (np.isclose(p[:, 0], 0.5) | np.isclose(p[:, 0], die - 0.5) | np.isclose(p[:, 1], 0.5)
               | np.isclose(p[:, 1], die - 0.5))
    assert on_edge.all()


def test_generator_is_deterministic_and_seeded():
    a = synth.generate("c0", seed=5)
    b = synth.generate("c0", seed=5)
    c = synth.generate("c0", seed=6)
    assert np.array_equal(a.pin_cell, b.pin_cell) and np.array_equal(a.net_start, b.net_start)
    assert not np.array_equal(a.pin_cell[:1000], c.pin_cell[:1000])


def test_macros_config_scaled():
    fd = synth.generate("c3", seed=1, scale=0.01)
    n_mov, n_mac = fd.meta["n_mov"], fd.meta["n_macros"]
    assert n_mac == 80
    pc = fd.pin_cell
    macro_pins = pc[(pc >= n_mov) & (pc < n_mov + n_mac)]
    per_macro = np.bincount(macro_pins - n_mov, minlength=n_mac)
    assert per_macro.min() >= 10 and per_macro.max() <= 50
    pos = fd.fixed_positions()[n_mov:n_mov + n_mac]
    assert np.isfinite(pos).all()


def test_filter_term_and_config_validation():
    with pytest.raises(ValueError):
        gb.FilterTerm(sigma=2.0, k=0, alpha=0.1)
    with pytest.raises(ValueError):
        gb.FilterTerm(sigma=-1.0, k=2, alpha=0.1)
    with pytest.raises(ValueError):
        gb.GiftConfig(terms=())
    with pytest.raises(ValueError):
        gb.GiftConfig(precision="bf16")
    assert [(t.sigma, t.k, t.alpha) for t in gb.DEFAULT_TERMS] == [(2.0, 2, 0.1), (4.0, 2, 0.7), (4.0, 4, 0.2)]


def anchored():
    cells = [
        gb.Cell(id=0, name="p_left", width=1.0, height=1.0, fixed=True, fixed_pos=(1.0, 2.0)),
        gb.Cell(id=1, name="m0", width=1.0, height=1.0),
        gb.Cell(id=2, name="m1", width=1.0, height=1.0),
        gb.Cell(id=3, name="p_right", width=1.0, height=1.0, fixed=True, fixed_pos=(11.0, 2.0)),
    ]
    nets = [gb.Net(id=0, name="n0", pins=[gb.Pin(0), gb.Pin(1)]), gb.Net(id=1, name="n1", pins=[gb.Pin(1), gb.Pin(2)]),
            gb.Net(id=2, name="n2", pins=[gb.Pin(2), gb.Pin(3)])]
    d = gb.Design(cells=cells, nets=nets, region=gb.Region(0.0, 0.0, 12.0, 4.0))
    d.validate()
    return d


def test_initial_signal_semantics():
    d = anchored()
    g = gb.initial_signal(d, gb.GiftConfig(seed=3))
    assert g[0].tolist() == [1.0, 2.0] and g[3].tolist() == [11.0, 2.0]
    z = gb.initial_signal(d, gb.GiftConfig(seed=3, jitter_scale=0.0))
    assert np.all(z[1:3] == np.array(d.region.center))
    assert np.array_equal(gb.initial_signal(d, gb.GiftConfig(seed=11)), gb.initial_signal(d, gb.GiftConfig(seed=11)))
    # movable jitter independent of which cells are fixed (gift.py:64-69)
    free = gb.Design([gb.Cell(id=c.id, name=c.name, width=1.0, height=1.0) for c in d.cells], d.nets, d.region)
    assert np.array_equal(gb.initial_signal(d, gb.GiftConfig(seed=5))[1:3],
                          gb.initial_signal(free, gb.GiftConfig(seed=5))[1:3])
    # default scale = 0.25 * min(w, h), numpy default_rng stream
    rng = np.random.default_rng(7)
    want = np.tile(d.region.center, (4, 1)) + rng.standard_normal((4, 2)) * 0.25 * 4.0
    want[[0, 3]] = [[1.0, 2.0], [11.0, 2.0]]
    assert np.array_equal(gb.initial_signal(d, gb.GiftConfig(seed=7)), want)


def test_flat_and_object_designs_agree():
    fd = synth.generate("c0", seed=2, scale=0.05)
    d = fd.to_design()
    ns, pc, _, _ = d.pin_table()
    assert np.array_equal(ns, fd.net_start) and np.array_equal(pc, fd.pin_cell)
    assert np.array_equal(d.fixed_mask(), fd.fixed_mask())
    assert np.array_equal(np.nan_to_num(d.fixed_positions(), nan=-1), np.nan_to_num(fd.fixed_positions(), nan=-1))
    assert np.array_equal(gb.initial_signal(d, gb.GiftConfig(seed=1)), gb.initial_signal(fd, gb.GiftConfig(seed=1)))
    assert d.num_fixed == fd.num_fixed and d.num_movable == fd.num_movable


def test_design_validation():
    with pytest.raises(gb.GiftPlaceError):
        gb.Design([gb.Cell(id=1, name="a", width=1, height=1)], [], gb.Region(0, 0, 1, 1)).validate()
    with pytest.raises(gb.GiftPlaceError):
        gb.Design([gb.Cell(id=0, name="a", width=1, height=1)], [gb.Net(0, "n", [gb.Pin(3)])],
                  gb.Region(0, 0, 1, 1)).validate()


def test_kernel_options_are_validated_and_restored():
    """_lib.set_option / options(): unknown names fail; values are kept for
    contexts created later and restored by the context manager."""
    from paper_2502_17632_b200 import _lib

    with pytest.raises(ValueError):
        _lib.set_option("no_such_option", 1)
    before = dict(_lib._options)
    with _lib.options(tile_rows=4096, graphs=0):
        assert _lib._options["tile_rows"] == 4096 and _lib._options["graphs"] == 0
    assert _lib._options == before
    assert set(_lib.DEFAULT_OPTIONS) >= {"tiled", "tile_rows", "col_bits", "fused", "graphs", "zero_copy", "balance",
                                         "implicit_above"}


def test_factored_model_arguments_are_checked_before_any_device_work():
    """implicit_above below 2 (or high_fanout='implicit' without a cap) is a
    ValueError on any machine; so is the same argument of gift_place_arrays."""
    from paper_2502_17632_b200 import synth

    fd = synth.generate("c0", seed=1, scale=0.02)
    for bad in (1, 0, -3):
        with pytest.raises(ValueError):
            gb.build_clique_graph(fd, implicit_above=bad)
        with pytest.raises(ValueError):
            gb.gift_place_arrays(fd.net_start, fd.pin_cell, np.zeros((fd.num_cells, 2), np.float32), fd.fixed_mask(),
                                 fd.fixed_positions(), fd.region.bounds(), implicit_above=bad)
    with pytest.raises(ValueError):
        gb.build_clique_graph(fd, high_fanout="implicit", implicit_above=4)


def test_peer_exchange_pull_tables():
    """PeerExchange._finish_tables: every ghost id maps to (owner rank, row in
    the owner's block); owners hold contiguous row ranges."""
    from paper_2502_17632_b200 import shard

    class Be:
        def upload(self, a):
            return np.asarray(a)

    bounds = np.array([0, 10, 25, 40])
    ghosts = np.array([0, 9, 25, 39])
    plan = shard.ShardPlan(3, 1, bounds, 10, 25, ghosts, [2, 0, 2], [0, 0, 0], np.zeros(0, np.int64))
    ex = shard.PeerExchange.__new__(shard.PeerExchange)
    ex._finish_tables(Be(), plan)
    assert ex.src_rank.tolist() == [0, 0, 2, 2]
    assert ex.src_row.tolist() == [0, 9, 0, 14]


def test_gift_config_output_dtype():
    assert gb.GiftConfig().output_dtype == "float64"
    assert gb.GiftConfig(output_dtype="float32").output_dtype == "float32"
    with pytest.raises(ValueError):
        gb.GiftConfig(output_dtype="float16")


def test_exchange_plan_groups_ghosts_by_owner():
    """shard.exchange_plan: ghosts are requested from the rank owning them,
    and the rows a rank is asked for come back as local row ids."""
    from paper_2502_17632_b200 import shard

    bounds = np.array([0, 10, 25, 40])
    asked_of = {}

    def fake_ids(requests):  # rank 1's all-to-all: echo what others would ask of it
        asked_of["req"] = requests
        return [np.array([10, 12]), np.zeros(0, np.int64), np.array([24])]

    plan = shard.exchange_plan(bounds, 1, np.array([3, 9, 30, 31]), fake_ids)
    assert (plan.r0, plan.r1) == (10, 25)
    assert plan.recv_counts == [2, 0, 2]
    assert [list(r) for r in asked_of["req"]] == [[3, 9], [], [30, 31]]
    assert plan.send_counts == [2, 0, 1] and list(plan.send_rows) == [0, 2, 14]
    assert plan.n_local == 15 and plan.n_ghost == 4


def test_split_block_host_restatement():
    from paper_2502_17632_b200 import shard

    # 4 x 4 symmetric pattern; rows [1, 3) own columns 1, 2
    indptr = np.array([0, 2, 5, 7, 8])
    indices = np.array([1, 3, 0, 2, 3, 1, 3, 0])
    ghosts, loc, gh = shard.split_block(indptr, indices, 1, 3)
    assert list(ghosts) == [0, 3]
    assert list(loc[0]) == [0, 1, 2] and list(loc[1]) == [1, 0] and list(loc[2]) == [3, 5]
    assert list(gh[0]) == [0, 2, 3] and list(gh[1]) == [2, 3, 3] and list(gh[2]) == [2, 4, 6]
