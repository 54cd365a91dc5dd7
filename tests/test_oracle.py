"""CPU: the oracle (oracle/gift_oracle.c) pinned against the reference.

Every golden vector in tests/golden/ was produced by the reference itself
(tests/golden/make_golden.py imports giftplace); here the oracle must
reproduce each bit for bit.  The introsort restatement is also checked
permutation-for-permutation against this toolchain's libstdc++ std::sort,
including adversarial inputs that force its heapsort fallback.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import assert_bits_equal

NETLIST_CASES = ["kat_two_pin", "kat_three_pin", "kat_parallel", "kat_degenerate", "kat_self_pairs",
                 "kat_cap", "kat_tri", "kat_brute", "dupnets"]
COO_CASES = ["rand_graph0", "rand_graph1", "rand_graph2", "rand_coo0", "rand_coo1", "rand_coo2", "adversary"]
DEFAULT = [(2.0, 2, 0.1), (4.0, 2, 0.7), (4.0, 4, 0.2)]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", NETLIST_CASES)
def test_clique_graph_matches_reference(orc, golden, case):
    n, cap = (int(x) for x in golden[f"{case}__n"])
    A = orc.build_clique_graph(n, golden[f"{case}__net_start"], golden[f"{case}__pin_cell"],
                               None if cap < 0 else cap)
    assert np.array_equal(A.indptr, golden[f"{case}__indptr"])
    assert np.array_equal(A.indices, golden[f"{case}__indices"])
    assert_bits_equal(A.data, golden[f"{case}__values"], f"{case} values")
    assert_bits_equal(orc.degrees(A), golden[f"{case}__degrees"], f"{case} degrees")
    for sigma in (0.0, 1.0, 2.0, 4.0):
        key = f"{case}__norm{sigma:g}"
        if f"{key}__isolated" in golden:
            with pytest.raises(LookupError) as exc:
                orc.normalized(A, sigma)
            assert exc.value.args[0] == int(golden[f"{key}__isolated"][0])
            continue
        op = orc.normalized(A, sigma)
        assert np.array_equal(op.indptr, golden[f"{key}__indptr"])
        assert np.array_equal(op.indices, golden[f"{key}__indices"])
        assert_bits_equal(op.data, golden[f"{key}__values"], key)
    if f"{case}__filter" in golden:
        assert_bits_equal(orc.gift_filter(A, golden[f"{case}__g"], DEFAULT), golden[f"{case}__filter"], case)


@pytest.mark.parametrize("case", COO_CASES)
def test_from_coo_matches_reference(orc, golden, case):
    coo = golden[f"{case}__coo"]
    n = int(golden[f"{case}__n"][0])
    A = orc.coo_to_csr(n, coo[0].astype(np.int64), coo[1].astype(np.int64), coo[2])
    assert np.array_equal(A.indptr, golden[f"{case}__indptr"])
    assert np.array_equal(A.indices, golden[f"{case}__indices"])
    assert_bits_equal(A.data, golden[f"{case}__values"], case)
    if f"{case}__degrees" in golden:
        assert_bits_equal(orc.degrees(A), golden[f"{case}__degrees"], f"{case} degrees")
    if f"{case}__filter" in golden:
        g = golden[f"{case}__g"]
        assert_bits_equal(orc.gift_filter(A, g, DEFAULT), golden[f"{case}__filter"], case)
        assert_bits_equal(orc.gift_filter(A, g, [(1.0, 1, 0.5), (1.0, 3, 0.5)]),
                          golden[f"{case}__filter_custom"], case)
        op = orc.normalized(A, 4.0)
        p = g
        for _ in range(3):
            p = orc.matmul(op, p)
        assert_bits_equal(p, golden[f"{case}__pow3"], case)


def test_adversary_exercises_heapsort(orc, golden):
    coo = golden["adversary__coo"]
    before = orc.heapsort_calls()
    orc.coo_to_csr(int(golden["adversary__n"][0]), coo[0].astype(np.int64), coo[1].astype(np.int64), coo[2])
    assert orc.heapsort_calls() > before


def test_order_sensitivity_is_real(orc, golden):
    """The dupnets case is meaningful: summing duplicates in stable emission
    order (what a naive radix sort gives) does NOT reproduce the reference."""
    ns, pc = golden["dupnets__net_start"], golden["dupnets__pin_cell"]
    rows, cols, vals = [], [], []
    for e in range(len(ns) - 1):
        cells = pc[ns[e]:ns[e + 1]]
        m = len(cells)
        for p in range(m):
            for q in range(p + 1, m):
                if cells[p] != cells[q]:
                    rows.append(min(cells[p], cells[q]))
                    cols.append(max(cells[p], cells[q]))
                    vals.append(2.0 / m)
    order = np.lexsort((np.arange(len(rows)), cols, rows))
    r, c, v = np.array(rows)[order], np.array(cols)[order], np.array(vals)[order]
    key = r * 1000 + c
    starts = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
    stable = np.array([sum_seq(v[a:b]) for a, b in zip(starts, np.r_[starts[1:], len(v)])])
    upper = orc.coo_to_csr(60, rows, cols, vals, drop_zeros=False)
    assert not np.array_equal(stable.view(np.int64), upper.data.view(np.int64))


def sum_seq(v):
    x = v[0]
    for y in v[1:]:
        x = x + y
    return x


def test_c0_matches_reference_hashes(orc, golden, golden_meta):
    from paper_2502_17632_b200 import synth
    import paper_2502_17632_b200 as gb

    meta = golden_meta["cases"]["c0"]
    fd = synth.generate("c0", seed=1)
    A = orc.build_clique_graph(fd.num_cells, fd.net_start, fd.pin_cell, None)
    assert A.nnz == meta["nnz"]
    assert sha(A.indptr) == meta["indptr_sha"]
    assert sha(A.indices) == meta["indices_sha"]
    assert sha(A.data) == meta["values_sha"]
    deg = orc.degrees(A)
    assert sha(deg) == meta["degrees_sha"]
    g0 = gb.initial_signal(fd, gb.GiftConfig(seed=0, jitter_scale=10.0))
    assert sha(g0) == meta["g0_sha"]
    g32 = g0.astype(np.float32).astype(np.float64)
    assert sha(orc.gift_filter(A, g32, DEFAULT, deg)) == meta["filter_g32_sha"]
    r = fd.region
    placed = orc.place_epilogue(orc.gift_filter(A, g0, DEFAULT, deg), fd.fixed_mask(), fd.fixed_positions(),
                                [r.xmin, r.ymin, r.xmax, r.ymax])
    assert sha(placed) == meta["place_sha"]


@pytest.mark.parametrize("kind", ["random", "sorted", "reversed", "organ", "few", "killer", "killer4"])
def test_introsort_restatement_matches_libstdcxx(orc, kind):
    rng = np.random.default_rng(hash(kind) % 2**32)
    for n in (0, 1, 2, 15, 16, 17, 33, 100, 257, 1000, 4099):
        if kind == "random":
            keys = rng.integers(0, max(n // 3, 1), n)
        elif kind == "sorted":
            keys = np.sort(rng.integers(0, 50, n))
        elif kind == "reversed":
            keys = np.sort(rng.integers(0, 50, n))[::-1].copy()
        elif kind == "organ":
            h = n // 2
            keys = np.concatenate([np.arange(h), np.arange(n - h)[::-1]])
        elif kind == "few":
            keys = rng.integers(0, 3, n)
        elif kind == "killer":
            keys = orc.antiqsort_keys(n)
        else:
            keys = orc.antiqsort_keys(n) // 4
        assert np.array_equal(orc.std_sort_perm_emulated(keys), orc.std_sort_perm_libstdcxx(keys)), (kind, n)


def _configs_meta():
    import json
    import os

    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "configs_meta.json")) as f:
        return json.load(f)["samples"]


@pytest.mark.parametrize("name", ["c1_full", "c2_s005", "c3_s003", "c4_s0004", "c2_s001_uncapped"])
def test_config_samples_match_reference_hashes(orc, name):
    """The oracle reproduces the reference bit for bit at c1 full size and on
    the scaled c2/c3/c4 samples the GPU parity tests use (hashes made by
    tests/golden/make_golden_configs.py from giftplace itself)."""
    from paper_2502_17632_b200 import synth
    import paper_2502_17632_b200 as gb

    meta = _configs_meta()[name]
    fd = synth.generate(meta["config"], seed=meta["seed"], scale=meta["scale"], window=meta["window"])
    A = orc.build_clique_graph(fd.num_cells, fd.net_start, fd.pin_cell, meta["cap"])
    assert A.nnz == meta["nnz"]
    assert sha(A.indptr) == meta["indptr_sha"]
    assert sha(A.indices) == meta["indices_sha"]
    assert sha(A.data) == meta["values_sha"]
    deg = orc.degrees(A)
    assert sha(deg) == meta["degrees_sha"]
    g0 = gb.initial_signal(fd, gb.GiftConfig(seed=0, jitter_scale=10.0))
    assert sha(g0) == meta["g0_sha"]
    g32 = g0.astype(np.float32).astype(np.float64)
    assert sha(orc.gift_filter(A, g32, DEFAULT, deg)) == meta["filter_g32_sha"]
    r = fd.region
    placed = orc.place_epilogue(orc.gift_filter(A, g0, DEFAULT, deg), fd.fixed_mask(), fd.fixed_positions(),
                                [r.xmin, r.ymin, r.xmax, r.ymax])
    assert sha(placed) == meta["place_sha"]


@pytest.mark.parametrize("cap", [0, 1, -2])
def test_caps_below_two_skip_every_net(orc, cap):
    """graph.py:136: nets with m > max_clique_pins are skipped, so a cap below 2
    (0 is a cap, not "no cap") leaves an empty graph."""
    ns = np.array([0, 2, 5, 9])
    pc = np.array([0, 1, 1, 2, 3, 0, 1, 2, 3])
    A = orc.build_clique_graph(4, ns, pc, cap)
    assert A.nnz == 0
    assert orc.build_clique_graph(4, ns, pc, 2).nnz == 2
    assert orc.build_clique_graph(4, ns, pc, None).nnz > 2
