"""Seeded synthetic netlists for the five BASELINE.json configurations.

The paper's ISPD2014 suite is not available in this environment, so these
generators stand in for it with the shapes BASELINE.json fixes (SURVEY.md
§8(d)): cell / pad / macro counts, net counts, the per-bin pin-count mix,
locality windows of +-W cell indices, 5% of nets carrying one boundary pad,
and (c3) fixed macros joined to 10-50 nets each. Everything is vectorised
numpy and emits a `FlatDesign` directly (a 10M-cell design in seconds).

Conventions (recorded in every design's `meta`):
* ids: movable cells 0..N_mov-1, then fixed macros, then fixed pads
  (movable-first as in benchgen.py:90-100);
* a net draws its bin, then m uniformly in the bin, a centre c uniform over
  movable ids, and m DISTINCT movable cells uniformly from
  [c-W, c+W] clipped to [0, N_mov); pin order is the draw order;
* with p = 0.05 one uniformly chosen pad is appended as the last pin (the
  pad counts toward m for 2/m and for max_clique_pins, graph.py:133-136);
* macros (c3) are appended after the movable pins of 10-50 random nets;
* die: c0 1000, c1 10000, c2-c4 10000*sqrt(N_mov/211000) (unspecified by
  BASELINE.json); pads evenly spaced on a ring inset 0.5 from the die edge
  (pad-ring convention of benchgen.py:107-119);
* initial signal: `initial_signal(design, GiftConfig(seed, jitter_scale=10))`,
  i.e. die centre + 10*N(0,1), rounded once to fp32 (`signal_fp32`).
"""

from __future__ import annotations

import math

import numpy as np

from .netlist import FlatDesign, Region

BINS_SMALL = ((2, 2, 0.60), (3, 3, 0.20), (4, 5, 0.10), (6, 20, 0.09), (21, 100, 0.01))
BINS_TAIL = ((2, 2, 0.55), (3, 3, 0.20), (4, 5, 0.12), (6, 20, 0.10), (21, 200, 0.025), (201, 2000, 0.005))

CONFIGS: dict[str, dict] = {
    "c0": dict(n_mov=10_000, n_pads=200, n_macros=0, n_nets=10_500, bins=BINS_SMALL, window=500,
               die=1000.0, widths=None, max_clique_pins=None),
    "c1": dict(n_mov=211_000, n_pads=540, n_macros=0, n_nets=221_000, bins=BINS_SMALL, window=2000,
               die=10000.0, widths=((1, 2, 3, 4), (0.5, 0.3, 0.15, 0.05)), max_clique_pins=None),
    "c2": dict(n_mov=1_100_000, n_pads=2000, n_macros=0, n_nets=1_200_000, bins=BINS_TAIL, window=5000,
               die=None, widths=None, max_clique_pins=200),
    "c3": dict(n_mov=2_180_000, n_pads=8900, n_macros=8000, n_nets=2_230_000, bins=BINS_TAIL, window=5000,
               die=None, widths=None, max_clique_pins=200),
    "c4": dict(n_mov=10_000_000, n_pads=20_000, n_macros=0, n_nets=10_500_000, bins=BINS_TAIL, window=20_000,
               die=None, widths=None, max_clique_pins=100),
}

PAD_PROB = 0.05
JITTER = 10.0


def _die(cfg: dict) -> float:
    if cfg["die"] is not None:
        return float(cfg["die"])
    return float(round(10000.0 * math.sqrt(cfg["n_mov"] / 211_000)))


def _ring(n_pads: int, die: float) -> np.ndarray:
    """Pad centres evenly along the boundary, inset 0.5 (benchgen.py:107-119 convention)."""
    t = (np.arange(n_pads) + 0.5) * (4.0 * die) / max(n_pads, 1)
    side = np.minimum((t // die).astype(np.int64), 3)
    u = t - side * die
    x = np.select([side == 0, side == 1, side == 2, side == 3], [u, die - 0.5, die - u, 0.5])
    y = np.select([side == 0, side == 1, side == 2, side == 3], [0.5, u, die - 0.5, die - u])
    return np.stack([x, y], axis=1)


def _distinct_window_pins(rng, m, lo, span):
    """For each net e draw m[e] distinct ints from [lo[e], lo[e]+span[e]) in draw order."""
    E = len(m)
    net_of = np.repeat(np.arange(E, dtype=np.int64), m)
    lo_p = np.repeat(lo, m)
    span_p = np.repeat(span, m)
    cell = lo_p + rng.integers(0, span_p)
    idx = np.arange(len(cell))  # pins still under suspicion (whole nets)
    while len(idx):
        nets = net_of[idx]
        key = nets * (int(span.max()) + 1) + (cell[idx] - lo_p[idx])
        order = np.argsort(key, kind="stable")
        sk = key[order]
        dup = np.zeros(len(idx), dtype=bool)
        dup[1:] = sk[1:] == sk[:-1]
        if not dup.any():
            break
        redo = idx[order[dup]]
        cell[redo] = lo_p[redo] + rng.integers(0, span_p[redo])
        bad_nets = np.unique(net_of[redo])
        idx = idx[np.isin(nets, bad_nets)]
    return cell


def generate(config: str = "c0", seed: int = 0, scale: float = 1.0, window: int | None = None) -> FlatDesign:
    """Build config `config` ('c0'..'c4'); `scale` shrinks every count (parity-sized variants)."""
    cfg = dict(CONFIGS[config])
    n_mov = max(int(round(cfg["n_mov"] * scale)), 8)
    n_pads = max(int(round(cfg["n_pads"] * scale)), 4)
    n_macros = int(round(cfg["n_macros"] * scale))
    n_nets = max(int(round(cfg["n_nets"] * scale)), 4)
    W = int(window if window is not None else cfg["window"])
    die = _die(cfg) * (1.0 if scale == 1.0 else math.sqrt(scale))
    rng = np.random.default_rng(seed)

    lows = np.array([b[0] for b in cfg["bins"]], dtype=np.int64)
    highs = np.array([b[1] for b in cfg["bins"]], dtype=np.int64)
    probs = np.array([b[2] for b in cfg["bins"]], dtype=float)
    probs = probs / probs.sum()
    b = rng.choice(len(probs), size=n_nets, p=probs)
    m = rng.integers(lows[b], highs[b] + 1)
    m = np.minimum(m, n_mov)
    centre = rng.integers(0, n_mov, n_nets)
    lo = np.maximum(centre - W, 0)
    hi = np.minimum(centre + W, n_mov - 1)
    span = hi - lo + 1
    m = np.minimum(m, span)
    mov_cells = _distinct_window_pins(rng, m, lo, span)

    n_fixed = n_macros + n_pads
    N = n_mov + n_fixed
    pad_base = n_mov + n_macros
    has_pad = rng.random(n_nets) < PAD_PROB
    pad_cell = pad_base + rng.integers(0, n_pads, n_nets)

    # macros: each joins k ~ U{10..50} distinct random nets
    if n_macros:
        k = rng.integers(10, 51, n_macros)
        mac_net = np.concatenate([rng.choice(n_nets, size=int(kk), replace=False) for kk in k])
        mac_cell = np.repeat(n_mov + np.arange(n_macros, dtype=np.int64), k)
        order = np.argsort(mac_net, kind="stable")
        mac_net, mac_cell = mac_net[order], mac_cell[order]
        mac_cnt = np.bincount(mac_net, minlength=n_nets)
    else:
        mac_net = np.zeros(0, dtype=np.int64)
        mac_cell = np.zeros(0, dtype=np.int64)
        mac_cnt = np.zeros(n_nets, dtype=np.int64)

    counts = m + mac_cnt + has_pad
    net_start = np.zeros(n_nets + 1, dtype=np.int64)
    np.cumsum(counts, out=net_start[1:])
    pin_cell = np.empty(int(net_start[-1]), dtype=np.int32)
    mov_start = np.zeros(n_nets + 1, dtype=np.int64)
    np.cumsum(m, out=mov_start[1:])
    net_of = np.repeat(np.arange(n_nets, dtype=np.int64), m)
    pin_cell[net_start[net_of] + (np.arange(len(mov_cells)) - mov_start[net_of])] = mov_cells
    if n_macros:
        first = np.searchsorted(mac_net, mac_net, side="left")
        rank = np.arange(len(mac_net)) - first
        pin_cell[net_start[mac_net] + m[mac_net] + rank] = mac_cell
    pn = np.flatnonzero(has_pad)
    pin_cell[net_start[pn + 1] - 1] = pad_cell[pn]

    fixed_mask = np.zeros(N, dtype=bool)
    fixed_mask[n_mov:] = True
    fixed_pos = np.full((N, 2), np.nan)
    widths = np.ones(N)
    heights = np.ones(N)
    if cfg["widths"] is not None:
        vals, p = cfg["widths"]
        widths[:n_mov] = rng.choice(np.array(vals, dtype=float), size=n_mov, p=np.array(p))
    if n_macros:
        g = int(math.ceil(math.sqrt(n_macros)))
        pitch = die / g
        mw = rng.uniform(20.0, 200.0, n_macros)
        mh = rng.uniform(20.0, 200.0, n_macros)
        slot = np.arange(n_macros)
        cx = (slot % g + 0.5) * pitch + rng.uniform(-1, 1, n_macros) * np.maximum(pitch - mw, 0) / 2
        cy = (slot // g + 0.5) * pitch + rng.uniform(-1, 1, n_macros) * np.maximum(pitch - mh, 0) / 2
        fixed_pos[n_mov:pad_base] = np.stack([cx, cy], axis=1)
        widths[n_mov:pad_base] = mw
        heights[n_mov:pad_base] = mh
    fixed_pos[pad_base:] = _ring(n_pads, die)

    meta = dict(config=config, seed=seed, scale=scale, window=W, die=die, n_mov=n_mov, n_macros=n_macros,
                n_pads=n_pads, n_nets=n_nets, pad_prob=PAD_PROB, max_clique_pins=cfg["max_clique_pins"],
                generator="paper_2502_17632_b200.synth v1")
    return FlatDesign(net_start, pin_cell, fixed_mask, fixed_pos, Region(0.0, 0.0, die, die),
                      widths, heights, meta)


def signal_fp32(design, seed: int = 0, jitter: float = JITTER) -> np.ndarray:
    """initial_signal(design, GiftConfig(seed, jitter_scale=jitter)) rounded once to fp32
    (gift.py:54-70; SURVEY.md §8(d) 'Initial signal')."""
    from .gift import GiftConfig, initial_signal

    g = initial_signal(design, GiftConfig(seed=seed, jitter_scale=jitter))
    return g.astype(np.float32)
