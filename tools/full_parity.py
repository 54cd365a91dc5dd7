"""Full-size parity of every BASELINE config against the CPU oracle.

    python tools/full_parity.py [c0 c1 c2 c3 c4]

For each config: GPU build_clique_graph vs oracle build (CSR indptr / indices /
fp64 values and fp64 degrees compared bit for bit via SHA-256 of the arrays),
then the fp32 fused bank + gift_place epilogue vs the oracle's fp64
gift_filter + epilogue on the same fp32-rounded seed (relative L2 on absolute
and on die-centred coordinates; bar 1e-5).  Prints one JSON line per config.
Test infrastructure: imports the oracle; needs a GPU and host RAM for the
oracle (c3/c4 ~40 GB).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_17632_b200 as gb  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2502_17632_b200 import synth  # noqa: E402

DEFAULT = [(2.0, 2, 0.1), (4.0, 2, 0.7), (4.0, 4, 0.2)]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def rel(a, b) -> float:
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run(config: str, seed: int = 1) -> dict:
    t0 = time.perf_counter()
    fd = synth.generate(config, seed=seed)
    cap = fd.meta["max_clique_pins"]
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    adj = gb.build_clique_graph(fd, max_clique_pins=cap)
    g_indptr = np.asarray(adj.indptr, np.int64)
    g_indices = np.asarray(adj.indices, np.int64)
    g_values = np.asarray(adj.values)
    g_deg = np.asarray(adj.degrees)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = orc.build_clique_graph(fd.num_cells, fd.net_start, fd.pin_cell, cap)
    deg = orc.degrees(ref)
    t_orc = time.perf_counter() - t0
    out = {
        "config": config, "n": fd.num_cells, "nets": fd.num_nets, "pins": fd.num_pins, "cap": cap,
        "nnz": int(adj.nnz), "nnz_oracle": int(ref.nnz),
        "indptr_equal": bool(np.array_equal(g_indptr, ref.indptr)),
        "indices_equal": bool(np.array_equal(g_indices, ref.indices)),
        "values_bit_equal": bool(np.array_equal(g_values.view(np.int64), ref.data.view(np.int64))),
        "degrees_bit_equal": bool(np.array_equal(g_deg.view(np.int64), deg.view(np.int64))),
        "sha_values": [sha(g_values), sha(ref.data)],
        "scipy_sorted_rows_skip": ref.input_rows_sorted,
        "t_generate_s": round(t_gen, 2), "t_gpu_build_s": round(t_gpu, 2), "t_oracle_build_s": round(t_orc, 2),
    }
    del g_indices, g_values
    g32 = synth.signal_fp32(fd, seed=0)
    t0 = time.perf_counter()
    want = orc.gift_filter(ref, g32.astype(np.float64), DEFAULT, deg)
    r = fd.region
    want_p = orc.place_epilogue(want, fd.fixed_mask(), fd.fixed_positions(), r.bounds())
    out["t_oracle_filter_s"] = round(time.perf_counter() - t0, 2)
    got = gb.gift_filter(adj, g32)
    centre = np.array(r.center)
    out["filter_rel_l2"] = rel(got, want)
    out["filter_rel_l2_centred"] = rel(got - centre, want - centre)
    placed, _ = gb.gift_place(fd, adj, gb.GiftConfig(seed=0, jitter_scale=10.0))
    out["place_rel_l2"] = rel(placed, want_p)
    mask = fd.fixed_mask()
    out["fixed_rows_exact"] = bool(np.array_equal(placed[mask], fd.fixed_positions()[mask]))
    out["pass"] = bool(out["indptr_equal"] and out["indices_equal"] and out["values_bit_equal"]
                       and out["degrees_bit_equal"] and out["filter_rel_l2"] <= 1e-5
                       and out["filter_rel_l2_centred"] <= 1e-5 and out["place_rel_l2"] <= 1e-5
                       and out["fixed_rows_exact"])
    return out


if __name__ == "__main__":
    orc.build()
    for cfg in sys.argv[1:] or ["c0", "c1", "c2", "c3", "c4"]:
        print(json.dumps(run(cfg)), flush=True)
