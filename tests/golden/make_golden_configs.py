"""Reference hashes for the BASELINE configs at the sizes the tests run.

Run in the build container, where the reference is importable:
    python tests/golden/make_golden_configs.py [/root/reference/pkg/src]

For config c1 at full size and the scaled c2 / c3 / c4 samples the GPU parity
tests use (tests/test_gpu_parity.py `SAMPLES`), it imports `giftplace` and
records SHA-256 hashes of what the reference computes:

  * build_clique_graph (graph.py:120-158): indptr / indices / fp64 values,
    SparseSymMatrix.degrees (graph.py:89-94);
  * initial_signal (gift.py:54-70) for GiftConfig(seed, jitter_scale=10);
  * gift_filter (gift.py:73-95) on that signal rounded once to fp32;
  * gift_place (gift.py:98-119) with the same config (fp64 end to end).

Output: tests/golden/configs_meta.json (hashes only; a few KB).  The oracle is
checked against it on CPU (tests/test_oracle.py) and the CUDA path on the GPU
(tests/test_gpu_parity.py).  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF_SRC = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import giftplace as gp  # noqa: E402  (the reference)
import scipy  # noqa: E402

from paper_2502_17632_b200 import synth  # noqa: E402

# (name, config, seed, scale, window, cap) -- must match SAMPLES in the tests
SAMPLES = [
    ("c1_full", "c1", 1, 1.0, None, None),
    ("c2_s005", "c2", 2, 0.05, 600, 200),
    ("c3_s003", "c3", 2, 0.03, 600, 200),
    ("c4_s0004", "c4", 2, 0.004, 600, 100),
    ("c2_s001_uncapped", "c2", 2, 0.01, 600, None),
]


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    meta = {"numpy": np.__version__, "scipy": scipy.__version__, "reference": REF_SRC, "samples": {}}
    for name, config, seed, scale, window, cap in SAMPLES:
        t0 = time.perf_counter()
        fd = synth.generate(config, seed=seed, scale=scale, window=window)
        d = fd.to_design(gp)
        adj = gp.build_clique_graph(d, max_clique_pins=cap)
        cfg = gp.GiftConfig(seed=0, jitter_scale=10.0)
        g0 = gp.initial_signal(d, cfg)
        g32 = g0.astype(np.float32).astype(np.float64)
        filt = gp.gift_filter(adj, g32)
        placed, _ = gp.gift_place(d, adj, cfg)
        meta["samples"][name] = {
            "config": config, "seed": seed, "scale": scale, "window": window, "cap": cap,
            "n": int(adj.n), "nnz": int(adj.nnz),
            "indptr_sha": h(np.asarray(adj.indptr, dtype=np.int64)),
            "indices_sha": h(np.asarray(adj.indices, dtype=np.int64)),
            "values_sha": h(np.asarray(adj.values, dtype=np.float64)),
            "degrees_sha": h(np.asarray(adj.degrees, dtype=np.float64)),
            "g0_sha": h(g0), "filter_g32_sha": h(filt), "place_sha": h(placed),
        }
        print(f"{name}: n={adj.n} nnz={adj.nnz} ({time.perf_counter() - t0:.1f} s)", flush=True)
    with open(os.path.join(HERE, "configs_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
