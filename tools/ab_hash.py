"""Hash of the fp32 bank on the tiled kernels for A/B library variants
(GIFT_LIB=...): variants that claim bit-identical results must print the
same hashes.   python tools/ab_hash.py [config scale ...]"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_17632_b200 as gb  # noqa: E402
from paper_2502_17632_b200 import _lib, synth  # noqa: E402

_lib.set_option("tiled_min_rows", 1)
_lib.set_option("tiled_min_mean", 1)
gb.set_tiled_policy("always")
args = sys.argv[1:] or ["c3", "0.05", "c4", "0.02", "c1", "0.3"]
for cfg, sc in zip(args[::2], args[1::2]):
    fd = synth.generate(cfg, seed=6, scale=float(sc))
    adj = gb.build_clique_graph(fd, max_clique_pins=fd.meta["max_clique_pins"])
    out = gb.gift_filter(adj, synth.signal_fp32(fd, seed=3))
    print(cfg, sc, hashlib.sha256(out.tobytes()).hexdigest()[:16], adj.tiled_info()["f4"]["built"], flush=True)
