"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
build + from_coo + fp64 and fp32 banks + BMT (forced on a small graph) + the
stepped sharded kernels with 2 virtual ranks.  Exits non-zero on any mismatch."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# the tiled hop is forced on small graphs through the option API (below)

import paper_2502_17632_b200 as gb  # noqa: E402
from paper_2502_17632_b200 import _lib, synth  # noqa: E402

_lib.set_option("tiled_min_rows", 1)
_lib.set_option("tiled_min_mean", 1)
gb.set_tiled_policy("always")

fd = synth.generate("c2", seed=5, scale=0.004, window=300)
adj = gb.build_clique_graph(fd, max_clique_pins=200)
g = synth.signal_fp32(fd, seed=1)
a = gb.gift_filter(adj, g)
b = gb.gift_filter(adj, g, gb.GiftConfig(precision="fp64"))
assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-5
p, _ = gb.gift_place(fd, adj, gb.GiftConfig(seed=1, jitter_scale=10.0))
op = gb.normalized_augmented_adjacency(adj, 2.0)
gb.apply_operator_power(op, g.astype(np.float64), 2)
c = gb.from_coo(4, [0, 1, 1, 2, 0, 2], [1, 0, 2, 1, 2, 0], [1.0, 1.0, 2.0, 2.0, 3.0, 3.0])
assert c.degrees.tolist() == [4.0, 3.0, 5.0, 0.0]
print("sanitize smoke ok", adj.n, adj.nnz)
