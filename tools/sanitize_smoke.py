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

# factored clique model (k_fact_tsum / k_fact_hop) and the implicit term on the tiled path
_lib.set_option("tiled_min_mean", 32)
adj_f = gb.build_clique_graph(fd, max_clique_pins=200, implicit_above=5)
f = gb.gift_filter(adj_f, g)
assert np.linalg.norm(f - b) / np.linalg.norm(b) < 1e-5
f64 = gb.gift_filter(adj_f, g, gb.GiftConfig(precision="fp64"))
assert np.linalg.norm(f64 - b) / np.linalg.norm(b) < 1e-11
pa, _ = gb.gift_place_arrays(fd.net_start, fd.pin_cell, g, fd.fixed_mask(), fd.fixed_positions(), fd.region.bounds(),
                             max_clique_pins=200, implicit_above=5)

# ghost rows through the peer-memory pull (threads as virtual ranks) on tiled local blocks
import threading  # noqa: E402

import torch  # noqa: E402

from paper_2502_17632_b200 import shard  # noqa: E402

_lib.set_option("tiled_min_mean", 1)
world = 2
hub = shard.ThreadPeerExchange(world)
outs, errs = [None] * world, []


def run(rank):
    try:
        torch.cuda.set_device(0)
        sf = shard.cuda_sharded_filter(adj, world, rank, 0, exchange=hub.for_rank(rank))
        r0, r1 = sf.plan.r0, sf.plan.r1
        gg = torch.from_numpy(np.ascontiguousarray(g[r0:r1])).cuda()
        out = torch.zeros((r1 - r0, 2), dtype=torch.float64, device="cuda")
        sf.run(gg, gb.DEFAULT_TERMS, out)
        torch.cuda.synchronize()
        outs[rank] = (r0, out.cpu().numpy())
        sf.ex.close(sf.be)
    except Exception as e:
        errs.append(repr(e))
        hub.barrier.abort()


ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
[t.start() for t in ts]
[t.join(timeout=600) for t in ts]
assert not errs, errs
full = np.zeros_like(b)
for r0, blk in outs:
    full[r0:r0 + len(blk)] = blk
assert np.linalg.norm(full - b) / np.linalg.norm(b) < 1e-5
print("sanitize smoke ok", adj.n, adj.nnz, adj_f.nnz)
