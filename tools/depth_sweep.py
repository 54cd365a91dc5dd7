"""Filter-depth sweep (BASELINE config 4): per-hop SpMM throughput vs graph build.

    python tools/depth_sweep.py [--config c4] [--depths 1 2 4 8 16 32] [--reps 5]

Builds the clique graph once (timed), then runs the single-term bank
((sigma=4, k, alpha=1),) for each depth k through the gift_filter C ABI with
device buffers and the fused placement epilogue, timed with CUDA events
(median of --reps after a warm-up that also builds the cached tiled copy).
Prints one JSON line per depth: ms per call, ms per hop (slope between
depths), nnz_op x hops / s, and the one-off costs (graph build, first call).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--depths", type=int, nargs="+", default=[1, 2, 4, 8, 16, 32])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()

    import torch

    import paper_2502_17632_b200 as gb
    from paper_2502_17632_b200 import _lib, synth

    lib = _lib.load_library()
    gb.set_tiled_policy("always")  # a resident graph: per-hop cost on the tiled kernels from the first call
    fd = synth.generate(args.config, seed=args.seed)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    adj = gb.build_clique_graph(fd, max_clique_pins=fd.meta["max_clique_pins"])
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    n = adj.n
    nnz_op = adj.nnz + n
    dev = torch.device("cuda", 0)
    dg = torch.from_numpy(synth.signal_fp32(fd, seed=0)).to(dev)
    dmask = torch.from_numpy(fd.fixed_mask().astype(np.uint8)).to(dev)
    dpos = torch.from_numpy(np.nan_to_num(fd.fixed_positions(), nan=0.0)).to(dev)
    dout = torch.empty((n, 2), dtype=torch.float64, device=dev)
    region = fd.region.bounds()
    ctx = _lib.context(0)
    rows = []
    for k in args.depths:
        sig = np.array([4.0])
        kk = np.array([k], dtype=np.int64)
        al = np.array([1.0])

        def call():
            _lib.check(lib.gift_filter(ctx, adj.handle, 1, sig.ctypes.data_as(_lib.c_dp),
                                       kk.ctypes.data_as(_lib.c_i64p), al.ctypes.data_as(_lib.c_dp), 2,
                                       _lib.GIFT_DTYPE_F32, _lib.dptr(dg), _lib.GIFT_DTYPE_F64, _lib.dptr(dout),
                                       _lib.dptr(dmask), _lib.dptr(dpos), region.ctypes.data_as(_lib.c_dp),
                                       _lib.GIFT_PREC_FP32))

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()
        torch.cuda.synchronize()
        first = time.perf_counter() - t0
        call()
        ts = []
        for _ in range(args.reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            call()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        rows.append((k, ms))
        print(json.dumps({"config": args.config, "n": n, "nnz_op": nnz_op, "depth_k": k, "ms_per_call": round(ms, 4),
                          "nnz_hops_per_s": nnz_op * k / (ms / 1e3), "first_call_s": round(first, 3),
                          "graph_build_s": round(build_s, 3)}), flush=True)
    if len(rows) >= 2:
        ks = np.array([r[0] for r in rows], dtype=float)
        ms = np.array([r[1] for r in rows])
        slope, icpt = np.polyfit(ks, ms, 1)
        print(json.dumps({"config": args.config, "fit": "ms_per_call = a + b * k", "a_ms": round(float(icpt), 4),
                          "b_ms_per_hop": round(float(slope), 4),
                          "per_hop_nnz_per_s": nnz_op / (slope / 1e3), "graph_build_s": round(build_s, 3)}))


if __name__ == "__main__":
    main()
