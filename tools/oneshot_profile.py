"""Where the one-shot (fresh process) placement time goes.

    python tools/oneshot_profile.py [--config c3] [--repeat 2]

In a fresh process: CUDA/torch init, library context, then `repeat` rounds of
netlist -> positions through the Python API with a device sync after every
phase (H2D of the pin table, clique build, degrees + s, first bank, D2H).
Round 1 is the cold (one-shot) path; later rounds show the warm cost.
Prints one JSON line per round.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--warm-small", action="store_true")
    args = ap.parse_args()
    t_proc = time.perf_counter()
    import numpy as np
    import torch

    import paper_2502_17632_b200 as gb
    from paper_2502_17632_b200 import _lib, synth

    t_import = time.perf_counter() - t_proc
    fd = synth.generate(args.config, seed=args.seed)
    cap = fd.meta["max_clique_pins"]
    t0 = time.perf_counter()
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    t_torch = time.perf_counter() - t0
    t0 = time.perf_counter()
    _lib.load_library()
    _lib.context(0)
    t_ctx = time.perf_counter() - t0
    print(json.dumps({"import_s": round(t_import, 3), "torch_cuda_init_s": round(t_torch, 3),
                      "gift_ctx_s": round(t_ctx, 3)}), flush=True)
    cfg = gb.GiftConfig(seed=0, jitter_scale=10.0)
    if args.warm_small:
        # a tiny build + bank first: loads the kernels' modules (lazy loading)
        # so the timed round below shows the size-dependent costs only
        t0 = time.perf_counter()
        tiny = synth.generate("c0", seed=1, scale=0.1)
        gb.gift_place(tiny, gb.build_clique_graph(tiny), cfg)
        torch.cuda.synchronize()
        print(json.dumps({"warm_small_s": round(time.perf_counter() - t0, 3)}), flush=True)
    import ctypes

    net_start, pin_cell = np.ascontiguousarray(fd.net_start, np.int64), np.ascontiguousarray(fd.pin_cell, np.int32)
    t0 = time.perf_counter()
    d_ns = torch.from_numpy(net_start).cuda()
    d_pc = torch.from_numpy(pin_cell).cuda()
    torch.cuda.synchronize()
    h2d_s = time.perf_counter() - t0
    lib = _lib.load_library()
    h = ctypes.c_void_p()
    t0 = time.perf_counter()
    _lib.check(lib.gift_build_clique_graph(_lib.context(0), fd.num_cells, len(net_start) - 1, _lib.dptr(d_ns),
                                           _lib.dptr(d_pc), cap if cap is not None else -1, ctypes.byref(h), None))
    torch.cuda.synchronize()
    dev_build_s = time.perf_counter() - t0
    lib.gift_csr_destroy(h)
    print(json.dumps({"pin_table_h2d_s": round(h2d_s, 4), "device_build_s (first)": round(dev_build_s, 4),
                      "pins": int(len(pin_cell))}), flush=True)
    for r in range(args.repeat):
        ph = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        adj = gb.build_clique_graph(fd, max_clique_pins=cap)
        torch.cuda.synchronize()
        ph["build_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        adj.degrees  # noqa: B018  (degrees + D2H of n doubles)
        ph["degrees_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        g0 = gb.initial_signal(fd, cfg)
        ph["initial_signal_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        placed, _ = gb.gift_place(fd, adj, cfg)
        torch.cuda.synchronize()
        ph["gift_place_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        placed2, _ = gb.gift_place(fd, adj, cfg)
        torch.cuda.synchronize()
        ph["gift_place_again_s"] = time.perf_counter() - t0
        ph = {k: round(v, 4) for k, v in ph.items()}
        ph["round"] = r
        ph["nnz"] = int(adj.nnz)
        ph["finite"] = bool(np.isfinite(placed).all()) and g0.shape == placed.shape
        print(json.dumps(ph), flush=True)
        del adj


if __name__ == "__main__":
    main()
