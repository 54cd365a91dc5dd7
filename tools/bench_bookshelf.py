"""Time the device Bookshelf reader on a synthetic design written as text.

    python tools/bench_bookshelf.py [--config c3] [--scale 1.0] [--ref /root/reference/pkg/src]

Writes <config> as Bookshelf files under a temp dir (names "c<i>", pin
offsets on half the pins), then times read_design (file read + device parse +
copy-out) and, with --ref (build container only), the reference parse_design
on the same files.  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def write_text(fd, d: str, seed: int = 0) -> dict:
    rng = np.random.default_rng(seed)
    n = fd.num_cells
    fixed = fd.fixed_mask()
    w, h = fd.widths.tolist(), fd.heights.tolist()
    with open(os.path.join(d, "d.nodes"), "w") as f:
        f.write(f"UCLA nodes 1.0\nNumNodes : {n}\nNumTerminals : {int(fixed.sum())}\n")
        f.writelines(f"c{i} {w[i]!r} {h[i]!r}{' terminal' if fixed[i] else ''}\n" for i in range(n))
    ns, pc = fd.net_start, fd.pin_cell.tolist()
    offs = np.round(rng.normal(size=(len(pc), 2)), 3).tolist()
    with open(os.path.join(d, "d.nets"), "w") as f:
        f.write(f"UCLA nets 1.0\nNumNets : {fd.num_nets}\nNumPins : {len(pc)}\n")
        for e in range(fd.num_nets):
            f.write(f"NetDegree : {ns[e + 1] - ns[e]} n{e}\n")
            f.writelines(f"  c{pc[k]} I : {offs[k][0]} {offs[k][1]}\n" if k & 1 else f"  c{pc[k]} O\n"
                         for k in range(ns[e], ns[e + 1]))
    fp = fd.fixed_positions().tolist()
    with open(os.path.join(d, "d.pl"), "w") as f:
        f.write("UCLA pl 1.0\n\n")
        f.writelines(f"c{i} {fp[i][0] - w[i] / 2!r} {fp[i][1] - h[i] / 2!r} : N /FIXED\n" if fixed[i]
                     else f"c{i} 0 0 : N\n" for i in range(n))
    with open(os.path.join(d, "d.aux"), "w") as f:
        f.write("RowBasedPlacement : d.nodes d.nets d.pl\n")
    sizes = {ext: os.path.getsize(os.path.join(d, f"d.{ext}")) for ext in ("nodes", "nets", "pl")}
    return sizes


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ref", default=None, help="reference source dir: also time giftplace.parse_design")
    args = ap.parse_args()
    from paper_2502_17632_b200 import synth

    fd = synth.generate(args.config, seed=0, scale=args.scale)
    out = {"workload": f"{args.config} scale {args.scale}: {fd.num_cells} cells, {fd.num_nets} nets, "
                       f"{fd.num_pins} pins as Bookshelf text"}
    with tempfile.TemporaryDirectory() as d:
        t0 = time.perf_counter()
        sizes = write_text(fd, d)
        out["write_text_s"] = round(time.perf_counter() - t0, 2)
        out["bytes"] = sizes
        total = sum(sizes.values())
        aux = os.path.join(d, "d.aux")
        if args.ref is None:
            import paper_2502_17632_b200 as gb

            gb.read_design(aux)  # warm-up (context, allocator pools)
            ts = []
            for _ in range(args.reps):
                t0 = time.perf_counter()
                got = gb.read_design(aux)
                ts.append(time.perf_counter() - t0)
            assert np.array_equal(got.pin_cell, fd.pin_cell) and np.array_equal(got.net_start, fd.net_start)
            # breakdown: file read, device parse alone
            import ctypes

            from paper_2502_17632_b200 import _lib, bookshelf

            t0 = time.perf_counter()
            paths = [os.path.join(d, f"d.{e}") for e in ("nodes", "nets", "pl")]
            texts = [bookshelf._read(p) for p in paths]
            out["file_read_s"] = round(time.perf_counter() - t0, 4)
            lib = _lib.load_library()
            tp = []
            for _ in range(args.reps):
                hnd = ctypes.c_void_p()
                t0 = time.perf_counter()
                _lib.check(lib.gift_bookshelf_parse(_lib.context(), texts[0], len(texts[0]), texts[1], len(texts[1]),
                                                    texts[2], len(texts[2]), ctypes.byref(hnd)))
                tp.append(time.perf_counter() - t0)
                lib.gift_bookshelf_destroy(_lib.context(), hnd)
            out["device_parse_s"] = round(min(tp), 4)
            best = min(ts)
            out.update({"read_design_s": round(best, 4), "MB_per_s": round(total / best / 1e6, 1),
                        "lines_per_s": round((fd.num_cells * 2 + fd.num_nets + fd.num_pins) / best, 1)})
        else:
            sys.path.insert(0, args.ref)
            import giftplace as gp

            t0 = time.perf_counter()
            gp.parse_design(aux)
            ref = time.perf_counter() - t0
            out.update({"reference_parse_design_s": round(ref, 3), "reference_MB_per_s": round(total / ref / 1e6, 2)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
