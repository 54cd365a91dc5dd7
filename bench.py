"""Benchmark: GiFt filter-bank throughput (nnz x hops / s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

A step is one GiFt filter pass (gift.py:73-95 + the gift_place epilogue
gift.py:112-118): the default bank 0.1 A_2^2 + 0.7 A_4^2 + 0.2 A_4^4 (6
algorithmic SpMM hops) over the clique graph of one synthetic netlist, with
the graph resident (built once, like SparseSymMatrix caching its degrees).
Metric = nnz_op * 6 / step time, nnz_op = nnz(A) + N (the stored entries of
A_sigma).

Workload (BASELINE.json configs[3], quoted "at 1/2/4/8 B200"): c3, 2.18M
movable cells + 8k macros + 8.9k pads, 2.23M nets, max_clique_pins=200,
seeded synthetic (the paper's ISPD2014 designs are not available).  The CSR
(~7 GB) is far larger than L2, so no explicit flush is needed between steps.

`value`  : device time of K steps with every input resident in HBM.
`e2e`    : the same metric through the C ABI call gift_filter_host with
           pinned HOST buffers (H2D of the fp32 seed + fixed mask/positions,
           D2H of the fp64 placement inside every step).
`roofline`: the dominant kernel (the fused hop), algorithmic bytes
           (8*nnz_op + 24*N + 8 per hop unit) / its mean CUDA-event time.
`cpu_baseline`: the oracle port (oracle/gift_oracle.c, fp64 reference
           operation order, OpenMP over rows) on a scaled sample, rank 0, N=1;
           `cpu_baseline.reference` times the reference's OWN gift_filter
           (giftplace, scipy, one core; staged in oracle/_ref by build()) on
           c1 and on the same scaled sample.
`oneshot_e2e`: the reference's real use -- one placement per design
           (cli.py:203-220) -- measured in FRESH processes: netlist arrays in
           host memory -> positions in host memory, through the Python API
           (build_clique_graph + gift_place) and through the C ABI
           (gift_place_host), CUDA context + library load included.
--impl reference: the reference arm: the oracle port (all host threads) on
           the SAME full config, one fp64 gift_filter per step (the reference
           is pure Python/scipy; its own single-core timing is in
           cpu_baseline.reference).
Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run, one
process per GPU) unless WORLD_SIZE is already set.  The SAME graph is
row-sharded over the ranks (strong scaling, paper_2502_17632_b200/shard.py):
each rank builds the graph on its GPU, cuts its nnz-balanced row block on the
device (no host copy of the CSR), and gets its ghost rows per hop straight
from the owners' signal buffers over NVLink peer memory (`--exchange peer`,
the default: CUDA IPC mappings + one kernel of peer loads, csrc/peer.cu;
falls back to the NCCL all_to_all of `--exchange nccl` if the mappings cannot
be made), overlapped with the local part of the hop; `value` counts the one
graph's nnz_op * 6 per step over the max-rank time.  `--config c4` is the
north-star scaling configuration (10M cells).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

FACTOR_ABOVE = 6  # the factored leg stores nets of up to 6 pins as entries (bench.py "factored")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gift_filter_nnz_hops_per_sec"
UNIT = "nnz*hops/s"
HOPS = 6
SAMPLE_SCALE = {"c0": 1.0, "c1": 0.5, "c2": 0.04, "c3": 0.03, "c4": 0.01}


def bytes_per_hop(nnz_op: int, n: int) -> int:
    """int32 col + fp32 value per stored entry, int64 rowptr,
    float2 read and float2 write per row."""
    return 8 * nnz_op + 24 * n + 8


def ncu_traffic(config: str, fin: int):
    """DRAM bytes per launch of the hop pass with fin floats per row, from the
    committed ncu --set full capture of this bench (profiles/r01_traffic_<config>.json),
    summed over the kernels the pass launches (BMT tile kernel + wide-row kernel)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_traffic_{config}.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        k = json.load(f)["kernels"]
    by_fout: dict[str, float] = {}
    for name, v in k.items():
        args = name[name.index("<") + 1:name.index(">")].split(",")
        if int(args[0]) != fin:
            continue
        by_fout[args[1].strip()] = by_fout.get(args[1].strip(), 0.0) + v["dram_bytes_per_launch"]
    return round(sum(by_fout.values()) / len(by_fout)) if by_fout else None


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines: list[str] = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_sample(config: str, seed: int, scale: float, steps: int = 1):
    """Time the oracle's gift_filter (fp64, reference order, OpenMP) on a scaled sample."""
    from oracle import oracle as orc
    from paper_2502_17632_b200 import synth

    fd = synth.generate(config, seed=seed, scale=scale)
    cap = fd.meta["max_clique_pins"]
    A = orc.build_clique_graph(fd.num_cells, fd.net_start, fd.pin_cell, cap)
    deg = orc.degrees(A)
    g = synth.signal_fp32(fd, seed=0).astype(np.float64)
    terms = [(2.0, 2, 0.1), (4.0, 2, 0.7), (4.0, 4, 0.2)]
    nnz_op = A.nnz + fd.num_cells
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        orc.gift_filter(A, g, terms, deg)
        times.append(time.perf_counter() - t0)
    return {
        "times": times, "nnz_op": nnz_op, "n": fd.num_cells, "cores": orc.num_threads(),
        "sample": f"{config} at scale {scale} ({fd.num_cells} cells, {fd.num_nets} nets, nnz_op {nnz_op}): "
                  f"oracle gift_filter (2 normalisations + 6 fp64 hops, csr_matvecs order)",
    }


def reference_giftplace(config: str, seed: int, scale: float, window=None):
    """The reference's own gift_filter (giftplace, gift.py:73-95: scipy, one
    core) on a design sample; None when the staged copy (oracle/_ref) is absent."""
    from oracle import oracle as orc
    from paper_2502_17632_b200 import synth

    gp = orc.reference_module()
    if gp is None:
        return None
    fd = synth.generate(config, seed=seed, scale=scale, window=window)
    d = fd.to_design(gp)
    adj = gp.build_clique_graph(d, max_clique_pins=fd.meta["max_clique_pins"])
    g = synth.signal_fp32(fd, seed=0).astype(np.float64)
    gp.gift_filter(adj, g)  # warm (imports, first-touch)
    t = []
    for _ in range(2):
        t0 = time.perf_counter()
        gp.gift_filter(adj, g)
        t.append(time.perf_counter() - t0)
    nnz_op = int(adj.nnz) + fd.num_cells
    per = min(t)
    return {"value": nnz_op * HOPS / per, "unit": UNIT, "cores": 1, "kind": "reference",
            "seconds_per_filter": round(per, 4),
            "sample": f"{config} at scale {scale} ({fd.num_cells} cells, nnz_op {nnz_op}): giftplace.gift_filter "
                      f"(the reference itself: 2 normalisations + 6 scipy csr matvec hops, single-threaded)"}


def run_reference(args) -> None:
    """Reference arm: the oracle port with every host thread, on the same
    full config as our arm; a step is one fp64 gift_filter (two
    normalisations + 6 hops in csr_matvecs order)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_2502_17632_b200 import synth

    fd = synth.generate(args.config, seed=args.seed)
    cap = fd.meta["max_clique_pins"]
    t0 = time.perf_counter()
    A = orc.build_clique_graph(fd.num_cells, fd.net_start, fd.pin_cell, cap)
    build_s = time.perf_counter() - t0
    deg = orc.degrees(A)
    g = synth.signal_fp32(fd, seed=0).astype(np.float64)
    terms = [(2.0, 2, 0.1), (4.0, 2, 0.7), (4.0, 4, 0.2)]
    nnz_op = A.nnz + fd.num_cells
    times = []
    for _ in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        orc.gift_filter(A, g, terms, deg)
        times.append(time.perf_counter() - t0)
    per = float(np.mean(times[args.warmup:]))
    value = nnz_op * HOPS / per
    sample = (f"{args.config} full size ({fd.num_cells} cells, {fd.num_nets} nets, nnz_op {nnz_op}): oracle port "
              f"gift_filter (fp64, csr_matvecs order, OpenMP over rows); graph build {build_s:.1f} s untimed")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} (same config as the GPU arm)", "seed": args.seed,
                   "n": fd.num_cells, "nnz_op": int(nnz_op), "same_config": True},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": orc.num_threads(), "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_oneshot(args) -> None:
    """One placement of a fresh design in a FRESH process (the reference's
    real use, cli.py:203-220): netlist arrays in host memory -> positions in
    host memory.  --oneshot python: build_clique_graph + gift_place (the
    drop-in API); --oneshot abi: gift_place_host (the C ABI).  Prints JSON."""
    t_proc = time.perf_counter()
    import torch

    import paper_2502_17632_b200 as gb
    from paper_2502_17632_b200 import synth

    import_s = time.perf_counter() - t_proc
    fd = synth.generate(args.config, seed=args.seed)
    cap = fd.meta["max_clique_pins"]
    cfg = gb.GiftConfig(seed=0, jitter_scale=10.0)
    g32 = synth.signal_fp32(fd, seed=0) if args.oneshot.startswith("abi") else None
    t0 = time.perf_counter()
    torch.cuda.init()
    from paper_2502_17632_b200 import _lib

    _lib.load_library()
    _lib.context(0)
    t1 = time.perf_counter()
    if args.oneshot in ("python", "python_factored"):
        adj = gb.build_clique_graph(fd, max_clique_pins=cap,
                                    implicit_above=FACTOR_ABOVE if args.oneshot == "python_factored" else None)
        t_b = time.perf_counter()
        placed, _ = gb.gift_place(fd, adj, cfg)
        nnz = adj.nnz
    else:
        t_b = None
        placed, nnz = gb.gift_place_arrays(fd.net_start, fd.pin_cell, g32, fd.fixed_mask(),
                                           fd.fixed_positions(), fd.region.bounds(), max_clique_pins=cap,
                                           implicit_above=FACTOR_ABOVE if args.oneshot == "abi_factored" else None)
    t2 = time.perf_counter()
    assert placed.shape == (fd.num_cells, 2) and np.isfinite(placed).all()
    out = {"api": {"python": "build_clique_graph + gift_place",
                   "python_factored": f"build_clique_graph(implicit_above={FACTOR_ABOVE}) + gift_place",
                   "abi": "gift_place_host (C ABI)",
                   "abi_factored": f"gift_place_host (C ABI, option implicit_above={FACTOR_ABOVE})"}[args.oneshot],
           "config": args.config, "nnz": int(nnz), "place_s": round(t2 - t1, 4),
           "cuda_init_s": round(t1 - t0, 4), "import_s": round(import_s, 3),
           "netlist_to_positions_s": round(t2 - t0, 4)}
    if t_b is not None:
        out["graph_build_s"] = round(t_b - t1, 4)
        out["gift_place_s"] = round(t2 - t_b, 4)
    print(json.dumps(out), flush=True)


def oneshot_e2e(config: str, seed: int) -> dict:
    """Both one-shot paths, each in its own fresh process."""
    res = {}
    for mode in ("python", "abi", "python_factored", "abi_factored"):
        try:
            p = subprocess.run([sys.executable, os.path.abspath(__file__), "--oneshot", mode, "--config", config,
                                "--seed", str(seed)], capture_output=True, text=True, timeout=600)
            res[mode] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else \
                {"error": p.stderr.strip().splitlines()[-1:] or ["rc %d" % p.returncode]}
        except Exception as e:  # reported, never fatal for the bench line
            res[mode] = {"error": repr(e)}
    res["note"] = ("fresh process each; netlist_to_positions_s = CUDA context + library load + graph build + "
                   "bank + epilogue + H2D/D2H, from host netlist arrays to host positions (python/torch import "
                   "excluded, listed as import_s)")
    return res


def self_launch(args) -> None:
    """`--gpus N` without a launcher: re-exec under torch.distributed.run with
    N ranks on this node (one process per GPU, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def dry_launch(args) -> None:
    """--dry-launch: form the process group (NCCL with GPUs, gloo without),
    check the ranks, print the world rank 0 saw.  CPU tests drive the launcher
    path with it."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if world > 1:
        dist.init_process_group(backend, init_method="env://")
        ranks = [None] * world
        dist.all_gather_object(ranks, {"rank": rank, "local_rank": local, "pid": os.getpid()})
        formed = dist.get_world_size()
    else:
        ranks, formed = [{"rank": 0, "local_rank": 0, "pid": os.getpid()}], 1
    if rank == 0:
        print(json.dumps({"dry_launch": True, "n_gpus": formed, "requested": args.gpus, "backend": backend,
                          "ranks": ranks}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c0", "c1", "c2", "c3", "c4"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-oneshot", action="store_true")
    ap.add_argument("--no-factored", action="store_true", help="skip the factored-clique-model leg")
    ap.add_argument("--factor-above", type=int, default=None, help="implicit_above of the factored leg")
    ap.add_argument("--scale", type=float, default=1.0, help=argparse.SUPPRESS)  # sweeps only: shrink the config
    ap.add_argument("--e2e-out", choices=["f32", "f64"], default="f32", help="placement dtype of the e2e leg")
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="kernel option (gift_ctx_set_option), e.g. tile_rows=4096; repeatable")
    ap.add_argument("--oneshot", choices=["python", "abi", "python_factored", "abi_factored"], default=None,
                    help=argparse.SUPPRESS)
    ap.add_argument("--exchange", choices=["peer", "nccl"], default="peer",
                    help="N > 1: ghost rows by NVLink peer loads (CUDA IPC) or by NCCL all_to_all")
    ap.add_argument("--dry-launch", action="store_true", help="form the process group and exit (launcher test)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.factor_above:
        global FACTOR_ABOVE
        FACTOR_ABOVE = args.factor_above
    if args.oneshot:
        run_oneshot(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)  # does not return
    if args.dry_launch:
        dry_launch(args)
        return

    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    n_formed = 1
    # GIFT_BENCH_SHARE_GPU=1 (launcher smoke test on a one-GPU box only): every
    # rank uses cuda:0 and the control group is gloo (NCCL refuses two ranks on
    # one device); the numbers of such a run mean nothing.
    share_gpu = os.environ.get("GIFT_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local = 0
    if world > 1:
        torch.cuda.set_device(local)
        if share_gpu:
            dist.init_process_group("gloo", init_method="env://")
        else:
            dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
        n_formed = dist.get_world_size()  # the group NCCL actually formed
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_2502_17632_b200 as gb
    from paper_2502_17632_b200 import _lib, synth

    lib = _lib.load_library()
    for kv in args.option:
        name, _, val = kv.partition("=")
        _lib.set_option(name, int(val))
    args.zero_copy = _lib._options.get("zero_copy", 1) != 0
    t0 = time.perf_counter()
    fd = synth.generate(args.config, seed=args.seed, scale=args.scale)
    gen_s = time.perf_counter() - t0
    cap = fd.meta["max_clique_pins"]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    adj = gb.build_clique_graph(fd, max_clique_pins=cap)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    n = adj.n
    nnz_op = adj.nnz + n
    unit_bytes = bytes_per_hop(nnz_op, n)

    g32 = synth.signal_fp32(fd, seed=0)
    mask = fd.fixed_mask().astype(np.uint8)
    fpos = np.nan_to_num(fd.fixed_positions(), nan=0.0)
    region = fd.region.bounds()
    sig = np.array([t.sigma for t in gb.DEFAULT_TERMS], dtype=np.float64)
    kk = np.array([t.k for t in gb.DEFAULT_TERMS], dtype=np.int64)
    al = np.array([t.alpha for t in gb.DEFAULT_TERMS], dtype=np.float64)
    ctx = _lib.context(local)
    sp_, kp_, ap_, rp_ = (sig.ctypes.data_as(_lib.c_dp), kk.ctypes.data_as(_lib.c_i64p),
                          al.ctypes.data_as(_lib.c_dp), region.ctypes.data_as(_lib.c_dp))
    if world == 1:
        r0, r1 = 0, n
    else:
        from paper_2502_17632_b200 import shard

        exchange_used = "nccl"
        sf = None
        if args.exchange == "peer":
            # every rank must take the same path: agree on whether the mappings worked
            ok = torch.ones(1, dtype=torch.int32, device=dev)
            try:
                sf = shard.cuda_sharded_filter(adj, world, rank, local,
                                               exchange=shard.PeerExchange(device=f"cuda:{local}"))
            except Exception as e:  # no peer access / IPC on this box
                print(f"[bench] rank {rank}: peer exchange unavailable ({e!r}); using NCCL", file=sys.stderr)
                ok.zero_()
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            exchange_used = "peer" if int(ok.item()) else "nccl"
        if exchange_used == "nccl":
            sf = shard.cuda_sharded_filter(adj, world, rank, local)
        r0, r1 = sf.plan.r0, sf.plan.r1
    dg = torch.from_numpy(np.ascontiguousarray(g32[r0:r1])).to(dev)
    dmask = torch.from_numpy(np.ascontiguousarray(mask[r0:r1])).to(dev)
    dpos = torch.from_numpy(np.ascontiguousarray(fpos[r0:r1])).to(dev)
    dout = torch.empty((r1 - r0, 2), dtype=torch.float64, device=dev)

    if world == 1:
        def step():
            _lib.check(lib.gift_filter(ctx, adj.handle, 3, sp_, kp_, ap_, 2, _lib.GIFT_DTYPE_F32, _lib.dptr(dg),
                                       _lib.GIFT_DTYPE_F64, _lib.dptr(dout), _lib.dptr(dmask), _lib.dptr(dpos),
                                       rp_, _lib.GIFT_PREC_FP32))
    else:
        def step():
            sf.run(dg, gb.DEFAULT_TERMS, dout, fixed_mask=dmask, fixed_pos=dpos, region=region)

    # warm-up: the first bank on the graph runs the row kernel (tiled policy
    # "on_reuse": a one-shot graph never pays for the tiled copy); the second
    # builds the tiled copies (cached on the graph, like its degrees)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    first_call_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    second_call_s = time.perf_counter() - t0
    for _ in range(args.warmup - 2):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, device events, max over ranks ----
    # Per-launch CUDA events (the roofline's kernel times) ride inside the
    # timed region, except on graphs small enough for the bank's CUDA-graph
    # replay (below the tiled hop's row threshold): per-launch events disable the replay, so there
    # the kernel times come from a profiled pass right after the timed one.
    tiled_thr = _lib._options.get("tiled_min_rows", _lib.DEFAULT_OPTIONS["tiled_min_rows"])
    graph_replay = world == 1 and n < min(tiled_thr, 262144)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    _lib.set_profiling(not graph_replay, local)
    _lib.drain_profile(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count(local)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count(local) - launches0
    recs = _lib.drain_profile(local)
    _lib.set_profiling(False, local)
    clk = clocks.stop()
    if graph_replay:
        _lib.set_profiling(True, local)
        for _ in range(args.steps):
            step()
        recs = _lib.drain_profile(local)
        _lib.set_profiling(False, local)
    ms = ev0.elapsed_time(ev1)
    t_rank = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_rank, op=dist.ReduceOp.MAX)
    ms_max = float(t_rank.item())
    per_step_ms = ms_max / args.steps
    # one graph per step whatever N is (row-sharded): strong scaling
    value = nnz_op * HOPS * args.steps / (ms_max / 1e3)

    # ---- roofline of the dominant kernel (rank-local bytes when sharded) ----
    pk = peaks()
    # this rank's stored entries (no host mirror of the graph: block shapes)
    local_nnz_op = (adj.nnz if world == 1 else sf.block_nnz()) + (r1 - r0)
    local_unit_bytes = bytes_per_hop(local_nnz_op, r1 - r0)
    by_kind: dict[int, list] = {}
    for kind, units, t in recs:
        by_kind.setdefault(kind, []).append((units, t))
    kernels = {}
    for kind, lst in by_kind.items():
        tot = sum(t for _, t in lst)
        kernels[kind] = {"launches": len(lst), "mean_ms": tot / len(lst), "share": tot, "units": lst[0][0],
                         "bytes": lst[0][0] * local_unit_bytes}
    total_prof = sum(k["share"] for k in kernels.values()) or 1.0
    hop_kinds = [k for k in kernels if k > 0]
    dom = max(hop_kinds, key=lambda k: kernels[k]["share"]) if hop_kinds else None

    tinfo = adj.tiled_info() if world == 1 else None

    def stored_bytes(kind):
        """Bytes this pass must move, counted live from the graph being timed:
        its tiled copy's stored slots (6 B each: u16 column + f32 weight) and
        residual CSR, or the CSR's (column, fp32 weight) pairs on the row
        kernel, plus one read and one write of the signal and the per-row
        vectors (s per chain, bank accumulator).  A lower bound on DRAM
        traffic that needs no profiler; the ncu capture (`traffic`) is the
        measured figure."""
        rows = n * (4 * kind + 4 * kind + 4 * max(kind // 2, 1) + 16)
        t = (tinfo or {}).get("f4" if kind == 4 else "f2") or {}
        if t.get("built") and t.get("usable"):
            return 6 * t["slots"] + rows
        return 8 * adj.nnz + 8 * n + rows

    def roof(kind):
        k = kernels[kind]
        ach = k["bytes"] / (k["mean_ms"] / 1e3) / 1e9
        traffic = ncu_traffic(args.config, kind) if world == 1 else None
        dram = traffic / (k["mean_ms"] / 1e3) / 1e9 if traffic else None
        stored = stored_bytes(kind) if world == 1 else None
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / pk["hbm_gbs"], 4), "traffic": traffic,
                "dram_achieved": round(dram, 1) if dram else None,
                "dram_frac": round(dram / pk["hbm_gbs"], 4) if dram else None,
                "stored_bytes": stored,
                "stored_frac": round(stored / (k["mean_ms"] / 1e3) / 1e9 / pk["hbm_gbs"], 4) if stored else None,
                "note": ("algorithmic bytes = units x (8 nnz_op + 24 N + 8); a launch advancing 2 packed "
                         "sigma-chains reads the matrix once for 2 hop units, and the BMT copy stores 6 B "
                         "per entry, so achieved (algorithmic) can exceed the copy peak; dram_* is the "
                         "ncu-measured DRAM traffic over the same launch time; stored_* counts, live from the "
                         "timed graph, the bytes the pass must move (6 B per stored slot + signal and row "
                         "vectors): a profiler-free lower bound on the same fraction"),
                "kernel": f"k_hop<FIN={kind}> ({k['units']} hop unit(s)/launch)",
                "bytes_per_launch": k["bytes"], "mean_launch_ms": round(k["mean_ms"], 5),
                "share_of_step": round(k["share"] / total_prof, 4), "peak_source": pk["source"]}

    roofline = roof(dom) if (dom is not None and world == 1) else None
    kernels_report = {f"k_hop_F{k}" if k else "k_prep": roof(k) if (k and world == 1) else
                      {"mean_launch_ms": round(v["mean_ms"], 5), "launches": v["launches"],
                       "share_of_step": round(v["share"] / total_prof, 4)}
                      for k, v in kernels.items()}

    # ---- e2e: host buffers in, host placement out, every step ----
    h_g = torch.from_numpy(np.ascontiguousarray(g32[r0:r1])).pin_memory()
    h_mask = torch.from_numpy(np.ascontiguousarray(mask[r0:r1])).pin_memory()
    h_pos = torch.from_numpy(np.ascontiguousarray(fpos[r0:r1])).pin_memory()
    # the configs ask for an N x 2 fp32 placement (BASELINE.json configs[0]);
    # fp32 output also halves the device-to-host bytes
    e2e_f64 = args.e2e_out == "f64"
    h_out = torch.empty((r1 - r0, 2), dtype=torch.float64 if e2e_f64 else torch.float32).pin_memory()

    if world == 1:
        e2e_api = ("gift_filter_host (C ABI, pinned host buffers; output written in place by the final hop; "
                   f"{args.e2e_out} placement)"
                   if args.zero_copy else "gift_filter_host (C ABI, pinned host buffers)")

        def step_e2e():
            _lib.check(lib.gift_filter_host(ctx, adj.handle, 3, sp_, kp_, ap_, 2, _lib.GIFT_DTYPE_F32,
                                            _lib.c_vp(h_g.data_ptr()),
                                            _lib.GIFT_DTYPE_F64 if e2e_f64 else _lib.GIFT_DTYPE_F32,
                                            _lib.c_vp(h_out.data_ptr()), _lib.c_vp(h_mask.data_ptr()),
                                            _lib.c_vp(h_pos.data_ptr()), rp_, _lib.GIFT_PREC_FP32))
    else:
        e2e_api = "ShardedFilter.run with per-rank pinned H2D/D2H"

        def step_e2e():
            dg.copy_(h_g, non_blocking=True)
            dmask.copy_(h_mask, non_blocking=True)
            dpos.copy_(h_pos, non_blocking=True)
            step()
            h_out.copy_(dout.to(h_out.dtype), non_blocking=True)
            torch.cuda.current_stream().synchronize()

    for _ in range(2):
        step_e2e()
    k_e2e = args.e2e_steps or args.steps
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k_e2e):
        step_e2e()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    t_e = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
    e2e_value = nnz_op * HOPS * k_e2e / float(t_e.item())
    zero_copy = world == 1 and args.zero_copy
    if zero_copy:  # pinned buffers used in place: fixed centres cross the bus for fixed rows only
        h2d = g32.nbytes + mask.nbytes + int(mask.sum()) * 16
    elif world == 1:
        h2d = g32.nbytes + mask.nbytes + fpos.nbytes
    else:
        h2d = int(h_g.numel() * 4 + h_mask.numel() + h_pos.numel() * 8)
    d2h = (r1 - r0) * 2 * (8 if e2e_f64 else 4)

    # ---- CPU baseline (rank 0, N = 1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        scale = SAMPLE_SCALE[args.config]
        res = cpu_sample(args.config, args.seed, scale, steps=2)
        per = min(res["times"])
        cpu = {"value": res["nnz_op"] * HOPS / per, "unit": UNIT, "cores": res["cores"], "kind": "port",
               "sample": res["sample"]}
        ref = {}
        for cfg_, sc_ in (("c1", 1.0), (args.config, scale)):
            try:
                r_ = reference_giftplace(cfg_, args.seed, sc_)
            except Exception as e:  # the reference is a reported baseline; never fatal
                r_ = {"error": repr(e)}
            if r_ is not None:
                ref[f"{cfg_}@{sc_}"] = r_
        cpu["reference"] = ref or None
    oneshot = None
    if rank == 0 and world == 1 and not args.no_oneshot:
        oneshot = oneshot_e2e(args.config, args.seed)

    # ---- the factored clique model (opt-in extension; not the headline) ----
    # Same operator, same seed, same bank: nets with more than FACTOR_ABOVE
    # pins are applied as the O(pins) implicit term instead of being stored
    # as O(pins^2) entries (build_clique_graph(..., implicit_above=T)).
    factored = None
    if rank == 0 and world == 1 and not args.no_factored:
        try:
            step()
            torch.cuda.synchronize()
            explicit_out = dout.cpu().numpy()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            adj_f = gb.build_clique_graph(fd, max_clique_pins=cap, implicit_above=FACTOR_ABOVE)
            torch.cuda.synchronize()
            fbuild_s = time.perf_counter() - t0

            def step_f():
                _lib.check(lib.gift_filter(ctx, adj_f.handle, 3, sp_, kp_, ap_, 2, _lib.GIFT_DTYPE_F32, _lib.dptr(dg),
                                           _lib.GIFT_DTYPE_F64, _lib.dptr(dout), _lib.dptr(dmask), _lib.dptr(dpos),
                                           rp_, _lib.GIFT_PREC_FP32))

            for _ in range(args.warmup):
                step_f()
            torch.cuda.synchronize()
            fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            fe0.record()
            for _ in range(args.steps):
                step_f()
            fe1.record()
            torch.cuda.synchronize()
            f_ms = fe0.elapsed_time(fe1) / args.steps
            f_out = dout.cpu().numpy()
            _lib.set_profiling(True, local)
            for _ in range(3):
                step_f()
            torch.cuda.synchronize()
            f_recs = _lib.drain_profile(local)
            _lib.set_profiling(False, local)
            f_pass = {}
            for kind, _units, t in f_recs:
                f_pass.setdefault(kind, []).append(t)
            dev_l2 = float(np.linalg.norm(f_out - explicit_out) / np.linalg.norm(explicit_out))
            factored = {
                "implicit_above": FACTOR_ABOVE, "ms_per_step": round(f_ms, 4),
                "value": nnz_op * HOPS / (f_ms / 1e3), "unit": UNIT + " (of the explicit graph it replaces)",
                "graph_build_s": round(fbuild_s, 3), "explicit_nnz": adj_f.nnz, "implicit_nets": adj_f.implicit_nets,
                "pass_ms": {(f"F{k}" if k else "prep"): round(sum(v) / len(v), 5) for k, v in f_pass.items()},
                "rel_l2_vs_explicit_path": dev_l2,
                "note": "opt-in: build_clique_graph(..., implicit_above=T); same operator as the reference's capped "
                        "clique graph in exact arithmetic, parity-tested against the oracle "
                        "(tests/test_gpu_parity.py::test_factored_clique_model_matches_oracle)",
            }
            del adj_f
        except Exception as e:  # an extension leg: never fatal to the bench line
            factored = {"error": repr(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_formed, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step_ms, "higher_is_better": True,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "scaling": "strong" if world > 1 else "weak",
            "config": {
                "workload": f"{args.config}{'' if args.scale == 1.0 else f' x{args.scale}'}: {fd.meta['n_mov']} movable + {fd.meta['n_macros']} macros + "
                            f"{fd.meta['n_pads']} pads, {fd.meta['n_nets']} nets, max_clique_pins={cap}, "
                            f"default bank (6 hops), fp32 fused path",
                "n": n, "nnz": adj.nnz, "nnz_op": nnz_op, "hops": HOPS, "seed": args.seed,
                "bytes_per_hop_unit": unit_bytes,
                "l2": "inputs larger than L2 (CSR col+w32 = %.2f GB per pass)" % (8 * adj.nnz / 1e9),
                "parallelism": (f"row-sharded x{world} (ghost rows pulled over NVLink peer memory per hop)"
                                if exchange_used == "peer" else
                                f"row-sharded x{world} (NCCL ghost all_to_all per hop)") if world > 1
                else "single GPU",
                "kernel_times": "per-launch CUDA events in the timed region" if not graph_replay else
                "per-launch CUDA events in a profiled pass after the timed region (the timed steps replay the "
                "bank as a CUDA graph)",
                "options": dict(_lib._options) or "defaults",
                "graph_build_s": round(build_s, 3), "generate_s": round(gen_s, 3),
                "first_filter_call_s": round(first_call_s, 3),
                "second_filter_call_s": round(second_call_s, 3),
                "tiled": adj.tiled_info() if world == 1 else None,
            },
            "roofline": roofline,
            "kernels": kernels_report,
            "effective_bank_gbs": round(HOPS * unit_bytes / (per_step_ms / 1e3) / 1e9, 1),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "api": e2e_api,
                    "ms_per_step": 1e3 * float(t_e.item()) / k_e2e},
            "oneshot_e2e": oneshot,
            "factored": factored,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
