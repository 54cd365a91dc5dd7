"""CPU: bench.py's multi-GPU launcher path.

`python bench.py --gpus N` (no WORLD_SIZE in the environment) re-executes
itself under torch.distributed.run with N ranks; `--dry-launch` forms the
process group (gloo here, NCCL on GPUs) and rank 0 prints the world it saw.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [2, 3])
def test_bench_launches_its_own_ranks(n):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--dry-launch"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["dry_launch"] and line["n_gpus"] == n and line["requested"] == n
    assert line["backend"] == "gloo"
    assert sorted(r["rank"] for r in line["ranks"]) == list(range(n))
    assert len({r["pid"] for r in line["ranks"]}) == n  # one process per rank


def test_bench_single_gpu_does_not_relaunch():
    env = {k: v for k, v in os.environ.items() if k != "WORLD_SIZE"}
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-launch"], capture_output=True,
                       text=True, timeout=300, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and len(line["ranks"]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ["peer", "nccl"])
def test_bench_two_ranks_sharing_the_gpu(exchange):
    """`bench.py --gpus 2` end to end on the one GPU of the test box: the
    launcher, two ranks, the device-side row split, the sharded bank and the
    JSON line.  GIFT_BENCH_SHARE_GPU=1 puts both ranks on cuda:0 with a gloo
    control group (NCCL refuses two ranks on one device); with --exchange peer
    the ghost rows still cross process boundaries through real CUDA IPC
    mappings.  A smoke test of the code path, not a measurement."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env["GIFT_BENCH_SHARE_GPU"] = "1"
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "3",
                        "--warmup", "3", "--exchange", exchange], capture_output=True, text=True, timeout=900,
                       cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["value"] > 0
    want = "peer memory" if exchange == "peer" else "all_to_all"
    assert want in line["config"]["parallelism"], line["config"]["parallelism"]
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
