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
