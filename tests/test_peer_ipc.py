"""GPU: the peer-memory ghost exchange across PROCESSES (real CUDA IPC).

Two processes share the one GPU of the test box; each owns a row block of
the same graph, allocates its signal buffers with gift_peer_alloc, publishes
the CUDA IPC handles through the (gloo) control group and opens the other's
(gift_peer_open) -- the exact shard.PeerExchange code a multi-GPU run uses,
except that the mapped memory sits on the same device instead of behind
NVLink, and the per-hop barrier is the host one (device synchronise + gloo
barrier), so no kernel of one process ever waits on the other's.  The
gathered placement must match the single-GPU bank.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

FP32_TOL = 1e-5


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2502_17632_b200 as gb
        from paper_2502_17632_b200 import shard, synth

        torch.cuda.set_device(0)
        fd = synth.generate("c2", seed=4, scale=0.02, window=600)
        adj = gb.build_clique_graph(fd, max_clique_pins=200)
        g32 = synth.signal_fp32(fd, seed=2)
        ex = shard.PeerExchange(device="cuda:0")
        assert not ex.nccl
        sf = shard.cuda_sharded_filter(adj, world, rank, 0, exchange=ex)
        r0, r1 = sf.plan.r0, sf.plan.r1
        g = torch.from_numpy(np.ascontiguousarray(g32[r0:r1])).cuda()
        out = torch.zeros((r1 - r0, 2), dtype=torch.float64, device="cuda")
        mask = torch.from_numpy(fd.fixed_mask()[r0:r1].astype(np.uint8)).cuda()
        pos = torch.from_numpy(np.nan_to_num(fd.fixed_positions()[r0:r1], nan=0.0)).cuda()
        sf.run(g, gb.DEFAULT_TERMS, out, fixed_mask=mask, fixed_pos=pos, region=fd.region.bounds())
        first = out.clone()
        sf.run(g, gb.DEFAULT_TERMS, out, fixed_mask=mask, fixed_pos=pos, region=fd.region.bounds())
        torch.cuda.synchronize()
        same = bool(torch.equal(first, out))
        opened = len(ex._opened)
        ex.close(sf.be)
        gathered = [None] * world if rank == 0 else None
        dist.gather_object((r0, out.cpu().numpy(), sf.plan.n_ghost, same, opened), gathered, dst=0)
        if rank == 0:
            full = np.zeros((fd.num_cells, 2))
            for r0_, blk, *_ in gathered:
                full[r0_:r0_ + len(blk)] = blk
            ref = gb.gift_filter(adj, g32)  # the single-GPU bank on the same seed signal
            r = fd.region.bounds()
            want = np.clip(ref, r[:2], r[2:])
            mk = fd.fixed_mask()
            want[mk] = fd.fixed_positions()[mk]
            err = float(np.linalg.norm(full - want) / np.linalg.norm(want))
            results.put({"err": err, "same": [x[3] for x in gathered], "ghosts": [x[2] for x in gathered],
                         "opened": [x[4] for x in gathered],
                         "fixed_exact": bool(np.array_equal(full[mk], fd.fixed_positions()[mk]))})
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_exchange_between_two_processes_on_one_gpu():
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = q.get(timeout=10)
    assert res["err"] <= FP32_TOL, res
    assert res["fixed_exact"]
    assert all(res["same"]), res
    assert all(g > 0 for g in res["ghosts"])
    assert res["opened"] == [2, 2]  # each rank mapped the other's two buffers
