"""CPU: the row-sharded multi-GPU path's host logic, end to end over gloo.

world_size 2 and 3 processes run shard.ShardedFilter -- the same bank
schedule, partition, ghost lists and per-hop all_to_all exchange the NCCL
path uses -- with a numpy stand-in for the k_hop kernel (same split
local/ghost semantics and epilogue), then compare the gathered placement
with the oracle's gift_place (fp64 reference order) at the fp32 tolerance.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2502_17632_b200 import shard

FP32_TOL = 1e-5
DEFAULT = [(2.0, 2, 0.1), (4.0, 2, 0.7), (4.0, 4, 0.2)]


class NumpyBackend:
    """k_hop / k_prep / gather semantics in numpy (fp32), on torch CPU tensors."""

    def empty(self, rows, cols, dtype="f32"):
        import torch

        return torch.zeros((max(rows, 1), cols), dtype=torch.float32 if dtype == "f32" else torch.float64)

    def upload(self, arr):
        import torch

        return torch.from_numpy(np.ascontiguousarray(arr))

    def block(self, indptr, indices, values):
        import scipy.sparse as sp

        n = len(indptr) - 1
        ncols = int(indices.max()) + 1 if len(indices) else 1
        return sp.csr_matrix((np.asarray(values, np.float64).astype(np.float32), indices, indptr),
                             shape=(n, max(ncols, 1)))

    def pack(self, n, wcols, s_list, g, ld, c0, F, zflat):
        z = zflat.numpy()[: n * F].reshape(n, F)
        z[:] = 0
        gn = g.numpy().reshape(n, ld)
        for j, s in enumerate(s_list):
            z[:, j * wcols:(j + 1) * wcols] = s[:, None] * gn[:, c0:c0 + wcols].astype(np.float32)

    def gather(self, idx, F, src, dst):
        s = src.numpy().reshape(-1, F)
        dst.numpy()[: len(idx) * F] = s[idx.numpy()].reshape(-1)

    def pull(self, n_rows, F, peers, src_rank, src_row, dst):
        """gift_pull_rows_f32 (csrc/peer.cu): dst[i] = peers[src_rank[i]][src_row[i]], rows of F floats."""
        rk, rw = src_rank.numpy(), src_row.numpy()
        d = dst.numpy()[: n_rows * F].reshape(n_rows, F)
        for q in np.unique(rk):
            sel = rk == q
            d[sel] = np.asarray(peers[q]).reshape(-1)[: (len(peers[q].reshape(-1)) // F) * F].reshape(-1, F)[rw[sel]]

    def pull_join(self):
        pass

    def hop(self, A, d):
        n, fin = d["row_end"], d["fin"]
        zin = d["zin"].numpy().reshape(-1, fin)
        zpad = np.zeros((max(A.shape[1], 1), fin), np.float32)
        m = min(len(zin), A.shape[1])
        zpad[:m] = zin[:m]
        acc = (A @ zpad).astype(np.float32)[:n]
        if d.get("part_out") is not None:
            d["part_out"].numpy()[: n * fin] = acc.reshape(-1)
            return
        if d.get("part_in") is not None:
            acc = d["part_in"].numpy()[: n * fin].reshape(n, fin) + acc
        wcols = d["wcols"]
        accbuf = d["acc"].numpy()
        o = np.zeros((n, wcols), np.float32)
        any_term = any(c["has_term"] for c in d["chains"])
        if any_term and d["acc_read"]:
            o[:] = accbuf.reshape(-1, 4)[:n, :wcols]
        fout = d["fout"]
        zout = d["zout"].numpy().reshape(-1, fout) if fout else None
        for f in range(len(d["chains"]) * wcols):
            ch = d["chains"][f // wcols]
            cc = f % wcols
            s = ch["s"][:n]
            y = s * (acc[:, f] + np.float32(ch["sigma"]) * zin[:n, f])
            if fout and ch["cont"] >= 0:
                zout[:n, ch["cont"] * wcols + cc] = s * y
            if ch["has_term"]:
                o[:, cc] = o[:, cc] + np.float32(ch["alpha"]) * y
        if not any_term:
            return
        if not d["is_final"]:
            accbuf.reshape(-1, 4)[:n, :wcols] = o
            return
        out = d["out"].numpy()
        v = o.astype(np.float64)
        mask = d.get("fixed_mask")
        if mask is not None:
            mk = mask.numpy().astype(bool)
            pos = d["fixed_pos"].numpy()
            reg = d["region"]
            for c in range(2):
                x = np.clip(v[:, c], reg[c], reg[c + 2])
                v[:, c] = np.where(mk, pos[:, c], x)
        out[:, d["out_c0"]:d["out_c0"] + wcols] = v


class MemmapPeerExchange(shard.PeerExchange):
    """CPU stand-in for NVLink peer memory: every rank's two signal buffers
    are files mapped by all ranks (one-sided reads, like CUDA IPC mappings);
    the per-hop barrier is a gloo barrier.  Runs PeerExchange's own schedule
    (barrier placement, pull tables) with the numpy backend."""

    def __init__(self, tmpdir):
        self.tmpdir = tmpdir
        self.plan = None
        self._ids = shard.TorchExchange(device="cpu")
        self.tables = []
        self.barriers = 0

    def alloc_signal(self, be, rows, plan):
        import torch
        import torch.distributed as dist

        rows = max(rows, 1)
        sizes = [None] * plan.world
        dist.all_gather_object(sizes, rows)
        mine = [np.lib.format.open_memmap(os.path.join(self.tmpdir, f"z{w}_{plan.rank}.npy"), mode="w+",
                                          dtype=np.float32, shape=(rows, 4)) for w in range(2)]
        for m in mine:
            m[:] = 0
            m.flush()
        dist.barrier()
        for w in range(2):
            self.tables.append([mine[w] if q == plan.rank else
                                np.lib.format.open_memmap(os.path.join(self.tmpdir, f"z{w}_{q}.npy"), mode="r")
                                for q in range(plan.world)])
        self._finish_tables(be, plan)
        return torch.from_numpy(mine[0]), torch.from_numpy(mine[1])

    def barrier(self):
        import torch.distributed as dist

        self.barriers += 1
        dist.barrier()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results, scale, window, mode="a2a", tmpdir=None):
    import torch
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_2502_17632_b200 import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fd = synth.generate("c2", seed=3, scale=scale, window=window)
        A = orc.build_clique_graph(fd.num_cells, fd.net_start, fd.pin_cell, 200)
        deg = orc.degrees(A)
        ex = shard.TorchExchange(device="cpu") if mode == "a2a" else MemmapPeerExchange(tmpdir)
        bounds = shard.nnz_balanced_bounds(A.indptr, world)
        ghosts, loc, gh = shard.split_block(A.indptr, A.indices, int(bounds[rank]), int(bounds[rank + 1]))
        plan = shard.exchange_plan(bounds, rank, ghosts, ex.ids)
        s_of = lambda sigma: (1.0 / np.sqrt(deg + sigma)).astype(np.float32)[plan.r0:plan.r1]  # noqa: E731
        be = NumpyBackend()
        sf = shard.ShardedFilter(plan, be.block(loc[0], loc[1], A.data[loc[2]]), be.block(gh[0], gh[1], A.data[gh[2]]),
                                 be, ex, s_of)
        g32 = synth.signal_fp32(fd, seed=1)
        r0, r1 = plan.r0, plan.r1
        g = torch.from_numpy(np.ascontiguousarray(g32[r0:r1]))
        out = torch.zeros((r1 - r0, 2), dtype=torch.float64)
        mask = torch.from_numpy(fd.fixed_mask()[r0:r1].astype(np.uint8))
        pos = torch.from_numpy(np.nan_to_num(fd.fixed_positions()[r0:r1], nan=0.0))
        sf.run(g, DEFAULT, out, fixed_mask=mask, fixed_pos=pos, region=fd.region.bounds())
        if mode == "pull":  # a second bank on the same buffers (the barrier before the pack protects them)
            first = out.clone()
            sf.run(g, DEFAULT, out, fixed_mask=mask, fixed_pos=pos, region=fd.region.bounds())
            assert torch.equal(first, out)
            assert ex.barriers == 2 * (1 + 4)  # one per pack, one per hop of the 4-pass default bank
        # plan invariants
        inv = {
            "recv": int(sum(plan.recv_counts)) == plan.n_ghost,
            "ghost_sorted": bool(np.all(np.diff(plan.ghosts) > 0)),
            "ghost_not_owned": bool(np.all((plan.ghosts < r0) | (plan.ghosts >= r1))),
            "send_in_range": bool(np.all((plan.send_rows >= 0) & (plan.send_rows < r1 - r0))),
            "nnz_split": int(loc[0][-1] + gh[0][-1]) == int(A.indptr[r1] - A.indptr[r0]),
        }
        gathered = [None] * world if rank == 0 else None
        dist.gather_object((r0, out.numpy(), inv, plan.n_ghost), gathered, dst=0)
        if rank == 0:
            full = np.zeros((fd.num_cells, 2))
            invs = []
            for r0_, blk, iv, ng in gathered:
                full[r0_:r0_ + len(blk)] = blk
                invs.append(iv)
            want = orc.place_epilogue(orc.gift_filter(A, g32.astype(np.float64), DEFAULT, deg), fd.fixed_mask(),
                                      fd.fixed_positions(), fd.region.bounds())
            err = float(np.linalg.norm(full - want) / np.linalg.norm(want))
            mk = fd.fixed_mask()
            results.put({"err": err, "fixed_exact": bool(np.array_equal(full[mk], fd.fixed_positions()[mk])),
                         "inv": invs, "ghosts": [x[3] for x in gathered]})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "a2a"), (3, "a2a"), (2, "pull"), (3, "pull")])
def test_sharded_bank_over_gloo_matches_oracle(world, mode, tmp_path):
    """mode "a2a": packed rows through all_to_all_single (TorchExchange);
    mode "pull": one-sided reads of the owners' buffers between per-hop
    barriers (PeerExchange's schedule; mapped files stand in for peer memory)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, 0.01, 300, mode, str(tmp_path)))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = q.get(timeout=10)
    assert res["err"] <= FP32_TOL, res
    assert res["fixed_exact"]
    for iv in res["inv"]:
        assert all(iv.values()), iv
    assert all(g > 0 for g in res["ghosts"])


def test_bank_plan_matches_reference_grouping():
    plan = shard.plan_bank(DEFAULT, 2)
    assert plan.sigmas == [2.0, 4.0]
    hops = [s for s in plan.steps if isinstance(s, shard.HopStep)]
    assert [h.fin for h in hops] == [4, 4, 2, 2]
    assert [h.fout for h in hops] == [4, 2, 2, 0]
    assert plan.hops == 6
    assert hops[1].chains[0].alpha == 0.1 and hops[1].chains[1].alpha == 0.7
    assert hops[-1].is_final == 1 and hops[-1].chains[0].alpha == 0.2
    # first-appearance sigma order and stable k order
    p2 = shard.plan_bank([(3.0, 1, 0.2), (1.0, 3, 0.25), (3.0, 1, 0.1), (0.5, 2, 0.3)], 2)
    assert p2.sigmas == [3.0, 1.0, 0.5]
    with pytest.raises(ValueError):
        shard.plan_bank([], 2)


def test_nnz_balanced_bounds():
    indptr = np.concatenate([[0], np.cumsum(np.r_[np.full(100, 10), np.full(100, 1)])])
    b = shard.nnz_balanced_bounds(indptr, 4)
    assert b[0] == 0 and b[-1] == 200 and np.all(np.diff(b) >= 0)
    work = np.diff((indptr + np.arange(201))[b])
    assert work.max() <= 1.2 * work.mean()
