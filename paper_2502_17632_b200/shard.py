"""Row-sharded GiFt filter bank over several GPUs (one process per GPU).

SURVEY.md §8(e): rows are independent given the signal, so the CSR is cut
into contiguous, nnz-balanced row blocks; the only exchange is, per hop, the
signal rows a block's columns reference outside the block ("ghosts").  For
netlists with index locality (every net inside a +-W window) the ghosts are a
2W-row halo on each side plus the fixed objects (pads/macros) referenced from
everywhere.

Per hop, each rank
  1. gets its ghost rows moving:
     * PeerExchange (NVLink peer memory, the default on GPUs): a stream-ordered
       barrier, then ONE kernel of peer loads pulls the ghost rows straight
       out of the owners' signal buffers (CUDA IPC mappings, csrc/peer.cu) on
       a forked stream -- no pack kernel, no staging, no collective;
     * TorchExchange (NCCL / gloo): packs the rows other ranks asked for
       (gift_gather_rows_f32) and starts an async all_to_all_single;
  2. runs the LOCAL part of the hop (columns it owns) -> partial row sums,
     overlapping the transfer,
  3. waits for the transfer (stream-ordered; the host never blocks),
  4. runs the GHOST part (columns owned elsewhere) plus the epilogue.  The bank schedule (chain packing, term accumulation,
fused re-pin/clamp) is `plan_bank`, the host mirror of bank_fp32 in
csrc/filter.cu; the numeric kernels are the same k_hop instances.

Degrees and s_sigma come from the FULL rows each rank owns, so they are the
single-GPU values bit for bit; only fp32 summation order differs (split
local/ghost partial sums), well inside the 1e-5 tolerance.

Everything except the kernel calls is backend-neutral: `CudaBackend` calls the
C ABI; tests drive the same schedule and exchange over gloo with a numpy
backend (tests/test_shard.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

# ------------------------------------------------------------------ bank plan


@dataclass
class ChainStep:
    group: int        # index into the sigma groups
    cont: int         # slot in zout, -1 if the chain ends here
    has_term: int
    alpha: float


@dataclass
class PackStep:
    c0: int
    wcols: int
    groups: list[int]
    F: int


@dataclass
class HopStep:
    c0: int
    wcols: int
    chains: list[ChainStep]
    fin: int
    fout: int
    acc_read: int
    is_final: int
    any_term: int


@dataclass
class BankPlan:
    sigmas: list[float]
    steps: list = field(default_factory=list)

    @property
    def hops(self) -> int:
        return sum(len(s.chains) for s in self.steps if isinstance(s, HopStep))


def _pow2(v: int) -> int:
    p = 1
    while p < v:
        p <<= 1
    return p


def plan_bank(terms, ncols: int) -> BankPlan:
    """Chain packing of gift.py:83-94: sigma groups in first-appearance order,
    each group's terms stable-sorted by k; groups packed 4 // wcols per pass."""
    groups: list[list] = []
    sigmas: list[float] = []
    for t in terms:
        sigma, k, alpha = (t.sigma, t.k, t.alpha) if hasattr(t, "sigma") else t
        if sigma < 0:
            raise ValueError(f"sigma must be >= 0, got {sigma}")
        if k < 1:
            raise ValueError(f"power k must be >= 1, got {k}")
        if sigma not in sigmas:
            sigmas.append(sigma)
            groups.append([])
        groups[sigmas.index(sigma)].append((int(k), float(alpha)))
    if not groups:
        raise ValueError("filter needs at least one term")
    for g in groups:
        g.sort(key=lambda x: x[0])  # list.sort is stable
    plan = BankPlan(sigmas=sigmas)
    for c0 in range(0, ncols, 4):
        wcols = min(4, ncols - c0)
        per = max(1, 4 // wcols)
        acc_written = False
        for g0 in range(0, len(groups), per):
            pack = list(range(g0, min(g0 + per, len(groups))))
            last_pack = pack[-1] == len(groups) - 1
            maxk = max(groups[j][-1][0] for j in pack)
            plan.steps.append(PackStep(c0, wcols, pack, _pow2(wcols * len(pack))))
            active = list(pack)
            for h in range(1, maxk + 1):
                nxt, chains, any_term = [], [], 0
                for j in active:
                    al = sum(a for k, a in groups[j] if k == h)
                    has = int(any(k == h for k, _ in groups[j]))
                    any_term |= has
                    if groups[j][-1][0] > h:
                        cont = len(nxt)
                        nxt.append(j)
                    else:
                        cont = -1
                    chains.append(ChainStep(j, cont, has, al))
                plan.steps.append(HopStep(
                    c0, wcols, chains, _pow2(wcols * len(active)), _pow2(wcols * len(nxt)) if nxt else 0,
                    int(acc_written), int(last_pack and h == maxk), any_term))
                if any_term:
                    acc_written = True
                active = nxt
    return plan


# ------------------------------------------------------------------ partition


def nnz_balanced_bounds(indptr: np.ndarray, world: int) -> np.ndarray:
    """Row boundaries r_0 = 0 < ... < r_P = n splitting nnz (+1 per row) evenly."""
    indptr = np.asarray(indptr, dtype=np.int64)
    n = len(indptr) - 1
    work = indptr + np.arange(n + 1)  # count each row once so empty rows still spread
    targets = (np.arange(1, world) * work[-1]) // world
    cuts = np.searchsorted(work, targets, side="left")
    b = np.concatenate([[0], np.clip(cuts, 0, n), [n]]).astype(np.int64)
    return np.maximum.accumulate(b)


@dataclass
class ShardPlan:
    """This rank's exchange lists.  Column ids of its blocks index
    z_ext = [owned rows | ghost rows]; `ghosts` are the global ids of the
    ghost rows, ascending (grouped by owner, since owners hold contiguous
    row ranges)."""

    world: int
    rank: int
    bounds: np.ndarray          # [world+1]
    r0: int
    r1: int
    ghosts: np.ndarray          # sorted global ids this rank reads but does not own
    recv_counts: list[int]      # ghosts owned by each rank (grouped, ascending)
    send_counts: list[int]      # rows each rank asked this rank for
    send_rows: np.ndarray       # local row ids to pack, grouped by destination rank

    @property
    def n_local(self) -> int:
        return self.r1 - self.r0

    @property
    def n_ghost(self) -> int:
        return len(self.ghosts)


def split_block(indptr, indices, r0, r1):
    """Host restatement of gift_csr_split_rows (csrc/shard.cu), used by the CPU
    tests: rows [r0, r1) -> (ghosts, local block, ghost block); a block is
    (indptr, remapped int32 columns, positions of its entries in the full
    value array), entry order kept."""
    lo, hi = int(indptr[r0]), int(indptr[r1])
    cols = np.asarray(indices[lo:hi], dtype=np.int64)
    rowlen = np.diff(np.asarray(indptr[r0:r1 + 1], dtype=np.int64))
    row_of = np.repeat(np.arange(r1 - r0), rowlen)
    owned = (cols >= r0) & (cols < r1)
    pos = np.arange(lo, hi, dtype=np.int64)
    ghosts = np.unique(cols[~owned])

    def block(mask, remap):
        cnt = np.bincount(row_of[mask], minlength=r1 - r0)
        ptr = np.zeros(r1 - r0 + 1, dtype=np.int64)
        np.cumsum(cnt, out=ptr[1:])
        return ptr, remap.astype(np.int32), pos[mask]

    loc = block(owned, cols[owned] - r0)
    gh = block(~owned, (r1 - r0) + np.searchsorted(ghosts, cols[~owned]))
    return ghosts, loc, gh


def exchange_plan(bounds, rank: int, ghosts, exchange_ids) -> ShardPlan:
    """This rank's plan from the row bounds and its ghost ids.
    `exchange_ids(send_lists) -> recv_lists` is an all-to-all of int64 id lists
    (setup only): rank p tells each owner which of its rows it needs."""
    bounds = np.asarray(bounds, dtype=np.int64)
    world = len(bounds) - 1
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    ghosts = np.asarray(ghosts, dtype=np.int64)
    owner = np.searchsorted(bounds, ghosts, side="right") - 1
    requests = [ghosts[owner == q] for q in range(world)]
    recv_counts = [len(x) for x in requests]
    asked = exchange_ids(requests)  # asked[q] = my rows rank q needs (global ids)
    send_counts = [len(x) for x in asked]
    send_rows = (np.concatenate(asked) - r0).astype(np.int64) if asked else np.zeros(0, np.int64)
    return ShardPlan(world, rank, bounds, r0, r1, ghosts, recv_counts, send_counts, send_rows)


# ------------------------------------------------------------------ exchange


class TorchExchange:
    """Per-hop ghost exchange with torch.distributed all_to_all_single
    (NCCL over NVLink for CUDA tensors; gloo for CPU tensors in tests)."""

    def __init__(self, plan: ShardPlan | None = None, group=None, device="cpu"):
        self.plan = plan
        self.group = group
        self.device = device

    def ids(self, requests):
        import torch
        import torch.distributed as dist

        counts = torch.tensor([len(r) for r in requests], dtype=torch.int64, device=self.device)
        recv = torch.empty_like(counts)
        dist.all_to_all_single(recv, counts, group=self.group)
        flat = np.concatenate(requests).astype(np.int64) if requests else np.zeros(0, np.int64)
        send = torch.from_numpy(flat).to(self.device)
        rc = recv.cpu().numpy()
        out = torch.empty(int(rc.sum()), dtype=torch.int64, device=self.device)
        dist.all_to_all_single(out, send, output_split_sizes=rc.tolist(), input_split_sizes=counts.cpu().tolist(),
                               group=self.group)
        parts = np.split(out.cpu().numpy(), np.cumsum(rc)[:-1])
        return [np.asarray(p, dtype=np.int64) for p in parts]

    def start(self, sendbuf, recvbuf, F: int):
        """Async all-to-all of packed rows (F floats each) into the ghost rows."""
        import torch.distributed as dist

        p = self.plan
        if p.world == 1:
            return None
        return dist.all_to_all_single(recvbuf, sendbuf, output_split_sizes=[c * F for c in p.recv_counts],
                                      input_split_sizes=[c * F for c in p.send_counts], group=self.group,
                                      async_op=True)


class ThreadExchange:
    """In-process stand-in for the collective: P virtual ranks as Python
    threads sharing one device and one stream.  Each hop, every rank deposits
    its packed rows, a host barrier orders them, and receivers copy their
    ghost rows out -- stream-ordered device copies, no kernel ever waits on
    another.  Used to run the exact sharded code path on a single GPU."""

    def __init__(self, world: int):
        import threading

        self.world = world
        self.barrier = threading.Barrier(world)
        self.box: dict = {}
        self.plans: dict = {}

    def for_rank(self, rank: int):
        return _ThreadRankExchange(self, rank)


class _ThreadRankExchange:
    def __init__(self, hub: ThreadExchange, rank: int):
        self.hub, self.rank, self.plan = hub, rank, None

    def ids(self, requests):
        self.hub.box[("ids", self.rank)] = requests
        self.hub.barrier.wait()
        got = [self.hub.box[("ids", q)][self.rank] for q in range(self.hub.world)]
        self.hub.barrier.wait()
        return got

    def start(self, sendbuf, recvbuf, F: int):
        p = self.plan
        offs = np.concatenate([[0], np.cumsum(p.send_counts)]) * F
        self.hub.box[("rows", self.rank)] = [sendbuf[offs[q]:offs[q + 1]] for q in range(p.world)]
        self.hub.barrier.wait()
        roff = np.concatenate([[0], np.cumsum(p.recv_counts)]) * F
        for q in range(p.world):
            src = self.hub.box[("rows", q)][self.rank]
            if src.numel():
                recvbuf[roff[q]:roff[q + 1]].copy_(src)
        self.hub.barrier.wait()
        return None


class _DevArray:
    """A raw device allocation as a __cuda_array_interface__ object (torch
    wraps it without a copy)."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 2, "strides": None}


class _PullWork:
    def __init__(self, be):
        self.be = be

    def wait(self):
        self.be.pull_join()


class PeerExchange:
    """Ghost rows over NVLink peer memory (csrc/peer.cu), one process per GPU.

    Each rank's two signal buffers are plain device allocations published by
    CUDA IPC handle; every rank opens its peers' buffers once.  Per hop:
    `barrier()` (every rank has written the rows others will read, and has
    finished reading what is about to be overwritten), then `pull()` copies
    the ghost rows with peer loads on a forked stream while the local part of
    the hop runs.  The barrier is stream-ordered on NCCL groups (a one-element
    all_reduce: the host never blocks); on a gloo control group (tests: two
    processes sharing one GPU) it is a device synchronise + host barrier.

    Setup traffic (ghost ids, IPC handles) goes through torch.distributed."""

    pull_mode = True

    def __init__(self, group=None, device="cuda:0"):
        import torch.distributed as dist

        self.group = group
        self.device = device
        self.plan = None
        self.nccl = dist.get_backend(group) == "nccl"
        self._ids = TorchExchange(group=group, device=device if self.nccl else "cpu")
        self._flag = None
        self._own: list[int] = []
        self._opened: list[int] = []
        self._keep: list = []
        self.tables: list = []

    def ids(self, requests):
        return self._ids.ids(requests)

    # -- setup: allocate, publish, open, build the pull tables
    def alloc_signal(self, be, rows: int, plan: ShardPlan):
        import torch
        import torch.distributed as dist

        lib, _lib = be.lib, be._lib
        ctx = be.ctx()
        world, rank = plan.world, plan.rank
        nbytes = max(rows, 1) * 4 * 4
        bufs, handles, err = [], [], None
        try:
            for _ in range(2):
                ptr = ctypes.c_void_p()
                h = (ctypes.c_ubyte * 64)()
                _lib.check(lib.gift_peer_alloc(ctx, nbytes, ctypes.byref(ptr), ctypes.cast(h, ctypes.c_void_p)))
                self._own.append(ptr.value)
                handles.append(bytes(h))
                holder = _DevArray(ptr.value, (max(rows, 1), 4))
                self._keep.append(holder)
                bufs.append(torch.as_tensor(holder, device=self.device))
        except Exception as e:  # keep the collective below matched on every rank
            handles, err = None, e
        everyone = [None] * world
        dist.all_gather_object(everyone, handles, group=self.group)
        if any(h is None for h in everyone):
            raise RuntimeError(f"peer memory unavailable on rank(s) "
                               f"{[q for q, h in enumerate(everyone) if h is None]}: {err!r}")
        for which in range(2):
            ptrs = np.zeros(world, dtype=np.int64)
            for q in range(world):
                if q == rank:
                    ptrs[q] = self._own[which]
                elif plan.recv_counts[q] > 0:  # map only the ranks this one reads from
                    p = ctypes.c_void_p()
                    hb = (ctypes.c_ubyte * 64).from_buffer_copy(everyone[q][which])
                    _lib.check(lib.gift_peer_open(ctx, ctypes.cast(hb, ctypes.c_void_p), ctypes.byref(p)))
                    self._opened.append(p.value)
                    ptrs[q] = p.value
            self.tables.append(be.upload(ptrs))
        self._finish_tables(be, plan)
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        return bufs[0], bufs[1]

    def _finish_tables(self, be, plan: ShardPlan):
        owner = np.searchsorted(plan.bounds, plan.ghosts, side="right") - 1
        self.src_rank = be.upload(owner.astype(np.int32))
        self.src_row = be.upload((plan.ghosts - plan.bounds[owner]).astype(np.int64))

    def barrier(self):
        import torch
        import torch.distributed as dist

        if self.plan is not None and self.plan.world == 1:
            return
        if self.nccl:
            dist.all_reduce(self._flag, group=self.group)  # ordered on the current stream
        else:
            torch.cuda.synchronize()
            dist.barrier(group=self.group)

    def pull(self, be, which: int, F: int, dst):
        be.pull(self.plan.n_ghost, F, self.tables[which], self.src_rank, self.src_row, dst)
        return _PullWork(be)

    def close(self, be):
        """Unmap the peers' buffers and free this rank's (collective)."""
        lib, _lib = be.lib, be._lib
        self.barrier()
        if self.nccl:
            be.torch.cuda.synchronize()
        for p in self._opened:
            _lib.check(lib.gift_peer_close(be.ctx(), ctypes.c_void_p(p)))
        self._opened = []
        self.barrier()
        if self.nccl:
            be.torch.cuda.synchronize()
        for p in self._own:
            _lib.check(lib.gift_peer_free(be.ctx(), ctypes.c_void_p(p)))
        self._own = []


class ThreadPeerExchange:
    """PeerExchange for P virtual ranks as threads of one process on one GPU
    (tests): the "peers" are allocations of the same process, shared by
    pointer instead of IPC handle (a process cannot open its own handles),
    and the barrier is a host barrier -- every thread enqueues on the same
    stream, so work enqueued after the barrier runs after what the other
    ranks enqueued before it; no kernel ever waits on another."""

    def __init__(self, world: int):
        import threading

        self.world = world
        self.barrier = threading.Barrier(world)
        self.box: dict = {}

    def for_rank(self, rank: int):
        return _ThreadPeerRank(self, rank)


class _ThreadPeerRank(PeerExchange):
    def __init__(self, hub: ThreadPeerExchange, rank: int):
        self.hub, self.rank, self.plan = hub, rank, None
        self.device = "cuda:0"
        self._own, self._opened, self._keep, self.tables = [], [], [], []

    def ids(self, requests):
        return _ThreadRankExchange.ids(self, requests)

    def alloc_signal(self, be, rows: int, plan: ShardPlan):
        import torch

        lib, _lib = be.lib, be._lib
        bufs = []
        for _ in range(2):
            ptr = ctypes.c_void_p()
            _lib.check(lib.gift_peer_alloc(be.ctx(), max(rows, 1) * 16, ctypes.byref(ptr), None))
            self._own.append(ptr.value)
            holder = _DevArray(ptr.value, (max(rows, 1), 4))
            self._keep.append(holder)
            bufs.append(torch.as_tensor(holder, device=self.device))
        self.hub.box[("ptrs", self.rank)] = list(self._own)
        self.hub.barrier.wait()
        for which in range(2):
            ptrs = np.array([self.hub.box[("ptrs", q)][which] for q in range(plan.world)], dtype=np.int64)
            self.tables.append(be.upload(ptrs))
        self._finish_tables(be, plan)
        return bufs[0], bufs[1]

    def barrier(self):
        self.hub.barrier.wait()

    def close(self, be):
        be.torch.cuda.synchronize()
        self.hub.barrier.wait()
        for p in self._own:
            be._lib.check(be.lib.gift_peer_free(be.ctx(), ctypes.c_void_p(p)))
        self._own = []


# ------------------------------------------------------------------ backends


class CudaBackend:
    """Kernel calls through libgiftb200.so on this rank's GPU."""

    def __init__(self, device: int):
        from . import _lib

        self._lib = _lib
        self.lib = _lib.load_library()
        self.device = device
        self.torch = _lib.torch_cuda()

    def ctx(self):
        return self._lib.context(self.device)

    def empty(self, rows: int, cols: int, dtype="f32"):
        t = self.torch
        return t.zeros((max(rows, 1), cols), dtype=t.float32 if dtype == "f32" else t.float64,
                       device=f"cuda:{self.device}")

    def upload(self, arr):
        return self.torch.from_numpy(np.ascontiguousarray(arr)).to(f"cuda:{self.device}")

    def pack(self, n, wcols, groups_s, g, ld, c0, F, z):
        arr = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(p) for p in groups_s] + [None] * (4 - len(groups_s)))
        in_dtype = self._lib.GIFT_DTYPE_F32 if g.dtype == self.torch.float32 else self._lib.GIFT_DTYPE_F64
        self._lib.check(self.lib.gift_pack_fp32(self.ctx(), n, wcols, len(groups_s),
                                                ctypes.cast(arr, ctypes.c_void_p), in_dtype, self._lib.dptr(g),
                                                ld, c0, F, self._lib.dptr(z)))

    def gather(self, idx, F, src, dst):
        self._lib.check(self.lib.gift_gather_rows_f32(self.ctx(), idx.numel(), F, self._lib.dptr(idx),
                                                      self._lib.dptr(src), self._lib.dptr(dst)))

    def hop(self, block, desc: dict):
        d = _hop_desc(desc)
        self._lib.check(self.lib.gift_hop_fp32(self.ctx(), block.h, ctypes.addressof(d)))

    def pull(self, n_rows, F, peers, src_rank, src_row, dst):
        self._lib.check(self.lib.gift_pull_rows_f32(self.ctx(), n_rows, F, self._lib.dptr(peers),
                                                    self._lib.dptr(src_rank), self._lib.dptr(src_row),
                                                    self._lib.dptr(dst)))

    def pull_join(self):
        self._lib.check(self.lib.gift_pull_join(self.ctx()))


class _Handle:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        if self.h:
            self.lib.gift_csr_destroy(self.h)
            self.h = None


class _Chain(ctypes.Structure):
    _fields_ = [("s", ctypes.c_void_p), ("sigma", ctypes.c_double), ("cont", ctypes.c_int),
                ("has_term", ctypes.c_int), ("alpha", ctypes.c_double)]


class _HopDesc(ctypes.Structure):
    _fields_ = [("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64), ("fin", ctypes.c_int),
                ("fout", ctypes.c_int), ("wcols", ctypes.c_int), ("nch", ctypes.c_int),
                ("zin", ctypes.c_void_p), ("zout", ctypes.c_void_p), ("part_in", ctypes.c_void_p),
                ("part_out", ctypes.c_void_p), ("chain", _Chain * 4), ("acc", ctypes.c_void_p),
                ("acc_read", ctypes.c_int), ("is_final", ctypes.c_int), ("out_dtype", ctypes.c_int),
                ("out", ctypes.c_void_p), ("out_ld", ctypes.c_int64), ("out_c0", ctypes.c_int64),
                ("fixed_mask", ctypes.c_void_p), ("fixed_pos", ctypes.c_void_p),
                ("region", ctypes.c_double * 4)]


def _ptr(t):
    return None if t is None else t.data_ptr()


def _hop_desc(d: dict) -> _HopDesc:
    h = _HopDesc()
    h.row_begin, h.row_end = d["row_begin"], d["row_end"]
    h.fin, h.fout, h.wcols, h.nch = d["fin"], d["fout"], d["wcols"], len(d["chains"])
    h.zin, h.zout = _ptr(d["zin"]), _ptr(d.get("zout"))
    h.part_in, h.part_out = _ptr(d.get("part_in")), _ptr(d.get("part_out"))
    for j, ch in enumerate(d["chains"]):
        h.chain[j] = _Chain(ch["s"], ch["sigma"], ch["cont"], ch["has_term"], ch["alpha"])
    h.acc = _ptr(d["acc"])
    h.acc_read, h.is_final = d["acc_read"], d["is_final"]
    h.out_dtype, h.out = d.get("out_dtype", 1), _ptr(d.get("out"))
    h.out_ld, h.out_c0 = d.get("out_ld", 0), d.get("out_c0", 0)
    h.fixed_mask, h.fixed_pos = _ptr(d.get("fixed_mask")), _ptr(d.get("fixed_pos"))
    reg = d.get("region")
    if reg is not None:
        for i in range(4):
            h.region[i] = float(reg[i])
    return h


# ------------------------------------------------------------------ driver


class ShardedFilter:
    """Runs the bank on this rank's row block with per-hop ghost exchange.

    plan        : ShardPlan
    local, ghost: this rank's two CSR blocks (backend handles: gift_csr for
                  CudaBackend, scipy matrices for the CPU tests)
    s_of        : sigma -> this block's s32 (backend handle)
    """

    def __init__(self, plan: ShardPlan, local, ghost, backend, exchange, s_of):
        self.plan = plan
        self.be = backend
        self.ex = exchange
        self.ex.plan = plan
        self.s_of = s_of
        self.local = local
        self.ghost = ghost
        n, ng = plan.n_local, plan.n_ghost
        self.pull_mode = bool(getattr(exchange, "pull_mode", False))
        if self.pull_mode:  # signal buffers the other ranks read through peer mappings
            self.zA, self.zB = exchange.alloc_signal(backend, n + ng, plan)
        else:
            self.zA = backend.empty(n + ng, 4)
            self.zB = backend.empty(n + ng, 4)
        self.acc = backend.empty(n, 4)
        self.part = backend.empty(n, 4)
        self.sendbuf = backend.empty(len(plan.send_rows), 4)
        self.send_idx = backend.upload(plan.send_rows)

    def block_nnz(self) -> int:
        """Stored entries of this rank's row block (local + ghost parts)."""
        from . import _lib

        tot = 0
        for blk in (self.local, self.ghost):
            n, nnz = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(_lib.load_library().gift_csr_shape(blk.h, ctypes.byref(n), ctypes.byref(nnz)))
            tot += nnz.value
        return tot

    def _exchange(self, z, F):
        p = self.plan
        n, ng = p.n_local, p.n_ghost
        flat = z.view(-1)
        if self.pull_mode:
            # every rank's rows of z are complete (and nobody still reads the
            # buffer this hop will overwrite): pull the ghosts from the owners
            self.ex.barrier()
            if ng == 0:
                return None
            return self.ex.pull(self.be, 0 if z is self.zA else 1, F, flat[n * F: (n + ng) * F])
        send = self.sendbuf.view(-1)[: len(p.send_rows) * F]
        if len(p.send_rows):
            self.be.gather(self.send_idx, F, flat, send)
        recv = flat[n * F: (n + ng) * F]
        if p.world == 1:
            return None
        return self.ex.start(send, recv, F)

    def run(self, g, terms, out, fixed_mask=None, fixed_pos=None, region=None):
        """g: [n_local, ncols] (f32/f64) on the backend; out: [n_local, ncols] f64."""
        p = self.plan
        n = p.n_local
        ncols = g.shape[1]
        bank = plan_bank(terms, ncols)
        zin, zout = self.zA, self.zB
        for st in bank.steps:
            if isinstance(st, PackStep):
                F = st.F
                if self.pull_mode:  # a slow peer may still pull its last ghosts of the previous bank from zA
                    self.ex.barrier()
                self.be.pack(n, st.wcols, [self.s_of(bank.sigmas[j]) for j in st.groups], g, ncols, st.c0, F,
                             self.zA.view(-1))
                zin, zout = self.zA, self.zB
                continue
            F = st.fin
            zin_f = zin.view(-1)
            zout_f = zout.view(-1)
            work = self._exchange(zin, F)
            chains = [dict(s=self.s_of(bank.sigmas[c.group]), sigma=bank.sigmas[c.group], cont=c.cont,
                           has_term=c.has_term, alpha=c.alpha) for c in st.chains]
            common = dict(row_begin=0, row_end=n, fin=F, fout=st.fout, wcols=st.wcols, chains=chains,
                          zin=zin_f, acc=self.acc, acc_read=st.acc_read, is_final=st.is_final)
            # local columns overlap the exchange
            self.be.hop(self.local, dict(common, part_out=self.part.view(-1), zout=None))
            if work is not None:
                work.wait()
            self.be.hop(self.ghost, dict(common, part_in=self.part.view(-1), zout=zout_f if st.fout else None,
                                         out=out, out_ld=ncols, out_c0=st.c0, out_dtype=1,
                                         fixed_mask=fixed_mask, fixed_pos=fixed_pos, region=region))
            zin, zout = zout, zin
        return out


# ------------------------------------------------------------------ CUDA entry


def cuda_sharded_filter(adj, world: int, rank: int, device: int, exchange=None, group=None) -> ShardedFilter:
    """Set up this rank's share of `adj` (a full SparseSymMatrix resident on
    `device`, built on every rank) without a host copy of the graph: row
    bounds and the local / ghost split run on the device
    (gift_csr_row_bounds / gift_csr_split_rows); only the ghost id list
    (halo + fixed objects, ~1e5 ids at c4) comes to the host for the exchange
    plan.  s_sigma comes from the full graph's degrees, sliced to the block,
    so it is the single-GPU vector."""
    from . import _lib

    if getattr(adj, "implicit_nets", 0):
        raise ValueError("row sharding does not support the implicit high-fanout term")
    be = CudaBackend(device)
    ex = exchange or TorchExchange(group=group, device=f"cuda:{device}")
    lib = _lib.load_library()
    ctx = _lib.context(device)
    bounds = np.zeros(world + 1, dtype=np.int64)
    _lib.check(lib.gift_csr_row_bounds(ctx, adj.handle, world, bounds.ctypes.data_as(_lib.c_i64p)))
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    hl, hg = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(lib.gift_csr_split_rows(ctx, adj.handle, r0, r1, ctypes.byref(hl), ctypes.byref(hg)))
    local, ghost = _Handle(lib, hl.value), _Handle(lib, hg.value)
    ids_p, n_ids = ctypes.c_void_p(), ctypes.c_int64()
    _lib.check(lib.gift_csr_ext_ids(ghost.h, ctypes.byref(ids_p), ctypes.byref(n_ids)))
    ghosts = np.empty(n_ids.value, dtype=np.int64)
    if n_ids.value:
        from .graph import _memcpy_d2h

        _memcpy_d2h(ghosts, ids_p.value)
    plan = exchange_plan(bounds, rank, ghosts, ex.ids)
    cache: dict = {}

    def s_of(sigma):
        if sigma not in cache:
            s64 = ctypes.c_void_p()
            s32 = ctypes.c_void_p()
            _lib.check(lib.gift_csr_scale(_lib.context(device), adj.handle, float(sigma), ctypes.byref(s64),
                                          ctypes.byref(s32)))
            cache[sigma] = (s32.value or 0) + 4 * plan.r0
        return cache[sigma]

    for sigma in {t.sigma for t in _default_terms()}:  # the usual bank's vectors, before any rank thread runs
        s_of(sigma)
    sf = ShardedFilter(plan, local, ghost, be, ex, s_of)
    sf._adj = adj  # s_sigma slices point into the full graph's arrays
    return sf


def _default_terms():
    from .gift import DEFAULT_TERMS

    return DEFAULT_TERMS
