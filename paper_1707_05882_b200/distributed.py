"""Order-sharded BRDF solves across ranks (one process per GPU), SURVEY.md §8(e).

Independent units are Fourier orders m (and bands).  Rank r solves the orders
m = r, r + W, r + 2W, ... of a solve (cyclic: per-order dense work is
m-independent, only the kernel assembly shrinks with m) through a device plan
with that order shard; the per-order tau = 0 upward stacks -- the only data the
cross-order step needs (reconstruction.cpp:201-227) -- move between GPUs as
device buffers (NCCL point-to-point over NVLink; gloo in the CPU tests), and
the owner of the solve runs the Fourier/Mueller synthesis over m = 0..L-1 in
fixed order on its device.  Every order is computed by the same kernels
regardless of the shard, so the table is bitwise identical for any world size.

Two layouts over W ranks:
  * one solve (`sharded_brdf`, latency): the W order shards of ONE solve,
    gathered to rank 0;
  * W solves in flight (`inflight_brdf`, throughput): every rank holds its
    order shard of each of W solves (W plans on its GPU, run concurrently) and
    an all-to-all hands solve j's shards to rank j, which synthesizes it -- the
    per-GPU work is one solve's worth, split into W order shards.
Both take a process group: on 8 GPUs the throughput layout runs as two groups
of 4 (orders sharded 4 ways inside a group, 4 solves in flight per group):
an order shard of a C3 solve stays large enough to keep its GPU busy.
"""
from __future__ import annotations

import threading

import numpy as np


def order_shard(L: int, world: int, rank: int):
    """(m_begin, m_stride, n_orders) of this rank's cyclic order shard."""
    return rank, world, len(range(rank, L, world))


def shard_orders(L: int, world: int, rank: int):
    return list(range(rank, L, world))


def _dist():
    import torch.distributed as dist
    return dist


def _peer(ranks, j):
    """Global rank of group member j (ranks: the group's global ranks, or None)."""
    return j if ranks is None else ranks[j]


def gather_order_stacks(local, L: int, world: int, rank: int, dst: int = 0, group=None, ranks=None):
    """Point-to-point gather of the order shards to `dst`: `local` is this
    rank's tensor [n_r, ...] of orders m = rank + k world; on dst returns the
    full [L, ...] tensor (order m at index m), None elsewhere.  CUDA tensors go
    over NCCL, CPU tensors over gloo.  world / rank / dst are positions in
    `ranks` (the group's global ranks; None = the default group)."""
    import torch
    dist = _dist()
    shape = tuple(local.shape[1:])
    if rank != dst:
        if local.shape[0] > 0:
            for r in dist.batch_isend_irecv([dist.P2POp(dist.isend, local.contiguous(), _peer(ranks, dst), group)]):
                r.wait()
        return None
    full = torch.empty((L,) + shape, dtype=local.dtype, device=local.device)
    ops, bufs = [], {}
    for src in range(world):
        n = len(range(src, L, world))
        if n == 0:
            continue
        if src == rank:
            full[src::world] = local
            continue
        bufs[src] = torch.empty((n,) + shape, dtype=local.dtype, device=local.device)
        ops.append(dist.P2POp(dist.irecv, bufs[src], _peer(ranks, src), group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for src, buf in bufs.items():
        full[src::world] = buf
    return full


def alltoall_order_stacks(locals_by_owner, L: int, world: int, rank: int, group=None, ranks=None):
    """All-to-all of order shards: locals_by_owner[j] is this rank's shard of
    solve j (orders m = rank + k world, [n_rank, ...]); returns the full
    [L, ...] stacks of solve `rank`, assembled from every rank's shard."""
    import torch
    dist = _dist()
    mine = locals_by_owner[rank]
    shape = tuple(mine.shape[1:])
    full = torch.empty((L,) + shape, dtype=mine.dtype, device=mine.device)
    full[rank::world] = mine
    ops, bufs = [], {}
    for j in range(world):
        if j != rank and locals_by_owner[j].shape[0] > 0:
            ops.append(dist.P2POp(dist.isend, locals_by_owner[j].contiguous(), _peer(ranks, j), group))
    for src in range(world):
        n = len(range(src, L, world))
        if src == rank or n == 0:
            continue
        bufs[src] = torch.empty((n,) + shape, dtype=mine.dtype, device=mine.device)
        ops.append(dist.P2POp(dist.irecv, bufs[src], _peer(ranks, src), group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for src, buf in bufs.items():
        full[src::world] = buf
    return full


def gather_orders(local_up, L: int, world: int, rank: int, device=None):
    """numpy convenience (CPU tests): the full [L, ...] stacks on every rank
    (an all-gather of the shards, gloo or NCCL)."""
    import torch
    dist = _dist()
    per = (L + world - 1) // world
    shape = tuple(local_up.shape[1:])
    buf = np.zeros((per,) + shape, dtype=np.float64)
    buf[: local_up.shape[0]] = local_up
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    out = torch.empty((world * per,) + shape, dtype=torch.float64, device=t.device)
    dist.all_gather_into_tensor(out, t)
    gathered = out.cpu().numpy().reshape((world, per) + shape)
    full = np.zeros((L,) + shape, dtype=np.float64)
    for r in range(world):
        for k, m in enumerate(shard_orders(L, world, r)):
            full[m] = gathered[r, k]
    return full


def _run_threads(fns, concurrency):
    """Run the callables on `concurrency` host threads (the C calls release the
    GIL; each plan has its own CUDA streams); re-raises the first failure."""
    errs = []
    groups = [fns[i::concurrency] for i in range(max(1, min(concurrency, len(fns))))]

    def work(g):
        try:
            for f in g:
                f()
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            errs.append(e)

    ths = [threading.Thread(target=work, args=(g,)) for g in groups[1:]]
    for th in ths:
        th.start()
    work(groups[0])
    for th in ths:
        th.join()
    if errs:
        raise errs[0]


class OrderShards:
    """This rank's order shards of n_solves solves (1: one solve, gathered to
    rank 0; W: W solves in flight, solve j owned by rank j), as device plans on
    `device`.  Creating the object solves the shards once; run() solves them
    again (device-resident inputs), exchange() moves the stacks, synthesize()
    builds the owned table on the device."""

    def __init__(self, materials, opts, mu_in, n_dphi=19, basis=None, world=1, rank=0, device=0,
                 group=None, concurrency=4, pooled=True, ranks=None):
        import paper_1707_05882_b200 as V
        if len(materials) not in (1, world):
            raise ValueError("OrderShards: one solve, or one solve per rank")
        self.world, self.rank, self.group, self.device, self.ranks = world, rank, group, device, ranks
        self.concurrency = max(1, concurrency)
        L = materials[0].info()[0]
        if any(m.info()[0] != L for m in materials):
            raise ValueError("OrderShards: the in-flight solves must share the order count L")
        if opts.order_cap > 0:
            L = min(L, opts.order_cap)
        self.L = L
        m_begin, m_stride, n = order_shard(L, world, rank)
        if n == 0:  # (sharded_brdf returns None on such ranks before getting here)
            raise ValueError("OrderShards: more ranks than Fourier orders")
        self.plans = [None] * len(materials)

        def make(j):
            def f():
                self.plans[j] = V.Plan(materials[j], opts, mu_in, n_dphi, basis, device=device,
                                       m_begin=m_begin, m_stride=m_stride, n_orders=n, pooled=pooled)
            return f

        _run_threads([make(j) for j in range(len(materials))], self.concurrency)
        self.full = None

    def run(self):
        _run_threads([(lambda p=p: p.run(1)) for p in self.plans], self.concurrency)

    def exchange(self):
        """The owned solve's full [L, 4 n_in, 4N] device stacks (None if this
        rank owns no solve).  NCCL moves the device buffers directly; a gloo
        group (tests: several ranks on one GPU) stages them through the host."""
        dist = _dist()
        host = dist.get_backend(self.group) == "gloo"
        ups = [p.up_device() for p in self.plans]
        if host:
            ups = [u.cpu() for u in ups]
        if len(self.plans) == 1:
            full = gather_order_stacks(ups[0], self.L, self.world, self.rank, 0, self.group, self.ranks)
        else:
            full = alltoall_order_stacks(ups, self.L, self.world, self.rank, self.group, self.ranks)
        if host and full is not None:
            import torch
            full = full.to(torch.device("cuda", self.plans[0].device))
        self.full = full
        return full

    def owner_plan(self):
        if len(self.plans) == 1:
            return self.plans[0] if self.rank == 0 else None
        return self.plans[self.rank]

    def synthesize(self, fetch=True):
        p = self.owner_plan()
        if p is None or self.full is None:
            return None
        return p.synthesize_device(self.full, fetch)

    def close(self):
        for p in self.plans:
            if p is not None:
                p.close()
        self.plans = []
        self.full = None


def _world(group):
    dist = _dist()
    return dist.get_world_size(group), dist.get_rank(group)


def _group_ranks(group):
    if group is None:
        return None
    dist = _dist()
    return dist.get_process_group_ranks(group)


def sharded_brdf(material, opts, mu_in, n_dphi=19, basis=None, group=None, device=None):
    """ONE BRDF table with its orders sharded across the ranks of the process
    group: host table [n_in, N, n_dphi, 4, 4] on rank 0, None elsewhere."""
    import torch
    world, rank = _world(group)
    L = material.info()[0] if opts.order_cap <= 0 else min(material.info()[0], opts.order_cap)
    if order_shard(L, world, rank)[2] == 0:
        return None  # more ranks than orders: nothing to solve or send here (rank 0 always has m = 0)
    dev = torch.cuda.current_device() if device is None else device
    sh = OrderShards([material], opts, mu_in, n_dphi, basis, world, rank, dev, group, ranks=_group_ranks(group))
    try:
        sh.exchange()
        return sh.synthesize(True)
    finally:
        sh.close()


def inflight_brdf(materials, opts, mu_in, n_dphi=19, basis=None, group=None, device=None, concurrency=4):
    """W BRDF tables at once over W ranks (materials[j] is solve j): every rank
    solves its order shard of all W, the shards are exchanged all-to-all, and
    rank j returns table j (host [n_in, N, n_dphi, 4, 4])."""
    import torch
    world, rank = _world(group)
    dev = torch.cuda.current_device() if device is None else device
    sh = OrderShards(materials, opts, mu_in, n_dphi, basis, world, rank, dev, group, concurrency,
                     ranks=_group_ranks(group))
    try:
        sh.exchange()
        return sh.synthesize(True)
    finally:
        sh.close()
