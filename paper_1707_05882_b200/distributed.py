"""Order-sharded BRDF solves across ranks (one process per GPU), SURVEY.md §8(e).

Independent units are Fourier orders m (and bands).  Rank r solves the orders
m = r, r + W, r + 2W, ... (cyclic: per-order dense work is m-independent, only
the kernel assembly shrinks with m) through a device-resident plan with an
order shard, then the per-order tau = 0 upward stacks are all-gathered
(NCCL over NVLink on GPUs, gloo in the CPU tests) and rank 0 re-assembles
them in order 0..L-1 and runs the Fourier/Mueller synthesis.  Because every
order is computed by the same kernels regardless of the shard and the
synthesis sums orders in fixed order, the table is bitwise identical for
any world size (asserted by the GPU tests).
"""
from __future__ import annotations

import numpy as np


def order_shard(L: int, world: int, rank: int):
    """(m_begin, m_stride, n_orders) of this rank's cyclic order shard."""
    return rank, world, len(range(rank, L, world))


def shard_orders(L: int, world: int, rank: int):
    return list(range(rank, L, world))


def gather_orders(local_up, L: int, world: int, rank: int, device=None):
    """All-gather per-rank order shards [n_r, ...] into the full [L, ...] stack
    (returned on every rank).  `local_up` is a numpy array; the exchange runs
    on torch.distributed (NCCL when `device` is a CUDA device, else gloo)."""
    import torch
    import torch.distributed as dist

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


def sharded_brdf(material, opts, mu_in, n_dphi=19, basis=None, world=None, rank=None, device=None,
                 local_device=-1):
    """One BRDF table computed with its orders sharded across the ranks of the
    default process group.  Returns a Brdf handle on rank 0, None elsewhere."""
    import torch.distributed as dist

    import paper_1707_05882_b200 as V

    world = dist.get_world_size() if world is None else world
    rank = dist.get_rank() if rank is None else rank
    L = material.info()[0] if opts.order_cap <= 0 else min(material.info()[0], opts.order_cap)
    m_begin, m_stride, n_orders = order_shard(L, world, rank)
    if n_orders == 0:
        # more ranks than orders: this rank holds no order but still joins the
        # collective (a plan with n_orders = 0 would mean "all orders")
        N = opts.quadrature_n
        local = np.zeros((0, len(mu_in) * 4 * 4 * N))
    else:
        plan = V.Plan(material, opts, mu_in, n_dphi, basis, device=local_device, m_begin=m_begin,
                      m_stride=m_stride, n_orders=n_orders)
        local = plan.up().reshape(n_orders, -1)
        plan.close()
    full = gather_orders(local, L, world, rank, device=device)
    if rank != 0:
        return None
    return V.brdf_from_stacks(material, opts, mu_in, n_dphi, basis, full)
