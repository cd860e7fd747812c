"""Order sharding + gather + fixed-order synthesis across ranks, on CPU with
gloo (world sizes 2 and 3).  The per-order tau=0 stacks come from the oracle
(identity basis); the test checks that the sharded/gathered stack equals the
unsharded one bitwise and that a fixed-order synthesis of it reproduces the
oracle's own table."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import pyoracle as O
from paper_1707_05882_b200 import distributed as D
from paper_1707_05882_b200 import materials as M

from helpers import oracle_material


def oracle_stacks(desc, N, mu, nd):
    """up[m, ii, c, io, r] from the oracle components with the identity basis."""
    r, _, comps = O.brdf(oracle_material(desc), N, mu, nd, basis=np.eye(4).ravel(), components=True)
    L = comps.shape[2]
    up = np.zeros((L, len(mu), 4, N, 4))
    for c in range(4):
        k = 0 if c < 2 else 1
        up[:, :, c] = comps[:, c, :, k, :].real.transpose(1, 0, 2).reshape(L, len(mu), N, 4)
    return up, r


def synthesize(up, mu, nd, basis=None):
    """Test-side restatement of reconstruction.cpp:201-227 + brdf.cpp:100-117."""
    L, n_in, _, N, _ = up.shape
    B = np.array([[1, 0, 0, 0], [1, 1, 0, 0], [1, 0, 1, 0], [1, 0, 0, 1.0]]) if basis is None else basis
    out = np.zeros((n_in, N, nd, 4, 4))
    for ii, mu0 in enumerate(mu):
        I = mu0 * B.T
        post = B.T @ (I.T @ np.linalg.inv(I @ I.T))
        for ip in range(nd):
            x = -2 * np.pi * ip / nd
            E = np.zeros((N, 4, 4))
            for m in range(L):
                sc = 1.0 if m == 0 else 2.0
                c, s = np.cos(m * x), np.sin(m * x)
                p1 = sc * np.array([c, c, s, s])
                p2 = sc * np.array([-s, -s, c, c])
                for ch in range(4):
                    E[:, :, ch] += 0.5 * (p1 if ch < 2 else p2) * up[m, ii, ch]
            out[ii, :, ip] = E @ post
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = M.config("C1")
    nodes, _ = O.quadrature(w.N)
    up, ref = oracle_stacks(w.material, w.N, nodes[:3], 7)
    L = up.shape[0]
    m_begin, m_stride, n = D.order_shard(L, world, rank)
    local = up[m_begin::m_stride]
    assert local.shape[0] == n
    full = D.gather_orders(local.reshape(n, -1), L, world, rank).reshape(up.shape)
    # the product's point-to-point gather (to rank 0) and all-to-all (solve j to rank j)
    import torch
    g = D.gather_order_stacks(torch.from_numpy(np.ascontiguousarray(local)), L, world, rank)
    # W in-flight solves: solve j = the stacks scaled by (j + 1) (distinct data per solve)
    a2a = D.alltoall_order_stacks([torch.from_numpy(np.ascontiguousarray(local * (j + 1))) for j in range(world)],
                                  L, world, rank)
    ok_a2a = bool(np.array_equal(a2a.numpy(), up * (rank + 1)))
    oks = [None] * world
    dist.all_gather_object(oks, ok_a2a)
    if rank == 0:
        q.put((np.array_equal(full, up) and np.array_equal(g.numpy(), up) and all(oks),
               float(np.abs(synthesize(full, nodes[:3], 7) - ref).max()), float(np.abs(ref).max())))
    else:
        assert g is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_order_sharded_gather_is_bitwise_and_synthesizes_the_table(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    same, err, scale = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert same
    assert err < 1e-12 * scale


def test_shard_partition_covers_every_order_once():
    for L in (1, 5, 12, 64, 256):
        for world in (1, 2, 3, 4, 8):
            seen = sorted(m for r in range(world) for m in D.shard_orders(L, world, r))
            assert seen == list(range(L))
            sizes = [D.order_shard(L, world, r)[2] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _group_worker(rank, world, port, q):
    """Two groups of 2 ranks: the all-to-all inside each group (global ranks
    mapped through the group's rank list)."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    groups = [[0, 1], [2, 3]]
    handles = [dist.new_group(ranks=g) for g in groups]
    mine = rank // 2
    L, g = 7, 2
    pos = rank % 2
    full = {j: np.arange(L * 3, dtype=np.float64).reshape(L, 3) * (10 * mine + j + 1) for j in range(g)}
    local = [torch.from_numpy(np.ascontiguousarray(full[j][pos::g])) for j in range(g)]
    got = D.alltoall_order_stacks(local, L, g, pos, handles[mine], groups[mine])
    ok = bool(np.array_equal(got.numpy(), full[pos]))
    oks = [None] * world
    dist.all_gather_object(oks, ok)
    if rank == 0:
        q.put(all(oks))
    dist.barrier()
    dist.destroy_process_group()


def test_alltoall_inside_process_subgroups():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_group_worker, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
