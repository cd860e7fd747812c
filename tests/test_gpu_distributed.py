"""Order-sharded solves across 2 ranks on the GPU (both ranks share cuda:0
here, so the exchange runs on gloo with host staging; on separate GPUs it is
NCCL on the device buffers): the one-solve gather and the two-solves-in-flight
all-to-all must give tables bitwise identical to single-plan solves (SURVEY
§8(e) determinism), synthesized on the device from the exchanged stacks."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import paper_1707_05882_b200 as V
    import pyoracle as O
    from paper_1707_05882_b200 import distributed as D
    from paper_1707_05882_b200 import materials as M
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    torch.cuda.set_device(0)
    w = M.config("C2")
    nodes, _ = O.quadrature(w.N)
    mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
    t = D.sharded_brdf(mat, V.options(w.N), nodes, 19, device=0)
    ok = True
    if rank == 0:
        single = V.compute_brdf(mat, V.options(w.N), nodes, 19).table()
        ok = bool(np.array_equal(t, single))
    else:
        ok = t is None
    # two C5 bands in flight: rank j gets band j
    N = 16
    nq, _ = O.quadrature(N)
    mats = [V.Material.load(M.config("C5", band=b).material.write(tempfile.mkdtemp(), "m")) for b in (0, 30)]
    tj = D.inflight_brdf(mats, V.options(N), nq, 7, device=0)
    single_j = V.compute_brdf(mats[rank], V.options(N), nq, 7).table()
    ok = ok and bool(np.array_equal(tj, single_j))
    oks = [None, None]
    dist.all_gather_object(oks, ok)
    if rank == 0:
        q.put(all(oks))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_order_sharded_tables_are_bitwise_identical():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
