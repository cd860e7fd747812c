"""Order-sharded single solve across 2 ranks on the GPU (both ranks share
cuda:0 here; the gather runs on gloo/CPU tensors): the gathered table must be
bitwise identical to the single-plan table (SURVEY §8(e) determinism)."""
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
    w = M.config("C2")
    nodes, _ = O.quadrature(w.N)
    mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
    b = D.sharded_brdf(mat, V.options(w.N), nodes, 19, local_device=0)
    if rank == 0:
        single = V.compute_brdf(mat, V.options(w.N), nodes, 19).table()
        q.put(bool(np.array_equal(b.table(), single)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_order_sharded_table_is_bitwise_identical():
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
