"""Multi-process (world_size 2 and 3, gloo) coverage of the N>1 host logic:
shard column ranges follow make_partition_plan (partition.hpp:31-41), IPC
handles are exchanged in rank order, and owned dist/pred slices gathered from
every rank reassemble the reference result (partitioned.hpp:208-223)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2504_03667_b200 import distributed as D
        C = oracle.C()
        adj = C.sparse(n, 7, True)
        d, p = C.serial(adj, n, 3)
        b, c = D.shard_range(n, world, rank)
        # the rank's column block is exactly what it would upload
        blk = adj.reshape(n, n)[:, b:b + c]
        assert blk.shape == (n, c)
        handles = D.exchange_handles(bytes([rank]) * 64)
        assert [h[0] for h in handles] == list(range(world))
        res = D.gather_result(3, n, d[b:b + c].copy(), p[b:b + c].copy())
        ok = np.array_equal(res.dist, d) and np.array_equal(res.pred, p)
        q.put((rank, ok, b, c))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 100), (3, 100), (2, 7), (3, 8)])
def test_gloo_shard_gather(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    out = sorted(q.get() for _ in range(world))
    assert all(ok for _, ok, _, _ in out)
    import oracle
    pn = oracle.C().pad_vertex_count(n, world)
    loc = pn // world
    assert [(b, c) for _, _, b, c in out] == [(r * loc, max(0, min(loc, n - r * loc))) for r in range(world)]
