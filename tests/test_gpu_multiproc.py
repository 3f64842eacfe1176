"""The real one-process-per-GPU path (torchrun-style ranks, CUDA IPC mailboxes,
device P2P stores, owned-slice gather) with world_size 2 -- both ranks on the
one available GPU.  Without MPS the two persistent kernels are time-sliced, so
every round waits for a context switch: only small graphs, generous watchdog."""
import os
import socket

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


def _rank(rank, world, port, n, seed, directed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2504_03667_b200 as P
        from paper_2504_03667_b200 import distributed as D
        b, c = D.shard_range(n, world, rank)
        block = P.generate_sparse(n, seed, directed, cols=(b, c))
        out = []
        for src in (0, n // 2):
            res = D.dijkstra_distributed(block, n, src, max_weight=100, device=0, timeout_ms=120000)
            adj = oracle.C().sparse(n, seed, directed)
            d, p = oracle.C().serial(adj, n, src)
            out.append(bool(np.array_equal(res.dist, d) and np.array_equal(res.pred, p)))
        q.put((rank, out))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,directed", [(40, False), (97, True)])
def test_two_ranks_one_gpu(gpu, n, directed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, n, 11, directed, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for pr in procs:
        pr.join(60)
    for rank, out in res:
        assert out == [True, True], (rank, out)
