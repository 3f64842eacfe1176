"""One process per GPU: the host side of the column-partitioned solve.

The reference's dijkstra_partitioned (partitioned.hpp:184-225) scatters column
blocks to p workers, runs padded_n rounds of local_min -> allreduce_minloc ->
relax_owned, then gathers.  Here each torchrun rank owns one shard on its own
GPU; the per-round allreduce_minloc runs INSIDE the persistent kernels as P2P
stores into every rank's mailbox (CUDA IPC handles exchanged once through
torch.distributed), so the only host collectives are the one-time handle
exchange and the final gather of owned dist/pred slices.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from . import ShardGraph, ShortestPathResult, _p64, pad_vertex_count


def shard_range(n: int, world: int, rank: int) -> tuple:
    """Real columns [begin, begin+count) of shard `rank` (partition.hpp:31-41;
    padding columns beyond n are owned but never materialised)."""
    loc_n = pad_vertex_count(n, world) // world
    begin = rank * loc_n
    return begin, max(0, min(loc_n, n - begin))


def exchange_handles(handle: bytes, group=None) -> list:
    """All-gathers every rank's exchange-buffer IPC handle, in rank order."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    return out


def gather_result(source: int, n: int, local_dist: np.ndarray, local_pred: np.ndarray,
                  group=None) -> ShortestPathResult:
    """Reassembles the owned slices of every rank (partitioned.hpp:208-223)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, (dist.get_rank(group), local_dist.tobytes(), local_pred.tobytes()),
                           group=group)
    dist_out = np.empty(n, np.uint64)
    pred_out = np.empty(n, np.uint64)
    for r, db, pb in parts:
        b, c = shard_range(n, world, r)
        dist_out[b:b + c] = np.frombuffer(db, np.uint64)
        pred_out[b:b + c] = np.frombuffer(pb, np.uint64)
    return ShortestPathResult(source, dist_out, pred_out)


def open_shard(block: np.ndarray, n: int, max_weight: int, device: int, group=None,
               **kw) -> ShardGraph:
    """Creates this rank's shard from its column block and connects it to the
    other ranks' shards."""
    import torch
    import torch.distributed as dist
    from . import block_weight_range
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    # every rank must pick the same engine: agree on the graph's weight range
    b, c = shard_range(n, world, rank)
    mn, mx = block_weight_range(block, n, b) if c else (None, 0)
    t = torch.tensor([-(2**62) if mn is None else -int(mn), int(mx)], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    gmin = int(-t[0])
    gmin = -1 if gmin >= 2**62 else gmin
    kw.setdefault("global_min_weight", gmin if gmin >= 0 else -1)
    sg = ShardGraph(block, n, world, rank, max(max_weight, int(t[1])), device, **kw)
    sg.connect(exchange_handles(sg.export(), group))
    return sg


def dijkstra_distributed(block: np.ndarray, n: int, source: int, max_weight: int, device: int,
                         group=None, **kw) -> ShortestPathResult:
    """Collective: every rank passes its n x count column block (shard_range)
    and receives the full ShortestPathResult."""
    sg = open_shard(block, n, max_weight, device, group, **kw)
    try:
        r = sg.solve(source)
    finally:
        # no rank may unmap its mailbox while a peer's kernel could still store
        # into it: close collectively
        import torch.distributed as dist
        dist.barrier(group)
        sg.close()
    return gather_result(source, n, r.dist, r.pred, group)


def solve_host_driven(dg, n: int, source: int, group=None) -> tuple:
    """The comparison path of SURVEY.md §8e: the reference's partitioned round
    (partitioned.hpp:142-154) with the per-round allreduce_minloc (:94-101)
    issued by the HOST -- local_min kernel, ``all_reduce(key, MIN)`` (NCCL on a
    GPU group; through a host copy on gloo), relax kernel -- for all padded_n
    rounds, as the reference runs them (:205).  ``dg`` is this rank's
    ShardGraph (or a one-shard DeviceGraph without a process group).  Returns
    (dist, pred of the owned columns, device seconds of the rounds).  Same
    results as the device P2P exchange; it exists to time that choice."""
    import ctypes

    import torch

    from . import _native
    lib = _native.lib
    world = 1
    dist = None
    if group is not None or _dist_ready():
        import torch.distributed as dist
        world = dist.get_world_size(group)
    rounds = pad_vertex_count(n, world)
    _native.check(lib.sssp_nccl_begin(dg._h, source), "sssp_nccl_begin")
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.ExternalStream(dg.stream_ptr(), device=dev)
    key = torch.empty(1, dtype=torch.int64, device=dev)
    host = dist is not None and world > 1 and dist.get_backend(group) != "nccl"
    keyh = torch.empty(1, dtype=torch.int64, pin_memory=True) if host else None
    kp = ctypes.c_void_p(key.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(rounds):
            _native.check(lib.sssp_nccl_local_min(dg._h, kp), "sssp_nccl_local_min")
            if dist is not None and world > 1:
                if host:
                    keyh.copy_(key)
                    stream.synchronize()
                    dist.all_reduce(keyh, op=dist.ReduceOp.MIN, group=group)
                    key.copy_(keyh, non_blocking=True)
                else:
                    dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
            _native.check(lib.sssp_nccl_relax(dg._h, kp), "sssp_nccl_relax")
        e1.record(stream)
    cols = dg.row_len
    d = np.empty(cols, np.uint64)
    p = np.empty(cols, np.uint64)
    _native.check(lib.sssp_nccl_end(dg._h, _p64(d), _p64(p)), "sssp_nccl_end")
    return d, p, e0.elapsed_time(e1) * 1e-3


def _dist_ready() -> bool:
    try:
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized()
    except Exception:
        return False
