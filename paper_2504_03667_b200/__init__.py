"""B200-native matrix-scan Dijkstra (arXiv 2504.03667) -- Python host API.

The product is ``libsssp_cuda.so`` (CUDA sm_100a + C ABI, ``include/sssp_cuda.h``);
the C++ drop-in for the reference is ``include/sssp/cuda.hpp``.  This module is
the thin Python mirror of the same reference interface, used by ``bench.py``
and the tests:

===============================  =============================================
reference (proj/include/sssp)    here
===============================  =============================================
``Graph`` (graph.hpp:33-58)      :class:`Graph` (numpy uint64 ``adj``, n*n)
``graph_from_edges`` (:73-88)    :func:`graph_from_edges`
``parse_edge_list`` (:172-174)   :func:`parse_edge_list` (``-w`` = directed)
``generate_dense/sparse``        :func:`generate_dense`, :func:`generate_sparse`
``ShortestPathResult``           :class:`ShortestPathResult` (``==`` compares
(result.hpp:13-19)               source, dist and pred, like the C++ default)
``dijkstra_serial(g, s)``        :func:`dijkstra` (runs on the GPU)
(serial.hpp:65-68)
``dijkstra_partitioned(g,s,p)``  :func:`dijkstra_partitioned` (P shards)
===============================  =============================================

Errors follow the reference: a source outside ``[0, n)`` raises ``ValueError``
(``std::invalid_argument``, serial.hpp:30), malformed edge lists raise
:class:`ParseError` with the offending line (graph.hpp:60-69).  Every other
failure raises :class:`SsspError`; nothing falls back to the CPU.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _native
from ._native import Options, SsspError, Stats, check, lib

INF = np.uint64(0xFFFFFFFFFFFFFFFF)       # kInfinity (weight.hpp:13)
NO_VERTEX = np.uint64(0xFFFFFFFFFFFFFFFF)  # kNoVertex (weight.hpp:21)
MAX_WEIGHT = 0xFFFFFFFF                    # kMaxWeight (weight.hpp:18)

__all__ = [
    "INF", "NO_VERTEX", "MAX_WEIGHT", "Graph", "ShortestPathResult", "ParseError", "SsspError",
    "graph_from_edges", "parse_edge_list", "generate_dense", "generate_sparse",
    "generate_bernoulli", "DeviceGraph", "ShardGraph", "dijkstra", "dijkstra_partitioned",
    "dijkstra_dataparallel",
    "pad_vertex_count", "Options", "Stats",
]


def _p64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


@dataclass
class Graph:
    """Dense adjacency matrix, row-major, ``adj[u*n+v]`` (graph.hpp:30-45)."""

    n: int
    directed: bool
    adj: np.ndarray  # uint64, shape (n*n,) or (n, n)

    def __post_init__(self):
        self.adj = np.ascontiguousarray(self.adj, dtype=np.uint64).reshape(self.n * self.n)

    @staticmethod
    def no_edges(n: int, directed: bool = False) -> "Graph":
        adj = np.full(n * n, INF, dtype=np.uint64)
        adj[:: n + 1] = 0
        return Graph(n, directed, adj)

    def at(self, u: int, v: int) -> int:
        return int(self.adj[u * self.n + v])

    def matrix(self) -> np.ndarray:
        return self.adj.reshape(self.n, self.n)


@dataclass
class ShortestPathResult:
    """``{source, dist[], pred[]}`` with value equality (result.hpp:13-19)."""

    source: int
    dist: np.ndarray
    pred: np.ndarray
    stats: dict = field(default_factory=dict, compare=False, repr=False)

    def __eq__(self, other) -> bool:
        if not isinstance(other, ShortestPathResult):
            return NotImplemented
        return (self.source == other.source and np.array_equal(self.dist, other.dist)
                and np.array_equal(self.pred, other.pred))


class ParseError(ValueError):
    """Edge-list format error carrying the 1-based line number (graph.hpp:60-69)."""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


def pad_vertex_count(n: int, p: int) -> int:
    """partition.hpp:25-29."""
    if n < 1 or p < 1:
        raise ValueError("pad_vertex_count: n, p >= 1")
    return p if p > n else n + (p - n % p) % p


def graph_from_edges(n: int, edges: Iterable[Sequence[int]], directed: bool) -> Graph:
    """graph.hpp:73-88: minimum over duplicates, mirrored when undirected."""
    e = np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges,
                   dtype=np.uint64).reshape(-1, 3)
    out = np.empty(n * n, dtype=np.uint64)
    rc = lib.sssp_graph_from_edges(n, _p64(np.ascontiguousarray(e)), len(e), int(directed), 0,
                                   n, n, _p64(out))
    if rc != 0:
        raise ValueError("graph_from_edges: endpoint out of range, self-loop or weight > 2^32-1")
    return Graph(n, directed, out)


def parse_edge_list(text: str, directed: bool) -> Graph:
    """graph.hpp:126-174: ``n m`` header then m ``u v w`` lines; '#' and blank
    lines skipped; CRLF tolerated.  ``directed`` is the CLI's ``-w`` switch.
    Parsed by the library on all host threads (sssp_parse_edge_list), with the
    reference's first error (ParseError line and message)."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    n = ctypes.c_uint64()
    m = ctypes.c_uint64()
    line = ctypes.c_uint64()
    err = ctypes.create_string_buffer(512)
    rc = lib.sssp_parse_edge_list(data, len(data), ctypes.byref(n), ctypes.byref(m), None, 0,
                                  ctypes.byref(line), err, len(err))
    if rc == 0:
        edges = np.empty(3 * m.value, dtype=np.uint64)
        rc = lib.sssp_parse_edge_list(data, len(data), ctypes.byref(n), ctypes.byref(m),
                                      _p64(edges), m.value, ctypes.byref(line), err, len(err))
    if rc != 0:
        if line.value:
            msg = err.value.decode()
            pe = ParseError(line.value, msg.split(": ", 1)[1] if ": " in msg else msg)
            raise pe
        check(rc, "sssp_parse_edge_list")
    return graph_from_edges(n.value, edges.reshape(-1, 3), directed)


def _gen(fn, n: int, *args, directed: bool, cols: Optional[tuple] = None) -> np.ndarray:
    cb, cc = (0, n) if cols is None else cols
    out = np.empty(n * cc, dtype=np.uint64)
    rc = fn(n, *args, int(directed), cb, cc, cc, _p64(out))
    if rc != 0:
        raise ValueError(f"generator rejected n={n}")
    return out


def generate_dense(n: int, seed: int, directed: bool = False, cols: Optional[tuple] = None):
    """graph_from_edges(generate_dense(n, seed), directed) (generate.hpp:38-48).
    With ``cols=(begin, count)`` only that column block is returned (n x count)."""
    out = _gen(lib.sssp_gen_dense, n, seed, directed=directed, cols=cols)
    return Graph(n, directed, out) if cols is None else out.reshape(n, cols[1])


def generate_sparse(n: int, seed: int, directed: bool = False, cols: Optional[tuple] = None):
    """graph_from_edges(generate_sparse(n, seed), directed) (generate.hpp:53-83)."""
    out = _gen(lib.sssp_gen_sparse, n, seed, directed=directed, cols=cols)
    return Graph(n, directed, out) if cols is None else out.reshape(n, cols[1])


def generate_bernoulli(n: int, p: float, seed: int, directed: bool = False,
                       cols: Optional[tuple] = None):
    """Bernoulli(p) graph of BASELINE configs 2/4."""
    q = int(round(p * (1 << 53)))
    out = _gen(lib.sssp_gen_bernoulli, n, q, seed, directed=directed, cols=cols)
    return Graph(n, directed, out) if cols is None else out.reshape(n, cols[1])


ENGINES = {"auto": 0, "grid": 1, "cluster": 2, "bucket": 3}
ENGINE_NAMES = {1: "grid", 2: "cluster", 3: "bucket", 4: "dataparallel", 5: "wide"}


def _options(flags: Optional[int], ctas: int, max_batch: int, timeout_ms: int,
             visit_order: bool, replicas: int = 0, engine: str = "auto",
             warps: int = 0, global_min_weight: int = -1, round_times: bool = False) -> Options:
    o = Options()
    o.record_round_times = int(round_times)
    o.global_min_weight = global_min_weight
    o.engine = ENGINES[engine]
    o.warps_per_cta = warps
    o.ctas_per_shard = ctas
    o.flags = _native.SSSP_FLAGS_DEFAULT if flags is None else flags
    o.max_batch = max_batch
    o.timeout_ms = timeout_ms
    o.record_visit_order = int(visit_order)
    o.replicas = replicas
    return o


class DeviceGraph:
    """A graph resident in HBM (one GPU, or P column shards in one process).

    ``devices`` lists the GPU of every shard (partition.hpp:31-41); repeating a
    device runs several shards on one GPU."""

    def __init__(self, g: Graph, devices: Sequence[int] = (0,), *, flags: Optional[int] = None,
                 ctas: int = 0, max_batch: int = 0, timeout_ms: int = 0,
                 visit_order: bool = False, replicas: int = 0, engine: str = "auto",
                 warps: int = 0, round_times: bool = False):
        self.n = g.n
        self._opt = _options(flags, ctas, max_batch, timeout_ms, visit_order, replicas, engine,
                             warps, round_times=round_times)
        devs = (ctypes.c_int * len(devices))(*devices)
        h = ctypes.c_void_p()
        check(lib.sssp_graph_create(_p64(g.adj), g.n, int(g.directed), devs, len(devices),
                                    ctypes.byref(self._opt), ctypes.byref(h)), "sssp_graph_create")
        self._h = h
        self.row_len = g.n

    @classmethod
    def from_edges(cls, n: int, edges, directed: bool, devices: Sequence[int] = (0,), **kw):
        """Builds the matrix ON THE DEVICE from (u, v, w) triples: the
        reference's graph_from_edges (graph.hpp:73-88) without the n*n host
        matrix.  Same keywords as the constructor."""
        self = cls.__new__(cls)
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint64).reshape(-1, 3))
        self.n = n
        self._opt = _options(kw.get("flags"), kw.get("ctas", 0), kw.get("max_batch", 0),
                             kw.get("timeout_ms", 0), kw.get("visit_order", False),
                             kw.get("replicas", 0), kw.get("engine", "auto"), kw.get("warps", 0))
        devs = (ctypes.c_int * len(devices))(*devices)
        h = ctypes.c_void_p()
        st = lib.sssp_graph_create_from_edges(n, _p64(e), len(e), int(directed), devs, len(devices),
                                              ctypes.byref(self._opt), ctypes.byref(h))
        if st == _native.SSSP_ERR_BAD_ARG:
            raise ValueError("graph_from_edges: endpoint out of range, self-loop or weight > 2^32-1")
        check(st, "sssp_graph_create_from_edges")
        self._h = h
        self.row_len = n
        return self

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib.sssp_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def info(self) -> dict:
        st = Stats()
        check(lib.sssp_graph_info(self._h, ctypes.byref(st)), "sssp_graph_info")
        d = st.as_dict()
        d["max_batch"] = d.pop("iterations")
        d["min_weight"] = d.pop("relax_checks")
        d["max_weight"] = d.pop("mispredicts")
        return d

    # -- solves
    def solve(self, source: int, visit_order: bool = False) -> ShortestPathResult:
        dist = np.empty(self.row_len, dtype=np.uint64)
        pred = np.empty(self.row_len, dtype=np.uint64)
        order = np.empty(self.n, dtype=np.uint64) if visit_order else None
        st = Stats()
        if source < 0:
            raise ValueError("dijkstra: source out of range")
        check(lib.sssp_solve(self._h, source, _p64(dist), _p64(pred),
                             _p64(order) if order is not None else None, ctypes.byref(st)),
              "sssp_solve")
        r = ShortestPathResult(source, dist, pred, st.as_dict())
        if order is not None:
            # all n rounds of dijkstra_serial: the reachable vertices in election
            # order, then the unreachable ones in ascending id (serial.hpp:41-48)
            r.stats["visit_order"] = order
        return r

    def solve_batch(self, sources: Sequence[int]) -> list:
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.uint64))
        k = len(src)
        dist = np.empty((k, self.row_len), dtype=np.uint64)
        pred = np.empty((k, self.row_len), dtype=np.uint64)
        st = Stats()
        check(lib.sssp_solve_batch(self._h, _p64(src), k, _p64(dist), _p64(pred),
                                   ctypes.byref(st)), "sssp_solve_batch")
        stats = st.as_dict()
        return [ShortestPathResult(int(s), dist[i], pred[i], stats) for i, s in enumerate(src)]

    # -- asynchronous form used for device-side timing
    def enqueue(self, sources: Sequence[int]) -> None:
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.uint64))
        check(lib.sssp_enqueue(self._h, _p64(src), len(src)), "sssp_enqueue")

    def finish(self) -> dict:
        st = Stats()
        check(lib.sssp_finish(self._h, ctypes.byref(st)), "sssp_finish")
        return st.as_dict()

    def solve_dataparallel(self, source: int) -> "ShortestPathResult":
        """The paper's data-parallel engine, dijkstra_dataparallel(g, s)
        (dataparallel.hpp:302-327): stats["rounds"] = DataParallelRun::rounds."""
        if source < 0:
            raise ValueError("dijkstra_dataparallel: source out of range")
        dist = np.empty(self.n, dtype=np.uint64)
        pred = np.empty(self.n, dtype=np.uint64)
        rounds = ctypes.c_uint64()
        st = Stats()
        check(lib.sssp_solve_dataparallel(self._h, source, _p64(dist), _p64(pred),
                                          ctypes.byref(rounds), ctypes.byref(st)),
              "sssp_solve_dataparallel")
        r = ShortestPathResult(source, dist, pred, st.as_dict())
        r.stats["rounds"] = rounds.value
        return r

    def validate(self, r: "ShortestPathResult") -> int:
        """validate_result (oracle.hpp:51-120) on the device; 0 = valid."""
        out = ctypes.c_uint64()
        d = np.ascontiguousarray(r.dist, np.uint64)
        p = np.ascontiguousarray(r.pred, np.uint64)
        check(lib.sssp_validate(self._h, r.source, _p64(d), _p64(p), ctypes.byref(out)),
              "sssp_validate")
        return out.value

    def round_times(self) -> np.ndarray:
        """Per-round %globaltimer stamps (ns) of the last scan-engine solve
        (needs ``round_times=True``); np.diff gives the per-round latency."""
        out = np.empty(self.n, dtype=np.uint64)
        cnt = ctypes.c_uint64()
        check(lib.sssp_round_times(self._h, _p64(out), self.n, ctypes.byref(cnt)), "sssp_round_times")
        return out[: cnt.value].copy()

    def probe_sync(self, rounds: int = 20000) -> float:
        """Seconds per exchange round of the solve's own launch shape (t_sync_min)."""
        out = ctypes.c_double()
        check(lib.sssp_probe_sync(self._h, rounds, ctypes.byref(out)), "sssp_probe_sync")
        return out.value

    def probe_skeleton(self, barriers: int, launches: int = 50) -> float:
        """Seconds per launch of the bucket engine's synchronisation skeleton:
        the solve's cooperative launch shape doing `barriers` grid barriers and
        nothing else (the floor under a solve with that many barriers)."""
        out = ctypes.c_double()
        check(lib.sssp_probe_skeleton(self._h, barriers, launches, ctypes.byref(out)),
              "sssp_probe_skeleton")
        return out.value

    def stream_ptr(self, local: int = 0) -> int:
        return lib.sssp_stream(self._h, local) or 0


class ShardGraph(DeviceGraph):
    """This process's shard of a column-partitioned graph (one process per GPU).

    ``block`` is the n x col_count uint64 column block of the shard (columns
    [rank*loc_n, ...)), ``max_weight`` the largest finite weight of the whole
    graph.  Call :meth:`export` on every rank, all-gather the handles in rank
    order, then :meth:`connect`."""

    def __init__(self, block: np.ndarray, n: int, world: int, rank: int, max_weight: int,
                 device: int = 0, *, flags: Optional[int] = None, ctas: int = 0,
                 timeout_ms: int = 0, replicas: int = 0, engine: str = "auto", warps: int = 0,
                 max_batch: int = 1, global_min_weight: int = -1):
        self.n = n
        self._opt = _options(flags, ctas, max_batch, timeout_ms, False, replicas, engine, warps,
                             global_min_weight)
        blk = np.ascontiguousarray(block, dtype=np.uint64)
        ld = blk.shape[1] if blk.ndim == 2 else max(1, blk.size // max(1, n))
        h = ctypes.c_void_p()
        check(lib.sssp_shard_create(_p64(blk), ld, n, world, rank, max_weight, device,
                                    ctypes.byref(self._opt), ctypes.byref(h)), "sssp_shard_create")
        self._h = h
        b = ctypes.c_uint64()
        c = ctypes.c_uint64()
        check(lib.sssp_shard_range(self._h, ctypes.byref(b), ctypes.byref(c)), "sssp_shard_range")
        self.col_begin, self.col_count = b.value, c.value
        self.row_len = self.col_count

    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(_native.SSSP_IPC_HANDLE_BYTES)
        check(lib.sssp_shard_export(self._h, buf), "sssp_shard_export")
        return buf.raw

    def connect(self, handles: Sequence[bytes]) -> None:
        blob = b"".join(handles)
        check(lib.sssp_shard_connect(self._h, ctypes.c_char_p(blob)), "sssp_shard_connect")


def block_weight_range(block: np.ndarray, n: int, col_begin: int) -> tuple:
    """(min finite off-diagonal weight or None, max finite weight) of an n x c column block."""
    blk = np.ascontiguousarray(block, dtype=np.uint64)
    c = blk.shape[1] if blk.ndim == 2 else 0
    mn, mx = ctypes.c_uint64(), ctypes.c_uint64()
    check(lib.sssp_block_weight_range(_p64(blk), max(c, 1), n, col_begin, c, ctypes.byref(mn),
                                      ctypes.byref(mx)), "sssp_block_weight_range")
    return (None if mn.value == 0xFFFFFFFFFFFFFFFF else mn.value), mx.value


def dijkstra(g: Graph, source: int, device: int = 0) -> ShortestPathResult:
    """Drop-in for ``dijkstra_serial(g, source)`` (serial.hpp:65-68), on a B200."""
    if not 0 <= source < g.n:
        raise ValueError("dijkstra: source out of range")
    with DeviceGraph(g, (device,)) as dg:
        return dg.solve(source)


def dijkstra_dataparallel(g: Graph, source: int, device: int = 0) -> ShortestPathResult:
    """Drop-in for ``dijkstra_dataparallel(g, source)`` (dataparallel.hpp:302-327):
    same dist, the reference's reconstructed pred, stats["rounds"] = run.rounds."""
    if not 0 <= source < g.n:
        raise ValueError("dijkstra_dataparallel: source out of range")
    with DeviceGraph(g, (device,)) as dg:
        return dg.solve_dataparallel(source)


def collective_stats(n: int, p: int) -> dict:
    """CollectiveStats of dijkstra_partitioned(g, s, p) as the reference defines
    them (partitioned.hpp:196-221): allreduce_count = padded_n, scatter_bytes =
    uint64 column blocks of workers 1..p-1, gather_bytes = their dist + pred."""
    padded = pad_vertex_count(n, p)
    loc = padded // p
    return {"allreduce_count": padded, "scatter_bytes": (p - 1) * padded * loc * 8,
            "gather_bytes": (p - 1) * loc * 16}


def dijkstra_partitioned(g: Graph, source: int, p: int,
                         devices: Optional[Sequence[int]] = None) -> ShortestPathResult:
    """Column-partitioned solve over p shards (partitioned.hpp:184-225), the
    PartitionedRun mirror: ``result.stats`` carries the reference's
    CollectiveStats for this p and ``phases`` = {scatter_s, rounds_s, gather_s}
    (upload, kernel, download).  The shards go to ``devices`` (default: all on
    GPU 0); at most SSSP_MAX_SHARDS = 8 shards are used for any p -- dist and
    pred do not depend on p (test_partitioned.cpp:135-165) -- and a graph that
    needs 64-bit distances runs on one shard."""
    if p < 1:
        raise ValueError("dijkstra_partitioned: p >= 1")
    if not 0 <= source < g.n:
        raise ValueError("dijkstra_partitioned: source out of range")
    devs = list(devices) if devices is not None else [0] * min(p, 8)
    try:
        dg = DeviceGraph(g, devs)
    except SsspError as e:
        if len(devs) == 1 or "64-bit" not in str(e):
            raise
        dg = DeviceGraph(g, devs[:1])
    with dg:
        r = dg.solve(source)
    r.stats.update(collective_stats(g.n, p))
    r.stats["phases"] = {"scatter_s": r.stats["transfer_in_s"], "rounds_s": r.stats["rounds_s"],
                         "gather_s": r.stats["transfer_out_s"]}
    return r
