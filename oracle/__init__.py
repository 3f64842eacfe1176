"""Parity checkers -- TEST INFRASTRUCTURE ONLY.

``C`` wraps ``oracle/build/liboracle_sssp.so`` (the C restatement in
``sssp_oracle.c``); ``REF`` wraps ``oracle/_ref/libref_sssp.so`` (the
reference's own headers compiled unmodified behind ``ref_shim.cpp``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline and
``--impl reference`` legs may import this package; the product never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle_sssp.so")
REF_SO = os.path.join(HERE, "_ref", "libref_sssp.so")
INF = 0xFFFFFFFFFFFFFFFF

_u64p = ctypes.POINTER(ctypes.c_uint64)


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a):
    return None if a is None else a.ctypes.data_as(_u64p)


def _load(path, sigs):
    if not os.path.exists(path):
        build()
    lib = ctypes.CDLL(path)
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


U64 = ctypes.c_uint64


class _Oracle:
    def __init__(self):
        self.lib = _load(ORACLE_SO, {
            "o_mt64_seed": (None, [ctypes.c_void_p, U64]),
            "o_mt64_next": (U64, [ctypes.c_void_p]),
            "o_generate_dense": (ctypes.c_int, [U64, U64, ctypes.c_int, _u64p]),
            "o_generate_sparse_edges": (ctypes.c_int, [U64, U64, _u64p]),
            "o_generate_bernoulli": (ctypes.c_int, [U64, U64, U64, ctypes.c_int, _u64p]),
            "o_graph_from_edges": (ctypes.c_int, [U64, _u64p, U64, ctypes.c_int, _u64p]),
            "o_dijkstra_serial": (ctypes.c_int, [_u64p, U64, U64, _u64p, _u64p, _u64p, _u64p]),
            "o_dijkstra_partitioned": (ctypes.c_int, [_u64p, U64, U64, U64, _u64p, _u64p, _u64p]),
            "o_pad_vertex_count": (U64, [U64, U64]),
            "o_all_pairs": (ctypes.c_int, [_u64p, U64, _u64p]),
            "o_validate": (U64, [_u64p, U64, U64, _u64p, _u64p]),
            "o_dijkstra_dataparallel": (ctypes.c_int, [_u64p, U64, U64, _u64p, _u64p, _u64p]),
        })

    # --- rng (for reproducing the reference tests' graph sweeps)
    def rng(self, seed):
        st = ctypes.create_string_buffer(312 * 8 + 16)
        self.lib.o_mt64_seed(st, seed)
        return lambda: self.lib.o_mt64_next(st)

    def dense(self, n, seed, directed=False):
        out = np.empty(n * n, np.uint64)
        assert self.lib.o_generate_dense(n, seed, int(directed), _p(out)) == 0
        return out

    def sparse_edges(self, n, seed):
        e = np.empty(9 * n, np.uint64)
        assert self.lib.o_generate_sparse_edges(n, seed, _p(e)) == 0
        return e.reshape(-1, 3)

    def from_edges(self, n, edges, directed):
        e = np.ascontiguousarray(np.asarray(edges, np.uint64).reshape(-1, 3))
        out = np.empty(n * n, np.uint64)
        rc = self.lib.o_graph_from_edges(n, _p(e), len(e), int(directed), _p(out))
        if rc:
            raise ValueError("graph_from_edges rejected input")
        return out

    def sparse(self, n, seed, directed=False):
        return self.from_edges(n, self.sparse_edges(n, seed), directed)

    def bernoulli(self, n, p, seed, directed=False):
        out = np.empty(n * n, np.uint64)
        q = int(round(p * (1 << 53)))
        assert self.lib.o_generate_bernoulli(n, q, seed, int(directed), _p(out)) == 0
        return out

    def serial(self, adj, n, source, visit_order=False, counters=False):
        adj = np.ascontiguousarray(adj, np.uint64)
        dist = np.empty(n, np.uint64)
        pred = np.empty(n, np.uint64)
        vo = np.empty(n, np.uint64) if visit_order else None
        ct = np.empty(2, np.uint64) if counters else None
        rc = self.lib.o_dijkstra_serial(_p(adj), n, source, _p(dist), _p(pred), _p(vo), _p(ct))
        if rc == 1:
            raise ValueError("dijkstra_serial: source out of range")
        out = [dist, pred]
        if visit_order:
            out.append(vo)
        if counters:
            out.append(ct)
        return tuple(out)

    def partitioned(self, adj, n, source, p, winners=False):
        adj = np.ascontiguousarray(adj, np.uint64)
        dist = np.empty(n, np.uint64)
        pred = np.empty(n, np.uint64)
        pn = self.lib.o_pad_vertex_count(n, p)
        w = np.empty(2 * pn, np.uint64) if winners else None
        rc = self.lib.o_dijkstra_partitioned(_p(adj), n, source, p, _p(dist), _p(pred), _p(w))
        if rc:
            raise ValueError("dijkstra_partitioned: bad argument")
        return (dist, pred, w.reshape(-1, 2)) if winners else (dist, pred)

    def pad_vertex_count(self, n, p):
        return int(self.lib.o_pad_vertex_count(n, p))

    def dataparallel(self, adj, n, source):
        """dijkstra_dataparallel (dataparallel.hpp:302-327) -> (dist, pred, rounds)."""
        adj = np.ascontiguousarray(adj, np.uint64)
        dist = np.empty(n, np.uint64)
        pred = np.empty(n, np.uint64)
        r = np.zeros(1, np.uint64)
        rc = self.lib.o_dijkstra_dataparallel(_p(adj), n, source, _p(dist), _p(pred), _p(r))
        if rc == 1:
            raise ValueError("dijkstra_dataparallel: source out of range")
        return dist, pred, int(r[0])

    def all_pairs(self, adj, n):
        d = np.empty(n * n, np.uint64)
        self.lib.o_all_pairs(_p(np.ascontiguousarray(adj, np.uint64)), n, _p(d))
        return d.reshape(n, n)

    def validate(self, adj, n, source, dist, pred):
        return int(self.lib.o_validate(_p(np.ascontiguousarray(adj, np.uint64)), n, source,
                                       _p(dist), _p(pred)))


class _Ref:
    """The reference's own code (oracle/_ref/libref_sssp.so)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.lib = _load(REF_SO, {
            "ref_last_error": (ctypes.c_char_p, []),
            "ref_generate_dense": (ctypes.c_int, [U64, U64, ctypes.c_int, _u64p]),
            "ref_generate_sparse_edges": (ctypes.c_int, [U64, U64, _u64p]),
            "ref_graph_from_edges": (ctypes.c_int, [U64, _u64p, U64, ctypes.c_int, _u64p]),
            "ref_parse_edge_list": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _u64p, _u64p,
                                                   U64, _u64p]),
            "ref_dijkstra_serial": (ctypes.c_int, [_u64p, U64, U64, _u64p, _u64p, _u64p, _u64p]),
            "ref_dijkstra_partitioned": (ctypes.c_int, [_u64p, U64, U64, U64, ctypes.c_int, _u64p,
                                                        _u64p, ctypes.POINTER(ctypes.c_double)]),
            "ref_timed_run": (ctypes.c_int, [ctypes.c_int, _u64p, U64, ctypes.c_int, U64, U64, U64,
                                             _u64p, _u64p, ctypes.POINTER(ctypes.c_double)]),
            "ref_graph_new": (ctypes.c_void_p, [_u64p, U64, ctypes.c_int]),
            "ref_graph_free": (None, [ctypes.c_void_p]),
            "ref_graph_serial": (ctypes.c_int, [ctypes.c_void_p, U64, _u64p, _u64p]),
            "ref_graph_partitioned": (ctypes.c_int, [ctypes.c_void_p, U64, U64, _u64p, _u64p,
                                                     ctypes.POINTER(ctypes.c_double)]),
            "ref_dijkstra_dataparallel": (ctypes.c_int, [_u64p, U64, U64, ctypes.c_int, _u64p,
                                                         _u64p, _u64p]),
        })

    def dense(self, n, seed, directed=False):
        out = np.empty(n * n, np.uint64)
        if self.lib.ref_generate_dense(n, seed, int(directed), _p(out)):
            raise ValueError(self.lib.ref_last_error().decode())
        return out

    def sparse_edges(self, n, seed):
        e = np.empty(9 * n, np.uint64)
        if self.lib.ref_generate_sparse_edges(n, seed, _p(e)):
            raise ValueError(self.lib.ref_last_error().decode())
        return e.reshape(-1, 3)

    def from_edges(self, n, edges, directed):
        e = np.ascontiguousarray(np.asarray(edges, np.uint64).reshape(-1, 3))
        out = np.empty(n * n, np.uint64)
        if self.lib.ref_graph_from_edges(n, _p(e), len(e), int(directed), _p(out)):
            raise ValueError(self.lib.ref_last_error().decode())
        return out

    def sparse(self, n, seed, directed=False):
        return self.from_edges(n, self.sparse_edges(n, seed), directed)

    def parse(self, text, directed, cap=1 << 20):
        n = ctypes.c_uint64()
        line = ctypes.c_uint64()
        adj = np.empty(cap, np.uint64)
        rc = self.lib.ref_parse_edge_list(text.encode(), int(directed), ctypes.byref(n), _p(adj),
                                          cap, ctypes.byref(line))
        if rc == 3:
            return ("parse_error", int(line.value), self.lib.ref_last_error().decode())
        if rc:
            return ("error", 0, self.lib.ref_last_error().decode())
        nn = int(n.value)
        return ("ok", nn, adj[: nn * nn].copy())

    def serial(self, adj, n, source, visit_order=False, counters=False):
        adj = np.ascontiguousarray(adj, np.uint64)
        dist = np.empty(n, np.uint64)
        pred = np.empty(n, np.uint64)
        vo = np.empty(n, np.uint64) if visit_order else None
        ct = np.empty(2, np.uint64) if counters else None
        rc = self.lib.ref_dijkstra_serial(_p(adj), n, source, _p(dist), _p(pred), _p(vo), _p(ct))
        if rc == 1:
            raise ValueError(self.lib.ref_last_error().decode())
        out = [dist, pred]
        if visit_order:
            out.append(vo)
        if counters:
            out.append(ct)
        return tuple(out)

    def graph(self, adj, n, directed=False):
        """Builds the reference Graph once (untimed); returns an opaque handle."""
        h = self.lib.ref_graph_new(_p(np.ascontiguousarray(adj, np.uint64)), n, int(directed))
        if not h:
            raise MemoryError("ref_graph_new failed")
        return h

    def graph_free(self, h):
        self.lib.ref_graph_free(h)

    def graph_serial(self, h, n, source):
        """dijkstra_serial on a prebuilt Graph; returns (dist, pred, seconds)."""
        import time
        dist = np.empty(n, np.uint64)
        pred = np.empty(n, np.uint64)
        t = time.perf_counter()
        rc = self.lib.ref_graph_serial(h, source, _p(dist), _p(pred))
        dt = time.perf_counter() - t
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())
        return dist, pred, dt

    def dataparallel(self, adj, n, source, schedule=0):
        """The reference's dijkstra_dataparallel -> (dist, pred, rounds);
        schedule 0 threaded, 1 sequential, 2 shuffled."""
        adj = np.ascontiguousarray(adj, np.uint64)
        dist = np.empty(n, np.uint64)
        pred = np.empty(n, np.uint64)
        r = np.zeros(1, np.uint64)
        rc = self.lib.ref_dijkstra_dataparallel(_p(adj), n, source, schedule, _p(dist), _p(pred),
                                                _p(r))
        if rc == 1:
            raise ValueError("dijkstra_dataparallel: source out of range")
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return dist, pred, int(r[0])

    def partitioned(self, adj, n, source, p, threaded=True):
        adj = np.ascontiguousarray(adj, np.uint64)
        dist = np.empty(n, np.uint64)
        pred = np.empty(n, np.uint64)
        ph = (ctypes.c_double * 3)()
        rc = self.lib.ref_dijkstra_partitioned(_p(adj), n, source, p, int(threaded), _p(dist),
                                               _p(pred), ph)
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())
        return dist, pred, tuple(ph)


_oracle = None
_ref = None


def C() -> _Oracle:
    global _oracle
    if _oracle is None:
        _oracle = _Oracle()
    return _oracle


def REF() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir("/root/reference/proj/include")
