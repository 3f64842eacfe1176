"""Pins the oracle's restatement of the paper's data-parallel engine
(oracle/sssp_oracle.c: o_dijkstra_dataparallel, dataparallel.hpp:302-327) to
the reference before the GPU engine is checked against it:

* the known answers of test_dataparallel.cpp:60-80 and :144-154,
* the reference's own compiled dijkstra_dataparallel (oracle/_ref) under all
  three lane schedules (threaded / sequential / shuffled, :22-27) on random
  graphs with zero weights, ties, directed edges and unreachable vertices,
* golden vectors produced by the reference (tests/golden/golden.json).
"""
import hashlib
import json
import os

import numpy as np
import pytest

INF = 0xFFFFFFFFFFFFFFFF
FOUR = [(0, 1, 2), (0, 2, 4), (1, 2, 1), (1, 3, 3), (2, 3, 5)]
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.uint64).tobytes()).hexdigest()


def unit_path(k):
    n = k + 1
    adj = np.full(n * n, INF, np.uint64)
    adj[:: n + 1] = 0
    for u in range(k):
        adj[u * n + u + 1] = 1
    return adj, n


def rand_adj(rng, n, wmax, density, directed):
    adj = np.full((n, n), INF, dtype=np.uint64)
    m = rng.random((n, n)) < density
    adj[m] = rng.integers(0, wmax + 1, size=int(m.sum()), dtype=np.uint64)
    if not directed:
        iu = np.triu_indices(n, 1)
        adj[(iu[1], iu[0])] = adj[iu]
    np.fill_diagonal(adj, 0)
    return adj.ravel()


def test_known_answers(oracle_c):
    adj = oracle_c.from_edges(4, FOUR, False)
    d, p, r = oracle_c.dataparallel(adj, 4, 0)  # test_dataparallel.cpp:60-66
    assert d.tolist() == [0, 2, 3, 5] and r <= 4
    assert oracle_c.validate(adj, 4, 0, d, p) == 0
    d, p, r = oracle_c.dataparallel(np.zeros(1, np.uint64), 1, 0)  # :68-73
    assert r == 1 and d.tolist() == [0] and p.tolist() == [INF]
    for k in range(1, 10):  # :75-82
        adj, n = unit_path(k)
        d, p, r = oracle_c.dataparallel(adj, n, 0)
        assert r == k + 1 and d.tolist() == list(range(n))
    with pytest.raises(ValueError):  # :181-184
        oracle_c.dataparallel(np.zeros(9, np.uint64), 3, 3)


def test_zero_weight_tie_fixture(oracle_c):
    # test_dataparallel.cpp:144-154: dist pinned by the test; pred by the
    # reference's reconstruct_predecessors (0 attaches to 2; 1 to 0 through the
    # zero-weight edge in the first pass, unlike serial's pred[1] = 2)
    adj = oracle_c.from_edges(4, [(2, 0, 5), (2, 1, 5), (0, 1, 0), (1, 3, 2)], False)
    d, p, r = oracle_c.dataparallel(adj, 4, 2)
    assert d.tolist() == [5, 5, 0, 7]
    assert p.tolist() == [2, 0, INF, 1]
    assert oracle_c.validate(adj, 4, 2, d, p) == 0


def test_golden(oracle_c):
    for case in GOLDEN["dataparallel"]:
        adj = np.array(case["adj"], np.uint64) if "adj" in case else oracle_c.dense(
            case["n"], case["seed"])
        d, p, r = oracle_c.dataparallel(adj, case["n"], case["source"])
        assert r == case["rounds"], case["name"]
        if "dist" in case:
            assert d.tolist() == case["dist"] and p.tolist() == case["pred"], case["name"]
        else:
            assert h(d) == case["dist_sha"] and h(p) == case["pred_sha"], case["name"]


@pytest.mark.parametrize("seed", range(6))
def test_live_vs_reference(oracle_c, ref, seed):
    rng = np.random.default_rng(4100 + seed)
    for _ in range(25):
        n = int(rng.integers(1, 48))
        adj = rand_adj(rng, n, int(rng.choice([0, 1, 2, 3, 100])), float(rng.uniform(0.02, 0.9)),
                       bool(rng.integers(0, 2)))
        s = int(rng.integers(0, n))
        d, p, r = oracle_c.dataparallel(adj, n, s)
        for sched in (0, 1, 2):
            rd, rp, rr = ref.dataparallel(adj, n, s, sched)
            assert np.array_equal(d, rd) and np.array_equal(p, rp) and r == rr, (n, s, sched)
        sd, _ = oracle_c.serial(adj, n, s)
        assert np.array_equal(d, sd)  # same dist as serial (the fixpoint)
