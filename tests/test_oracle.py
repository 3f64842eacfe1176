"""Pins the CPU oracle (oracle/sssp_oracle.c) to the reference before it is
trusted as the GPU path's checker:

* the known answers of the reference's unit suite (test_serial.cpp:11-75,
  test_partitioned.cpp:194-246, test_dataparallel.cpp:144-154),
* golden vectors produced by the reference's own compiled code
  (tests/golden/make_golden.py -> golden.json), and
* live comparison with oracle/_ref (the reference headers, unmodified) on the
  acceptance sweep (acceptance.cpp:42-80) and tie-heavy random graphs.
"""
import hashlib
import json
import os

import numpy as np
import pytest

INF = 0xFFFFFFFFFFFFFFFF
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.uint64).tobytes()).hexdigest()


FOUR = [(0, 1, 2), (0, 2, 4), (1, 2, 1), (1, 3, 3), (2, 3, 5)]


def test_mt19937_64_reference_value(oracle_c):
    # [rand.predef]: the 10000th output of default-seeded mt19937_64
    r = oracle_c.rng(5489)
    for _ in range(9999):
        r()
    assert r() == 9981545732273789042


def test_four_vertex_known_answer(oracle_c):
    adj = oracle_c.from_edges(4, FOUR, False)
    d, p, vo, ct = oracle_c.serial(adj, 4, 0, visit_order=True, counters=True)
    assert d.tolist() == [0, 2, 3, 5]
    assert p.tolist() == [INF, 0, 1, 1]
    assert vo.tolist() == [0, 1, 2, 3]
    assert ct.tolist() == [16, 16]


def test_directed_and_trivial_known_answers(oracle_c):
    adj = oracle_c.from_edges(4, FOUR, True)
    d, p = oracle_c.serial(adj, 4, 3)
    assert d.tolist() == [INF, INF, INF, 0] and p.tolist() == [INF] * 4
    d, p = oracle_c.serial(np.zeros(1, np.uint64), 1, 0)
    assert d.tolist() == [0] and p.tolist() == [INF]
    with pytest.raises(ValueError):
        oracle_c.serial(np.zeros(9, np.uint64), 3, 3)


def test_zero_weight_fixture(oracle_c):
    adj = oracle_c.from_edges(4, [(2, 0, 5), (2, 1, 5), (0, 1, 0), (1, 3, 2)], False)
    d, p = oracle_c.serial(adj, 4, 2)
    assert d.tolist() == [5, 5, 0, 7] and p.tolist() == [2, 2, INF, 1]


@pytest.mark.parametrize("case", GOLDEN["cases"], ids=lambda c: c["name"])
def test_golden_cases(oracle_c, case):
    n = case["n"]
    name = case["name"]
    if name.startswith("config1_dense"):
        adj = oracle_c.dense(n, 42)
    elif name.startswith("config1_sparse"):
        adj = oracle_c.sparse(n, 42)
    elif name == "single_vertex":
        adj = np.zeros(1, np.uint64)
    elif name.startswith("zero_weight"):
        adj = oracle_c.from_edges(4, [(2, 0, 5), (2, 1, 5), (0, 1, 0), (1, 3, 2)], False)
    else:
        adj = oracle_c.from_edges(4, FOUR, case["directed"])
    assert h(adj) == case["adj_sha256"], "oracle graph builder != reference"
    d, p, vo, ct = oracle_c.serial(adj, n, case["source"], visit_order=True, counters=True)
    assert h(d) == case["dist_sha256"] and h(p) == case["pred_sha256"]
    assert h(vo) == case["visit_order_sha256"]
    assert ct.tolist() == case["counters"]
    if "dist" in case:
        assert d.tolist() == case["dist"] and p.tolist() == case["pred"]


def test_golden_acceptance_sweep(oracle_c):
    """acceptance.cpp:42-80 graphs (rng 20240601): oracle graph + result hashes
    equal the reference's."""
    rng = oracle_c.rng(20240601)
    for (n, seed, s, dense, directed, ha, hd, hp) in GOLDEN["acceptance_sweep"]:
        n2 = 7 + rng() % 194
        seed2 = rng()
        adj = oracle_c.dense(n2, seed2, bool(directed)) if dense else oracle_c.sparse(n2, seed2, bool(directed))
        s2 = rng() % n2
        assert (n2, seed2, s2) == (n, seed, s)
        assert h(adj) == ha
        d, p = oracle_c.serial(adj, n2, s2)
        assert h(d) == hd and h(p) == hp


def test_golden_generators(oracle_c):
    for key, hh in GOLDEN["generate_dense_matrix"].items():
        n, s = map(int, key.split(":"))
        assert h(oracle_c.dense(n, s)) == hh
    for key, hh in GOLDEN["generate_sparse_edges"].items():
        n, s = map(int, key.split(":"))
        assert h(oracle_c.sparse_edges(n, s)) == hh


def test_oracle_distances_match_floyd_warshall(oracle_c):
    # test_serial.cpp:53-67 (rng 17, 40 graphs, n <= 90)
    rng = oracle_c.rng(17)
    for i in range(40):
        dense, directed = i % 2 == 0, i % 4 < 2
        n = 7 + rng() % (90 - 7 + 1)
        seed = rng()
        adj = oracle_c.dense(n, seed, directed) if dense else oracle_c.sparse(n, seed, directed)
        s = rng() % n
        d, p = oracle_c.serial(adj, n, s)
        fw = oracle_c.all_pairs(adj, n)
        assert np.array_equal(d, fw[s])
        assert oracle_c.validate(adj, n, s, d, p) == 0


def test_partitioned_restatement_matches_serial_and_winner_trace(oracle_c):
    """partitioned.hpp:142-154 sequential rounds == serial (full result), and
    winners follow the serial visit order then (INF, padded_n)
    (test_partitioned.cpp:206-228)."""
    rng = np.random.default_rng(41)
    for i in range(30):
        n = int(rng.integers(1, 60))
        adj = np.full((n, n), INF, np.uint64)
        m = rng.random((n, n)) < 0.2
        adj[m] = rng.integers(0, 3, size=int(m.sum()), dtype=np.uint64)
        np.fill_diagonal(adj, 0)
        s = int(rng.integers(0, n))
        d, p, vo = oracle_c.serial(adj, n, s, visit_order=True)
        finite = int(np.count_nonzero(d != INF))
        for P in (1, 2, 3, 4, 7, 32):
            d2, p2, w = oracle_c.partitioned(adj, n, s, P, winners=True)
            assert np.array_equal(d, d2) and np.array_equal(p, p2)
            pn = oracle_c.pad_vertex_count(n, P)
            assert len(w) == pn
            assert w[:finite, 1].tolist() == vo[:finite].tolist()
            assert all(x == INF for x in w[finite:, 0])
            assert all(x == pn for x in w[finite:, 1])


def test_pad_vertex_count_grid(oracle_c):
    # partition.hpp:25-29 properties (test_partition.cpp)
    import paper_2504_03667_b200 as P
    assert oracle_c.pad_vertex_count(4, 3) == 6 and oracle_c.pad_vertex_count(3, 8) == 8
    for n in range(1, 80):
        for p in range(1, 20):
            pn = oracle_c.pad_vertex_count(n, p)
            assert pn % p == 0 and pn >= max(n, p)
            if p <= n:
                assert pn - n < p
            assert P.pad_vertex_count(n, p) == pn


# ---- live comparison with the reference build (skipped if oracle/_ref is absent)

def test_oracle_equals_reference_acceptance_sweep(oracle_c, ref):
    rng = oracle_c.rng(20240601)
    for dense in (False, True):
        for directed in (False, True):
            for _ in range(100):
                n = 7 + rng() % 194
                seed = rng()
                if dense:
                    a1, a2 = oracle_c.dense(n, seed, directed), ref.dense(n, seed, directed)
                else:
                    a1, a2 = oracle_c.sparse(n, seed, directed), ref.sparse(n, seed, directed)
                assert np.array_equal(a1, a2)
                s = rng() % n
                d1, p1 = oracle_c.serial(a1, n, s)
                d2, p2 = ref.serial(a2, n, s)
                assert np.array_equal(d1, d2) and np.array_equal(p1, p2)


def test_oracle_equals_reference_tie_heavy(oracle_c, ref):
    rng = np.random.default_rng(2504)
    for i in range(150):
        n = int(rng.integers(1, 120))
        adj = np.full((n, n), INF, np.uint64)
        m = rng.random((n, n)) < float(rng.choice([0.05, 0.3, 1.0]))
        adj[m] = rng.integers(0, 3, size=int(m.sum()), dtype=np.uint64)
        if i % 2:
            adj = np.minimum(adj, adj.T)
        np.fill_diagonal(adj, 0)
        s = int(rng.integers(0, n))
        d1, p1, v1 = oracle_c.serial(adj, n, s, visit_order=True)
        d2, p2, v2 = ref.serial(adj, n, s, visit_order=True)
        assert np.array_equal(d1, d2) and np.array_equal(p1, p2) and np.array_equal(v1, v2)
        P = int(rng.integers(1, 9))
        d3, p3, _ = ref.partitioned(adj, n, s, P, threaded=False)
        d4, p4 = oracle_c.partitioned(adj, n, s, P)
        assert np.array_equal(d3, d4) and np.array_equal(p3, p4)
