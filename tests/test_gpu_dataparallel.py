"""The paper's data-parallel engine on the B200 (sssp_solve_dataparallel,
dataparallel_kernel.cuh) against the oracle's restatement of the reference's
dijkstra_dataparallel (dataparallel.hpp:302-327), which
tests/test_oracle_dataparallel.py pins to the reference's compiled code:
bit-exact dist, the reference's reconstructed pred, and the same round count
(DataParallelRun::rounds).  Cases mirror test_dataparallel.cpp:60-184 plus
zero-weight multi-pass reconstructions, every weight encoding and BASELINE
sizes."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
INF = 0xFFFFFFFFFFFFFFFF
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def rand_graph(gpu, rng, n, wlo, whi, density, directed):
    adj = np.full((n, n), INF, dtype=np.uint64)
    m = rng.random((n, n)) < density
    adj[m] = rng.integers(wlo, whi + 1, size=int(m.sum()), dtype=np.uint64)
    if not directed:
        iu = np.triu_indices(n, 1)
        adj[(iu[1], iu[0])] = adj[iu]
    np.fill_diagonal(adj, 0)
    return gpu.Graph(n, directed, adj.ravel())


def check(gpu, oracle_c, g, s):
    d, p, r = oracle_c.dataparallel(g.adj, g.n, s)
    res = gpu.dijkstra_dataparallel(g, s)
    ok = np.array_equal(res.dist, d) and np.array_equal(res.pred, p)
    if not ok:
        bad = np.nonzero((res.dist != d) | (res.pred != p))[0]
        i = int(bad[0])
        raise AssertionError(f"n={g.n} s={s}: {len(bad)} mismatches, v={i} gpu=({res.dist[i]},"
                             f"{res.pred[i]}) want=({d[i]},{p[i]})")
    assert res.stats["rounds"] == r, (res.stats["rounds"], r)
    return res


def test_known_answers(gpu, oracle_c):
    g = gpu.graph_from_edges(4, [(0, 1, 2), (0, 2, 4), (1, 2, 1), (1, 3, 3), (2, 3, 5)], False)
    r = check(gpu, oracle_c, g, 0)  # test_dataparallel.cpp:60-66
    assert r.dist.tolist() == [0, 2, 3, 5] and r.stats["rounds"] <= 4
    r = check(gpu, oracle_c, gpu.Graph.no_edges(1), 0)  # :68-73
    assert r.stats["rounds"] == 1 and r.dist.tolist() == [0]
    for k in range(1, 10):  # :75-82 unit paths settle in k + 1 rounds
        g = gpu.graph_from_edges(k + 1, [(u, u + 1, 1) for u in range(k)], True)
        r = check(gpu, oracle_c, g, 0)
        assert r.stats["rounds"] == k + 1 and r.dist.tolist() == list(range(k + 1))
    with pytest.raises(ValueError):  # :181-184
        gpu.dijkstra_dataparallel(gpu.Graph.no_edges(3), 3)


def test_zero_weight_fixture_and_golden(gpu, oracle_c):
    g = gpu.graph_from_edges(4, [(2, 0, 5), (2, 1, 5), (0, 1, 0), (1, 3, 2)], False)
    r = check(gpu, oracle_c, g, 2)  # :144-154
    assert r.dist.tolist() == [5, 5, 0, 7] and r.pred.tolist() == [2, 0, INF, 1]
    for case in GOLDEN["dataparallel"]:
        if "adj" not in case:
            continue
        g = gpu.Graph(case["n"], True, np.array(case["adj"], np.uint64))
        r = gpu.dijkstra_dataparallel(g, case["source"])
        assert r.dist.tolist() == case["dist"] and r.pred.tolist() == case["pred"], case["name"]
        assert r.stats["rounds"] == case["rounds"], case["name"]


@pytest.mark.parametrize("seed", range(6))
def test_tie_heavy_zero_weights(gpu, oracle_c, seed):
    # weights {0,1,2}: zero-weight tight edges force the multi-pass rebuild
    rng = np.random.default_rng(5100 + seed)
    for _ in range(12):
        n = int(rng.integers(2, 160))
        g = rand_graph(gpu, rng, n, 0, int(rng.choice([1, 2, 3])), float(rng.uniform(0.02, 0.6)),
                       bool(rng.integers(0, 2)))
        check(gpu, oracle_c, g, int(rng.integers(0, n)))


@pytest.mark.parametrize("whi", [100, 30000, 3_000_000])
def test_weight_encodings(gpu, oracle_c, whi):
    rng = np.random.default_rng(whi)
    for directed in (False, True):
        g = rand_graph(gpu, rng, 700, 1, whi, 0.05, directed)
        r = check(gpu, oracle_c, g, 3)
        assert r.stats["weight_bytes"] == (1 if whi < 255 else 2 if whi < 65535 else 4)


def test_config1_and_golden_hash(gpu, oracle_c):
    import hashlib
    for kind in ("sparse", "dense"):
        g = gpu.generate_sparse(1000, 42) if kind == "sparse" else gpu.generate_dense(1000, 42)
        check(gpu, oracle_c, g, 0)
    case = [c for c in GOLDEN["dataparallel"] if c["name"] == "config1_dense_n1000_seed42"][0]
    r = gpu.dijkstra_dataparallel(gpu.generate_dense(1000, 42), 0)
    h = lambda a: hashlib.sha256(np.ascontiguousarray(a, np.uint64).tobytes()).hexdigest()
    assert h(r.dist) == case["dist_sha"] and h(r.pred) == case["pred_sha"]
    assert r.stats["rounds"] == case["rounds"]


def test_config2_full_size(gpu, oracle_c):
    # BASELINE config 2 (n=16384, ~50 % density): dist == serial's, pred == the
    # reference reconstruction, rounds == the reference's
    g = gpu.generate_bernoulli(16384, 0.5, 16384)
    r = check(gpu, oracle_c, g, 0)
    sd, _ = oracle_c.serial(g.adj, g.n, 0)
    assert np.array_equal(r.dist, sd)
    with gpu.DeviceGraph(g) as dg:
        assert dg.validate(r) == 0


@pytest.mark.parametrize("n,density,whi", [(8191, 0.3, 200), (8193, 0.3, 40000), (9001, 0.05, 400_000)])
def test_ragged_sizes_across_frontier_chunks(gpu, oracle_c, n, density, whi):
    # frontiers larger than one enumeration chunk (kDpChunk = 8192 vertices)
    # and row strides that are not a multiple of the 16-byte load width
    rng = np.random.default_rng(n)
    g = rand_graph(gpu, rng, n, 1, whi, density, bool(n % 2))
    check(gpu, oracle_c, g, int(rng.integers(0, n)))


def test_long_path_many_rounds(gpu, oracle_c):
    # a shuffled chain plus sparse shortcuts: over a hundred relaxation rounds with
    # tiny frontiers, and ties on the shortcuts
    n = 4099
    rng = np.random.default_rng(41)
    adj = np.full((n, n), INF, dtype=np.uint64)
    order = rng.permutation(n)
    adj[order[:-1], order[1:]] = rng.integers(1, 4, size=n - 1, dtype=np.uint64)
    k = n // 8
    u, v = rng.integers(0, n, size=k), rng.integers(0, n, size=k)
    adj[u, v] = rng.integers(2, 50, size=k, dtype=np.uint64)
    np.fill_diagonal(adj, 0)
    g = gpu.Graph(n, True, adj.ravel())
    r = check(gpu, oracle_c, g, int(order[0]))
    assert r.stats["rounds"] > 100
