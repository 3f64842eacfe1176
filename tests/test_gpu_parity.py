"""Parity of the B200 path (C ABI via ctypes) against the CPU oracle.

Bit-exact dist[] AND pred[] (ShortestPathResult operator==, result.hpp:18)
versus dijkstra_serial (serial.hpp:26-68) restated in oracle/sssp_oracle.c,
which tests/test_oracle.py pins to the reference's own compiled code.
Cases mirror the reference suite: test_serial.cpp:11-75,
test_partitioned.cpp:135-228, test_dataparallel.cpp:144-154 and the
acceptance sweep (acceptance.cpp:42-80).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

INF = 0xFFFFFFFFFFFFFFFF


def serial(oracle_c, g, s):
    d, p = oracle_c.serial(g.adj, g.n, s)
    return d, p


def assert_same(res, d, p, ctx=""):
    if not (np.array_equal(res.dist, d) and np.array_equal(res.pred, p)):
        bad = np.nonzero((res.dist != d) | (res.pred != p))[0]
        i = int(bad[0])
        raise AssertionError(f"{ctx}: {len(bad)} mismatches, first v={i}: gpu=({res.dist[i]},"
                             f"{res.pred[i]}) oracle=({d[i]},{p[i]})")


def four(gpu, directed):
    return gpu.graph_from_edges(4, [(0, 1, 2), (0, 2, 4), (1, 2, 1), (1, 3, 3), (2, 3, 5)],
                                directed)


def test_four_vertex_example(gpu):
    # test_serial.cpp:11-19
    r = gpu.dijkstra(four(gpu, False), 0)
    assert r.dist.tolist() == [0, 2, 3, 5]
    assert r.pred.tolist() == [INF, 0, 1, 1]
    assert r.source == 0


def test_four_vertex_visit_order(gpu):
    # test_serial.cpp:69-75
    with gpu.DeviceGraph(four(gpu, False), visit_order=True) as dg:
        r = dg.solve(0, visit_order=True)
    assert r.stats["visit_order"].tolist() == [0, 1, 2, 3]


def test_directed_sink_reaches_nothing(gpu):
    # test_serial.cpp:21-26
    r = gpu.dijkstra(four(gpu, True), 3)
    assert r.dist.tolist() == [INF, INF, INF, 0]
    assert r.pred.tolist() == [INF] * 4


def test_single_vertex(gpu):
    # test_serial.cpp:28-33
    r = gpu.dijkstra(gpu.Graph.no_edges(1), 0)
    assert r.dist.tolist() == [0] and r.pred.tolist() == [INF]


def test_source_out_of_range(gpu):
    # test_serial.cpp:35-38 (std::invalid_argument)
    g = gpu.Graph.no_edges(3)
    with gpu.DeviceGraph(g) as dg:
        with pytest.raises(ValueError):
            dg.solve(3)


def test_zero_weight_tie_fixture(gpu):
    # test_dataparallel.cpp:144-154 graph; serial pred = [2, 2, NONE, 1]
    g = gpu.graph_from_edges(4, [(2, 0, 5), (2, 1, 5), (0, 1, 0), (1, 3, 2)], False)
    r = gpu.dijkstra(g, 2)
    assert r.dist.tolist() == [5, 5, 0, 7]
    assert r.pred.tolist() == [2, 2, INF, 1]


def test_isolated_source(gpu):
    # test_partitioned.cpp:198-204
    g = gpu.Graph.no_edges(5, True)
    g.adj[1 * 5 + 2] = 4
    r = gpu.dijkstra(g, 0)
    assert r.dist.tolist() == [0, INF, INF, INF, INF]


def random_tie_graph(rng, n, wmax, density, directed):
    adj = np.full((n, n), INF, dtype=np.uint64)
    mask = rng.random((n, n)) < density
    w = rng.integers(0, wmax + 1, size=(n, n), dtype=np.uint64)
    adj[mask] = w[mask]
    if not directed:
        iu = np.triu_indices(n, 1)
        adj[(iu[1], iu[0])] = adj[iu]
    np.fill_diagonal(adj, 0)
    return adj


ENGINES = ["cluster", "grid"]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("seed", range(6))
def test_tie_heavy_sweep(gpu, oracle_c, seed, engine):
    """Weights in {0..3} (zero-weight ties), random density, both directions."""
    rng = np.random.default_rng(1000 + seed)
    with_graphs = 0
    for i in range(40):
        n = int(rng.integers(1, 300))
        directed = bool(i % 2)
        adj = random_tie_graph(rng, n, 3, float(rng.choice([0.01, 0.05, 0.2, 0.6, 1.0])), directed)
        g = gpu.Graph(n, directed, adj)
        s = int(rng.integers(0, n))
        with gpu.DeviceGraph(g, engine=engine) as dg:
            r = dg.solve(s)
        d, p = serial(oracle_c, g, s)
        assert_same(r, d, p, f"seed={seed} i={i} n={n}")
        with_graphs += 1
    assert with_graphs == 40


def test_acceptance_sweep_graphs(gpu, oracle_c):
    """acceptance.cpp:42-80: 400 graphs, dense/sparse x dir/undir, n in 7..200,
    rng 20240601 -- full ShortestPathResult equality with serial."""
    rng = oracle_c.rng(20240601)
    checked = 0
    for dense in (False, True):
        for directed in (False, True):
            for _ in range(100):
                n = 7 + rng() % 194
                seed = rng()
                adj = (oracle_c.dense(n, seed, directed) if dense else
                       oracle_c.sparse(n, seed, directed))
                s = rng() % n
                g = gpu.Graph(n, directed, adj)
                r = gpu.dijkstra(g, s)
                d, p = serial(oracle_c, g, s)
                assert_same(r, d, p, f"dense={dense} directed={directed} n={n}")
                checked += 1
    assert checked == 400


@pytest.mark.parametrize("kind", ["sparse", "dense"])
def test_config1_n1000(gpu, oracle_c, kind):
    """BASELINE config 1: n=1000 generate_{sparse,dense}(1000, 42), s=0."""
    g = (gpu.generate_sparse if kind == "sparse" else gpu.generate_dense)(1000, 42)
    r = gpu.dijkstra(g, 0)
    d, p = serial(oracle_c, g, 0)
    assert_same(r, d, p, kind)
    assert oracle_c.validate(g.adj, g.n, 0, r.dist, r.pred) == 0


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("flags", [0, 1, 2, 3])
def test_prefetch_flags_are_semantic_noops(gpu, oracle_c, flags, engine):
    g = gpu.generate_dense(3000, 7)
    d, p = serial(oracle_c, g, 5)
    with gpu.DeviceGraph(g, flags=flags, engine=engine) as dg:
        assert_same(dg.solve(5), d, p, f"flags={flags}")


@pytest.mark.parametrize("n", [2, 31, 127, 128, 129, 255, 4095, 4097, 9000])
@pytest.mark.parametrize("ctas", [0, 1, 3, 7])
def test_layout_edges_grid(gpu, oracle_c, n, ctas):
    """n around the 128-column CTA slice and odd CTA counts (padding columns)."""
    rng = np.random.default_rng(n * 31 + ctas)
    adj = random_tie_graph(rng, n, 2, min(1.0, 8.0 / n + 0.01), False)
    g = gpu.Graph(n, False, adj)
    s = int(rng.integers(0, n))
    d, p = serial(oracle_c, g, s)
    try:
        dg = gpu.DeviceGraph(g, ctas=ctas, engine="grid")
    except gpu.SsspError as e:  # too many columns for that few CTAs
        assert ctas and n > ctas * 2048, str(e)
        return
    with dg:
        assert_same(dg.solve(s), d, p, f"n={n} ctas={ctas}")


@pytest.mark.parametrize("n", [2, 127, 1025, 4097, 9000, 17000])
@pytest.mark.parametrize("ctas,warps", [(0, 4), (0, 8), (0, 16), (1, 8), (3, 4), (16, 16)])
def test_layout_edges_cluster(gpu, oracle_c, n, ctas, warps):
    """cluster sizes 1..16, 4/8/16 warps, padding participants and columns."""
    rng = np.random.default_rng(n * 7 + ctas + warps)
    adj = random_tie_graph(rng, n, 2, min(1.0, 8.0 / n + 0.01), True)
    g = gpu.Graph(n, True, adj)
    s = int(rng.integers(0, n))
    d, p = serial(oracle_c, g, s)
    try:
        dg = gpu.DeviceGraph(g, ctas=ctas, warps=warps, engine="cluster")
    except gpu.SsspError as e:  # cluster sizes are powers of two (Q = C*NW)
        cmax = 1 << (ctas.bit_length() - 1) if ctas else 16
        assert n > cmax * warps * 32 * 32, str(e)
        return
    with dg:
        assert_same(dg.solve(s), d, p, f"n={n} ctas={ctas} warps={warps}")


@pytest.mark.parametrize("wmax,wbytes", [(254, 1), (255, 2), (40000, 2), (65534, 2),
                                         (65535, 4), (3_000_000, 4)])
def test_weight_encodings(gpu, oracle_c, wmax, wbytes):
    rng = np.random.default_rng(wmax)
    n = 700
    adj = np.full((n, n), INF, dtype=np.uint64)
    mask = rng.random((n, n)) < 0.02
    adj[mask] = rng.integers(0, wmax + 1, size=int(mask.sum()), dtype=np.uint64)
    adj[0, 1] = wmax  # make sure the max is present
    np.fill_diagonal(adj, 0)
    g = gpu.Graph(n, True, adj)
    d, p = serial(oracle_c, g, 0)
    with gpu.DeviceGraph(g) as dg:
        info = dg.info()
        assert info["weight_bytes"] == wbytes
        assert_same(dg.solve(0), d, p, f"wmax={wmax}")


def test_unpacked_key_path(gpu, oracle_c):
    """Distances too wide for the single-redux packed key use the 2-stage redux."""
    rng = np.random.default_rng(5)
    n = 3000
    adj = random_tie_graph(rng, n, 1, 0.01, True)
    big = rng.integers(0, 1_000_000, size=(n, n), dtype=np.uint64)
    adj = np.where(adj == INF, adj, adj * big)
    np.fill_diagonal(adj, 0)
    g = gpu.Graph(n, True, adj)
    d, p = serial(oracle_c, g, 0)
    with gpu.DeviceGraph(g) as dg:
        assert dg.info()["packed_key"] == 0
        assert_same(dg.solve(0), d, p, "unpacked")


KMAX = 0xFFFFFFFF  # kMaxWeight (weight.hpp:18): a legal finite weight


def wide_graph(rng, n, directed, wlo, whi, density, zero_frac=0.0):
    adj = np.full((n, n), INF, dtype=np.uint64)
    mask = rng.random((n, n)) < density
    w = rng.integers(wlo, whi, size=(n, n), dtype=np.uint64, endpoint=True)
    if zero_frac:
        w = np.where(rng.random((n, n)) < zero_frac, np.uint64(0), w)
    adj[mask] = w[mask]
    for u in range(n - 1):  # a spanning path keeps most vertices reachable
        adj[u, u + 1] = min(int(adj[u, u + 1]), int(rng.integers(wlo, whi, endpoint=True)))
    if not directed:
        adj = np.minimum(adj, adj.T)
    np.fill_diagonal(adj, 0)
    return adj.reshape(-1)


def test_kmaxweight_fixture_is_exact(gpu, oracle_c):
    """A weight of exactly kMaxWeight = 2^32-1 (weight.hpp:18, graph.hpp:79) is a
    legal finite weight: the solve runs on 64-bit distances (engine WIDE) and
    equals dijkstra_serial -- no SSSP_ERR_WEIGHT_RANGE."""
    for directed in (False, True):
        g = gpu.graph_from_edges(6, [(0, 1, KMAX), (1, 2, KMAX), (0, 2, 7), (2, 3, KMAX - 1),
                                     (3, 4, 1), (1, 4, 0)], directed)
        for s in range(6):
            d, p = serial(oracle_c, g, s)
            with gpu.DeviceGraph(g) as dg:
                assert dg.info()["engine"] == 5 and dg.info()["weight_bytes"] == 8
                r = dg.solve(s)
            assert_same(r, d, p, f"kmax directed={directed} s={s}")


@pytest.mark.parametrize("directed", [False, True])
@pytest.mark.parametrize("wlo,whi", [(1 << 31, KMAX - 1), (3_000_000_000, KMAX), (1, KMAX)])
def test_distances_beyond_32_bits(gpu, oracle_c, directed, wlo, whi):
    """n * max_weight >= 2^32: distances past the 32-bit encoding (u32 weights,
    u64 distances; or u64 weights when kMaxWeight occurs) -- bit-exact."""
    rng = np.random.default_rng(wlo % 1000 + directed)
    for n, dens in [(257, 0.02), (1000, 0.005), (1500, 0.3)]:
        g = gpu.Graph(n, directed, wide_graph(rng, n, directed, wlo, whi, dens))
        for s in (0, n // 2):
            d, p = serial(oracle_c, g, s)
            with gpu.DeviceGraph(g) as dg:
                assert dg.info()["engine"] == 5
                r = dg.solve(s)
            assert_same(r, d, p, f"n={n} s={s}")
            if wlo >= 1 << 31:  # every path of >= 3 edges passes 2^32
                assert int(d[d != INF].max()) > 0xFFFFFFFF


def test_wide_zero_weights_ties_unreachable(gpu, oracle_c):
    """Tie-heavy wide graphs with zero weights and unreachable vertices (the
    strict '<' and lowest-id rules of serial.hpp:42-56 at 64 bits)."""
    rng = np.random.default_rng(77)
    for trial in range(6):
        n = int(rng.integers(50, 700))
        adj = wide_graph(rng, n, bool(trial % 2), KMAX - 2, KMAX, 0.05, zero_frac=0.3)
        adj = adj.reshape(n, n)
        adj[:, n - 3:] = INF  # the last 3 vertices unreachable
        np.fill_diagonal(adj, 0)
        g = gpu.Graph(n, bool(trial % 2), adj.reshape(-1))
        s = int(rng.integers(0, n - 3))
        d, p, vo = oracle_c.serial(g.adj, n, s, visit_order=True)
        with gpu.DeviceGraph(g, visit_order=True) as dg:
            r = dg.solve(s, visit_order=True)
            batch = dg.solve_batch([s, 0, n - 1])
        assert_same(r, d, p, f"trial {trial}")
        assert np.array_equal(r.stats["visit_order"], vo)
        for src, rb in zip([s, 0, n - 1], batch):
            d2, p2 = serial(oracle_c, g, src)
            assert_same(rb, d2, p2, f"batch s={src}")


def test_wide_edge_list_and_partitioned(gpu, oracle_c):
    """The device edge-list build and dijkstra_partitioned take kMaxWeight too
    (a wide graph runs on one shard: the result does not depend on p)."""
    edges = [(0, 1, KMAX), (1, 2, 5), (2, 3, KMAX), (0, 3, KMAX), (3, 4, KMAX), (4, 5, 0)]
    for directed in (False, True):
        g = gpu.graph_from_edges(6, edges, directed)
        d, p = serial(oracle_c, g, 0)
        with gpu.DeviceGraph.from_edges(6, edges, directed) as dg:
            assert_same(dg.solve(0), d, p, "edges")
        r = gpu.dijkstra_partitioned(g, 0, 3)
        assert_same(r, d, p, "partitioned")
        assert r.stats["allreduce_count"] == 6


def test_reference_counters_and_collective_stats(gpu, oracle_c):
    """OpCounters (serial.hpp:16-19, pinned by test_serial.cpp:40-51: n*n each)
    and CollectiveStats (partitioned.hpp:196-221: padded_n, scatter / gather
    bytes, zero for one worker -- test_partitioned.cpp:132, 162, 230-237)."""
    g = gpu.generate_sparse(1001, 3)
    d, p, ct = oracle_c.serial(g.adj, g.n, 0, counters=True)
    with gpu.DeviceGraph(g) as dg:
        r = dg.solve(0)
    st = r.stats
    assert st["extract_min_scans"] == ct[0] == 1001 * 1001
    assert st["ref_relax_checks"] == ct[1] == 1001 * 1001
    assert st["allreduce_count"] == 1001 and st["scatter_bytes"] == 0 and st["gather_bytes"] == 0
    assert st["download_bytes"] == 1001 * 16 and st["upload_bytes"] == 1001 * 1001 * st["weight_bytes"]
    assert st["exchanges"] >= 1 and st["barriers"] >= st["exchanges"] - 1
    for P in (2, 3, 8, 12):
        rp = gpu.dijkstra_partitioned(g, 0, P)
        assert_same(rp, d, p, f"P={P}")
        padded = gpu.pad_vertex_count(1001, P)
        loc = padded // P
        assert rp.stats["allreduce_count"] == padded
        assert rp.stats["scatter_bytes"] == (P - 1) * padded * loc * 8
        assert rp.stats["gather_bytes"] == (P - 1) * loc * 16
        assert rp.stats["phases"]["rounds_s"] > 0
    # the device's own exchange counts: n-round engines one per election
    with gpu.DeviceGraph(g, engine="cluster") as dg:
        rc = dg.solve(0)
    assert rc.stats["exchanges"] == rc.stats["iterations"] == int(np.count_nonzero(d != INF))
    # bucket: one exchange per distance class, barriers counted by the kernel
    gd = gpu.generate_dense(2048, 5)
    with gpu.DeviceGraph(gd, engine="bucket") as dg:
        rb = dg.solve(0)
    assert rb.stats["exchanges"] == rb.stats["classes"] and rb.stats["barriers"] >= 2
    # matrix bytes the kernel loaded: at most the rows it touched (+ the source row)
    assert 0 < rb.stats["bytes_read"] <= (rb.stats["rows_read"] + 1) * 2048 * rb.stats["weight_bytes"]
    # the C ABI struct carries the shard count's CollectiveStats too
    with gpu.DeviceGraph(g, [0, 0, 0]) as dg:
        r3 = dg.solve(0)
    assert r3.stats["allreduce_count"] == gpu.pad_vertex_count(1001, 3)
    assert r3.stats["scatter_bytes"] == 2 * 1002 * 334 * 8


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_logical_shards_bit_identical(gpu, oracle_c, P, engine):
    """P column shards on one GPU run the multi-GPU exchange protocol (peer
    stores into every shard's array); result == serial (test_partitioned.cpp
    :149-165, 184-196)."""
    for n, seed in [(1000, 3), (2049, 4)]:
        g = gpu.generate_sparse(n, seed) if seed % 2 else gpu.generate_dense(n, seed)
        d, p = serial(oracle_c, g, 7)
        with gpu.DeviceGraph(g, [0] * P, engine=engine) as dg:
            r = dg.solve(7)
        assert_same(r, d, p, f"P={P} n={n}")


def test_shards_p_greater_than_n(gpu, oracle_c):
    # test_partitioned.cpp:149-165 includes p > n (padding-only shards)
    g = four(gpu, False)
    d, p = serial(oracle_c, g, 0)
    assert_same(gpu.dijkstra_partitioned(g, 0, 7), d, p, "p>n")


@pytest.mark.parametrize("engine", ENGINES)
def test_batch_sources(gpu, oracle_c, engine):
    g = gpu.generate_dense(2000, 11)
    sources = list(range(0, 2000, 31))
    with gpu.DeviceGraph(g, engine=engine) as dg:
        res = dg.solve_batch(sources)
    for s, r in zip(sources, res):
        d, p = serial(oracle_c, g, s)
        assert_same(r, d, p, f"s={s}")


def test_repeated_solves_are_deterministic(gpu):
    g = gpu.generate_sparse(5000, 8)
    with gpu.DeviceGraph(g) as dg:
        a = dg.solve(0)
        b = dg.solve(0)
        c = dg.solve(17)
        d = dg.solve(0)
    assert a == b == d and not (a == c)


def test_visit_order_matches_serial(gpu, oracle_c):
    g = gpu.generate_sparse(3000, 9, directed=True)
    d, p, vo = oracle_c.serial(g.adj, g.n, 0, visit_order=True)
    finite = int(np.count_nonzero(d != INF))
    with gpu.DeviceGraph(g, visit_order=True) as dg:
        r = dg.solve(0, visit_order=True)
    assert r.stats["iterations"] == finite
    # all n rounds, unreachable vertices included (serial.hpp:41-48)
    assert np.array_equal(r.stats["visit_order"], vo)


def test_config2_n16384_bernoulli(gpu, oracle_c):
    """BASELINE config 2: n=16384, Bernoulli(0.5), undirected, s=0."""
    g = gpu.generate_bernoulli(16384, 0.5, 16384)
    r = gpu.dijkstra(g, 0)
    d, p = serial(oracle_c, g, 0)
    assert_same(r, d, p, "config2")


@pytest.fixture(scope="module")
def config3(gpu, oracle_c):
    g = gpu.generate_dense(32768, 32768)
    d, p = serial(oracle_c, g, 0)
    return g, d, p


@pytest.mark.parametrize("engine", ENGINES)
def test_config3_n32768_dense(gpu, config3, engine):
    """BASELINE config 3 on one GPU: generate_dense(32768, 32768), s=0."""
    g, d, p = config3
    with gpu.DeviceGraph(g, engine=engine) as dg:
        r = dg.solve(0)
        st = r.stats
    assert_same(r, d, p, "config3")
    assert st["iterations"] == 32768 and st["weight_bytes"] == 1


def test_config3_two_logical_shards(gpu, config3):
    """Config 3 column-partitioned over 2 shards (cluster engine, P2P mailbox)."""
    g, d, p = config3
    with gpu.DeviceGraph(g, [0, 0]) as dg:
        assert_same(dg.solve(0), d, p, "config3 P=2")


def test_cpp_dropin_against_reference_binary(gpu):
    """include/sssp/cuda.hpp compiled with the reference headers
    (oracle/_ref/test_dropin): cuda::dijkstra(g,s) == dijkstra_serial(g,s)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "test_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASS" in out.stdout


@pytest.mark.parametrize("engine", ["auto", "cluster", "grid"])
def test_queued_enqueues_then_finish(gpu, oracle_c, engine):
    """Several sssp_enqueue calls queue in stream order; finish reports the last."""
    g = gpu.generate_dense(1500, 3)
    with gpu.DeviceGraph(g, engine=engine) as dg:
        for s in (5, 9, 11):
            dg.enqueue([s])
        st = dg.finish()
        assert st["iterations"] == 1500 and st["rounds_s"] > 0
        r = dg.solve(11)
    d, p = oracle_c.serial(g.adj, g.n, 11)
    assert np.array_equal(r.dist, d) and np.array_equal(r.pred, p)


@pytest.mark.parametrize("warps", [4, 8, 16])
@pytest.mark.parametrize("P", [1, 2])
def test_hierarchical_cluster_variant(gpu, oracle_c, warps, P):
    """flag 8: CTA pre-reduction + C-key DSMEM exchange (+ P2P mailbox for P>1)."""
    rng = np.random.default_rng(warps * 10 + P)
    for i in range(12):
        n = int(rng.integers(2, 3000))
        directed = bool(i % 2)
        adj = random_tie_graph(rng, n, 3, float(rng.choice([0.002, 0.05, 0.5])), directed)
        g = gpu.Graph(n, directed, adj)
        s = int(rng.integers(0, n))
        d, p = serial(oracle_c, g, s)
        with gpu.DeviceGraph(g, [0] * P, engine="cluster", flags=3 | 8, warps=warps) as dg:
            assert_same(dg.solve(s), d, p, f"hier n={n} warps={warps} P={P}")


def test_round_times_trace(gpu, oracle_c):
    # per-round %globaltimer stamps of the n-round kernel; tracing
    # must not change the result, and AUTO stays on a scan engine with it
    g = gpu.generate_dense(3000, 77)
    d, p = oracle_c.serial(g.adj, g.n, 5)
    with gpu.DeviceGraph(g, round_times=True) as dg:
        r = dg.solve(5)
        t = dg.round_times()
        assert r.stats["engine"] in (1, 2)
        assert np.array_equal(r.dist, d) and np.array_equal(r.pred, p)
        assert len(t) == r.stats["iterations"] == g.n
        assert np.all(np.diff(t.astype(np.int64)) > 0)
        r2 = dg.solve(6)  # stamps restart for every solve
        assert len(dg.round_times()) == r2.stats["iterations"]


@pytest.mark.parametrize("engine", ["auto", "cluster"])
def test_interleaved_graphs_of_different_sizes(gpu, oracle_c, engine):
    # the per-kernel dynamic shared-memory limit is process-wide: a small graph
    # created after a large one must not break the large one's launches
    big = gpu.generate_dense(8192, 5)
    small = gpu.generate_dense(500, 6)
    db, pb = oracle_c.serial(big.adj, big.n, 3)
    ds, ps = oracle_c.serial(small.adj, small.n, 3)
    with gpu.DeviceGraph(big, engine=engine) as gb:
        r1 = gb.solve(3)
        with gpu.DeviceGraph(small, engine=engine) as gs:
            r2 = gs.solve(3)
            r3 = gb.solve(3)
    assert np.array_equal(r1.dist, db) and np.array_equal(r1.pred, pb)
    assert np.array_equal(r2.dist, ds) and np.array_equal(r2.pred, ps)
    assert np.array_equal(r3.dist, db) and np.array_equal(r3.pred, pb)
