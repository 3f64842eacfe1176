"""The distance-class (bucket) engine: bit-identical to dijkstra_serial
whenever every finite off-diagonal weight is >= 1 (bucket_kernel.cuh), and
never selected otherwise.  Covers push and pull steps, symmetric (pull from
the matrix) and asymmetric (pull from the transpose) graphs, many classes,
all weight encodings and batches."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
INF = 0xFFFFFFFFFFFFFFFF


def rand_graph(rng, n, wlo, whi, density, directed):
    adj = np.full((n, n), INF, dtype=np.uint64)
    m = rng.random((n, n)) < density
    adj[m] = rng.integers(wlo, whi + 1, size=int(m.sum()), dtype=np.uint64)
    if not directed:
        iu = np.triu_indices(n, 1)
        adj[(iu[1], iu[0])] = adj[iu]
    np.fill_diagonal(adj, 0)
    return adj


def check(gpu, oracle_c, g, s, devices=(0,), **kw):
    d, p = oracle_c.serial(g.adj, g.n, s)
    with gpu.DeviceGraph(g, devices, **kw) as dg:
        info = dg.info()
        r = dg.solve(s)
    ok = np.array_equal(r.dist, d) and np.array_equal(r.pred, p)
    if not ok:
        bad = np.nonzero((r.dist != d) | (r.pred != p))[0]
        i = int(bad[0])
        raise AssertionError(f"n={g.n} s={s}: {len(bad)} mismatches, v={i} gpu=({r.dist[i]},"
                             f"{r.pred[i]}) want=({d[i]},{p[i]}) engine={info['engine']}")
    return info, r


@pytest.mark.parametrize("seed", range(8))
def test_bucket_tie_heavy_positive_weights(gpu, oracle_c, seed):
    rng = np.random.default_rng(300 + seed)
    for i in range(25):
        n = int(rng.integers(2, 400))
        directed = bool(i % 2)
        g = gpu.Graph(n, directed, rand_graph(rng, n, 1, 3, float(rng.choice([0.005, 0.02, 0.1, 0.5, 1.0])),
                                             directed))
        info, r = check(gpu, oracle_c, g, int(rng.integers(0, n)), engine="bucket")
        assert info["engine"] == 3


def test_auto_selects_bucket_only_when_exact(gpu, oracle_c):
    rng = np.random.default_rng(7)
    g = gpu.Graph(300, False, rand_graph(rng, 300, 1, 5, 0.1, False))
    info, _ = check(gpu, oracle_c, g, 0)
    assert info["engine"] == 3
    g0 = gpu.Graph(300, False, rand_graph(rng, 300, 0, 5, 0.1, False))  # zero weights
    info, _ = check(gpu, oracle_c, g0, 0)
    assert info["engine"] == 2
    with pytest.raises(gpu.SsspError):
        gpu.DeviceGraph(g0, engine="bucket")


@pytest.mark.parametrize("kind", ["dense", "sparse", "sparse_directed", "bern_directed"])
def test_bucket_generated_graphs(gpu, oracle_c, kind):
    for n, seed in [(1000, 42), (2049, 5), (5000, 11)]:
        if kind == "dense":
            g = gpu.generate_dense(n, seed)
        elif kind == "sparse":
            g = gpu.generate_sparse(n, seed)
        elif kind == "sparse_directed":
            g = gpu.generate_sparse(n, seed, directed=True)
        else:
            g = gpu.generate_bernoulli(n, 0.01, seed, directed=True)
        for s in (0, n // 3, n - 1):
            info, r = check(gpu, oracle_c, g, s, engine="bucket")
            assert r.stats["engine"] == 3 and r.stats["classes"] >= 1


@pytest.mark.parametrize("wmax,wbytes", [(254, 1), (3000, 2), (70000, 4)])
def test_bucket_weight_encodings(gpu, oracle_c, wmax, wbytes):
    rng = np.random.default_rng(wmax)
    for directed in (False, True):
        g = gpu.Graph(600, directed, rand_graph(rng, 600, 1, wmax, 0.05, directed))
        info, _ = check(gpu, oracle_c, g, 3, engine="bucket")
        assert info["weight_bytes"] == wbytes


def test_bucket_batch_and_repeat(gpu, oracle_c):
    g = gpu.generate_dense(3000, 17)
    srcs = [0, 1, 999, 2999, 1500]
    with gpu.DeviceGraph(g, engine="bucket") as dg:
        res = dg.solve_batch(srcs)
        again = dg.solve(999)
    for s, r in zip(srcs, res):
        d, p = oracle_c.serial(g.adj, g.n, s)
        assert np.array_equal(r.dist, d) and np.array_equal(r.pred, p)
    assert again == res[2]


def test_bucket_unreachable_and_isolated(gpu, oracle_c):
    g = gpu.Graph.no_edges(700, True)
    g.adj[5 * 700 + 6] = 3
    g.adj[6 * 700 + 9] = 1
    check(gpu, oracle_c, g, 5, engine="bucket")
    check(gpu, oracle_c, g, 0, engine="bucket")


def test_bucket_config3(gpu, oracle_c):
    g = gpu.generate_dense(32768, 32768)
    info, r = check(gpu, oracle_c, g, 0, engine="bucket")
    assert r.stats["classes"] == 4


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_bucket_logical_shards(gpu, oracle_c, P):
    """Bucket engine over P column shards on one GPU: global class bitmap
    all-gathered by every tile into every shard, cross-shard barrier by
    system-scope atomics, pull from the sharded transpose."""
    rng = np.random.default_rng(P)
    cases = [gpu.generate_dense(1000, 3), gpu.generate_sparse(2049, 4),
             gpu.generate_sparse(1500, 5, directed=True),
             gpu.Graph(700, True, rand_graph(rng, 700, 1, 3, 0.02, True))]
    for g in cases:
        for s in (0, g.n - 1):
            info, r = check(gpu, oracle_c, g, s, devices=[0] * P)
            assert info["engine"] == 3 and info["shards"] == P


def test_bucket_logical_shards_config3(gpu, oracle_c):
    g = gpu.generate_dense(32768, 32768)
    info, r = check(gpu, oracle_c, g, 0, devices=[0, 0])
    assert info["engine"] == 3 and r.stats["classes"] == 4


@pytest.mark.parametrize("directed", [False, True])
@pytest.mark.parametrize("wmax", [3, 200, 5000, 100000])
def test_device_build_from_edges(gpu, oracle_c, directed, wmax):
    """sssp_graph_create_from_edges == graph_from_edges (graph.hpp:73-88) on the
    host: duplicates keep the minimum, undirected edges are mirrored."""
    rng = np.random.default_rng(wmax + directed)
    n, m = 900, 6000
    u = rng.integers(0, n, m)
    v = (u + rng.integers(1, n, m)) % n           # no self-loops
    w = rng.integers(0 if wmax == 3 else 1, wmax + 1, m)
    e = np.stack([u, v, w], 1).astype(np.uint64)
    e = np.concatenate([e, e[:500] * np.array([1, 1, 0], np.uint64) + np.array([0, 0, 1], np.uint64)])
    g = gpu.graph_from_edges(n, e, directed)
    for s in (0, 450):
        d, p = oracle_c.serial(g.adj, n, s)
        with gpu.DeviceGraph.from_edges(n, e, directed) as dg:
            r = dg.solve(s)
        assert np.array_equal(r.dist, d) and np.array_equal(r.pred, p)


def test_device_build_rejects_like_reference(gpu):
    for bad in ([(0, 5, 1)], [(2, 2, 1)], [(0, 1, 1 << 32)]):
        with pytest.raises(ValueError):
            gpu.DeviceGraph.from_edges(5, bad, False)


def test_device_build_config1_and_shards(gpu, oracle_c):
    e = oracle_c.sparse_edges(1000, 42)
    adj = oracle_c.from_edges(1000, e, False)
    d, p = oracle_c.serial(adj, 1000, 0)
    for devs in ([0], [0, 0, 0]):
        with gpu.DeviceGraph.from_edges(1000, e, False, devs) as dg:
            r = dg.solve(0)
        assert np.array_equal(r.dist, d) and np.array_equal(r.pred, p)


@pytest.mark.parametrize("tile_bytes", [256, 512, 1024])
def test_bucket_tile_sizes(gpu, oracle_c, tile_bytes, monkeypatch):
    # wider tiles (fewer CTAs, more positions per CTA): push slices of 16 B
    # per thread over more row groups, more pulled columns per CTA range
    monkeypatch.setenv("SSSP_BUCKET_TILE_BYTES", str(tile_bytes))
    rng = np.random.default_rng(tile_bytes)
    for directed in (False, True):
        g = gpu.Graph(1500, directed, rand_graph(rng, 1500, 1, 9, 0.3, directed).ravel())
        info, _ = check(gpu, oracle_c, g, 11, engine="bucket")
        assert info["engine"] == 3
    g = gpu.generate_dense(4096, 4096)
    info, _ = check(gpu, oracle_c, g, 0, engine="bucket")
    assert info["engine"] == 3


@pytest.mark.parametrize("directed", [False, True])
def test_bucket_multislot_batches(gpu, oracle_c, directed):
    # several independent solves share one launch (slots); sources finish after
    # different class counts (one isolated, one on a long path), k is not a
    # multiple of the slot count, and pull steps occur in some slots only
    rng = np.random.default_rng(77 + directed)
    n = 1200
    adj = rand_graph(rng, n, 1, 30, 0.05, directed)
    adj[7, :] = INF
    adj[:, 7] = INF
    adj[7, 7] = 0  # vertex 7 isolated: its solve ends after class 0
    for u in range(100, 140):  # a light path: many classes from vertex 100
        adj[u, u + 1] = 1
    g = gpu.Graph(n, directed, adj.ravel())
    srcs = [0, 7, 100, 5, 999, 3, 100, 42, 1199, 7, 64, 12, 300]
    with gpu.DeviceGraph(g, engine="bucket") as dg:
        res = dg.solve_batch(srcs)
        assert dg.info()["engine"] == 3
    for s, r in zip(srcs, res):
        d, p = oracle_c.serial(g.adj, n, s)
        assert np.array_equal(r.dist, d) and np.array_equal(r.pred, p), s


@pytest.mark.parametrize("engine", ["bucket", "auto"])
def test_long_chain_thousands_of_classes(gpu, oracle_c, engine):
    # a shuffled chain with sparse shortcuts: distance classes >> n/8, so AUTO
    # leaves the bucket engine; forced, it must still be exact
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
    info, _ = check(gpu, oracle_c, g, int(order[0]), engine=engine)
    if engine == "bucket":
        assert info["engine"] == 3


def test_auto_picks_scan_engine_on_the_first_call(gpu, oracle_c):
    """The drop-in creates a handle per call, so AUTO must choose per call: a
    graph with more than n/12 distance classes (config 1 sparse: 154 at
    n=1000) stops the bucket solve on its class budget and reruns on the
    n-round cluster engine inside the same dijkstra(G, s) -- exact either way."""
    g = gpu.generate_sparse(1000, 42)
    d, p = oracle_c.serial(g.adj, g.n, 0)
    r = gpu.dijkstra(g, 0)
    assert np.array_equal(r.dist, d) and np.array_equal(r.pred, p)
    assert r.stats["engine"] == 2
    with gpu.DeviceGraph(g) as dg:
        r1 = dg.solve(0)
        assert r1.stats["engine"] == 2 and dg.info()["engine"] == 2  # kept for later solves
        r2 = dg.solve(999)
    d2, p2 = oracle_c.serial(g.adj, g.n, 999)
    assert np.array_equal(r2.dist, d2) and np.array_equal(r2.pred, p2)
    # few classes: AUTO stays on the bucket engine
    gd = gpu.generate_dense(1000, 42)
    rd = gpu.dijkstra(gd, 0)
    assert rd.stats["engine"] == 3


@pytest.mark.parametrize("wmax", [100, 3000, 70000])
@pytest.mark.parametrize("n", [256, 1000, 4096])
def test_bucket_symmetry_detection_single_element(gpu, oracle_c, n, wmax):
    """The upload's symmetry check (symmetric_check_wide_kernel on 128 B row
    segments, symmetric_check_kernel otherwise) decides whether pull steps may
    read row v as column v: a symmetric matrix keeps no transpose, and ONE
    asymmetric element anywhere -- including the first and last rows and
    columns -- makes the upload build it (matrix_bytes doubles)."""
    rng = np.random.default_rng(n + wmax)
    adj = rand_graph(rng, n, 1, wmax, 0.3, False)
    g = gpu.Graph(n, False, adj.copy())
    info, _ = check(gpu, oracle_c, g, 0, engine="bucket")
    base = info["matrix_bytes"]
    for (u, v) in [(0, n - 1), (n - 1, 0), (n // 2, n // 3), (1, 0)]:
        a2 = adj.copy()
        a2[u, v] = INF if a2[u, v] != INF else np.uint64(wmax)
        g2 = gpu.Graph(n, True, a2)
        for s in (0, u, v):
            info2, _ = check(gpu, oracle_c, g2, s, engine="bucket")
        assert info2["matrix_bytes"] > base, (u, v)  # the transpose was built


@pytest.mark.parametrize("wmax", [30, 254, 3000])
@pytest.mark.parametrize("n,density,directed", [(1000, 0.01, True), (1500, 0.004, False),
                                                (3000, 0.002, True), (4096, 0.02, False)])
def test_bucket_sparse_tile_lists(gpu, oracle_c, n, density, directed, wmax):
    # density <= 1/32 (u8) / 1/16 (u16): the upload builds per-tile finite-entry
    # lists (tile_list_kernel) and every push reads them instead of the dense
    # row slices, pulls off; n not a power of two pads the positions.  Kernel-
    # counted bytes drop below a dense slice per pushed row.
    rng = np.random.default_rng(n + wmax + directed)
    adj = rand_graph(rng, n, 1, wmax, density, directed)
    for u in range(10, 60):  # a light path: many classes, small B_d
        adj[u, u + 1] = 1
    g = gpu.Graph(n, directed, adj.ravel())
    srcs = [0, 10, n - 1, 17]
    want = [oracle_c.serial(g.adj, n, s) for s in srcs]
    with gpu.DeviceGraph(g, engine="bucket") as dg:
        info = dg.info()
        assert info["engine"] == 3 and info["weight_bytes"] == (1 if wmax < 255 else 2)
        for s, (d, p) in zip(srcs, want):
            r = dg.solve(s)
            assert np.array_equal(r.dist, d) and np.array_equal(r.pred, p), (s, "single")
            # dense: every pushed row costs its whole (padded) row across the
            # tiles; sparse: 8 B of offsets per tile + 4 B per finite entry
            wb = info["weight_bytes"]
            if r.stats["rows_read"] > 8:
                assert r.stats["bytes_read"] < r.stats["rows_read"] * n * wb / 2, r.stats
        for s, r in zip(srcs, dg.solve_batch(srcs)):
            d, p = want[srcs.index(s)]
            assert np.array_equal(r.dist, d) and np.array_equal(r.pred, p), (s, "batch")


@pytest.mark.parametrize("split", ["1", "0"])
def test_bucket_sparse_row_split_push(split):
    # the row-split push (classes of >= SSSP_SPLIT_ROWS rows: rows divided over
    # every warp, global atomicMin into the per-column keys, one extra barrier)
    # forced on every class after the first (1), and the tile-local sparse push
    # only (0): the sparse-list cases above rerun in a fresh process (the
    # switch is read once per process)
    import os
    import subprocess
    import sys
    env = dict(os.environ, SSSP_SPLIT_ROWS=split)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        f"{__file__}::test_bucket_sparse_tile_lists", f"{__file__}::test_bucket_multislot_batches"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
