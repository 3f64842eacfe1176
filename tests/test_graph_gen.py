"""Host-side graph builders of the product (include/sssp_graph_gen.h and the
Python parse_edge_list mirror) against the reference: generate.hpp:15-83,
graph.hpp:73-88 and :126-174 (test_generate.cpp, test_graph.cpp)."""
import ctypes
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2504_03667_b200 as P

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.uint64).tobytes()).hexdigest()


def test_dense_generator_golden():
    for key, hh in GOLDEN["generate_dense_matrix"].items():
        n, s = map(int, key.split(":"))
        assert h(P.generate_dense(n, s).adj) == hh


def test_generators_match_reference(ref):
    for n in (7, 8, 13, 64, 257):
        for seed in (0, 1, 99):
            for directed in (False, True):
                assert np.array_equal(P.generate_dense(n, seed, directed).adj, ref.dense(n, seed, directed))
                assert np.array_equal(P.generate_sparse(n, seed, directed).adj, ref.sparse(n, seed, directed))


def test_column_blocks_match_full_matrix():
    n = 211
    full = {"dense": P.generate_dense(n, 5).matrix(), "sparse": P.generate_sparse(n, 5).matrix(),
            "bern": P.generate_bernoulli(n, 0.3, 5, directed=True).matrix()}
    for cb, cc in [(0, 211), (0, 53), (53, 53), (159, 52), (100, 0)]:
        assert np.array_equal(P.generate_dense(n, 5, cols=(cb, cc)), full["dense"][:, cb:cb + cc])
        assert np.array_equal(P.generate_sparse(n, 5, cols=(cb, cc)), full["sparse"][:, cb:cb + cc])
        assert np.array_equal(P.generate_bernoulli(n, 0.3, 5, True, cols=(cb, cc)),
                              full["bern"][:, cb:cb + cc])


def test_bernoulli_matches_oracle(oracle_c):
    for n, p, seed, directed in [(300, 0.5, 16384, False), (400, 0.001, 65536, True), (50, 1.0, 1, True)]:
        assert np.array_equal(P.generate_bernoulli(n, p, seed, directed).adj,
                              oracle_c.bernoulli(n, p, seed, directed))


def test_dense_and_sparse_edge_counts():
    # test_generate.cpp: n(n-1)/2 and 3n distinct edges, undirected symmetric
    for n in (10, 100):
        g = P.generate_dense(n, 3).matrix()
        assert np.count_nonzero(np.triu(g != P.INF, 1)) == n * (n - 1) // 2
        s = P.generate_sparse(n, 3).matrix()
        assert np.count_nonzero(np.triu(s != P.INF, 1)) == 3 * n
        assert np.array_equal(s, s.T)
    with pytest.raises(ValueError):
        P.generate_sparse(6, 1)
    with pytest.raises(ValueError):
        P.generate_dense(1, 1)


def test_graph_from_edges_semantics(ref):
    edges = [(0, 1, 9), (1, 0, 4), (0, 1, 6), (2, 3, 0), (3, 1, 0xFFFFFFFF)]
    for directed in (False, True):
        assert np.array_equal(P.graph_from_edges(4, edges, directed).adj, ref.from_edges(4, edges, directed))
    for bad in ([(0, 4, 1)], [(1, 1, 1)], [(0, 1, 0x100000000)]):
        with pytest.raises(ValueError):
            P.graph_from_edges(4, bad, False)


@pytest.mark.parametrize("key", sorted(GOLDEN["parse"]["results"]))
def test_parse_edge_list_matches_reference_golden(key):
    name, directed = key.rsplit(":", 1)
    text = GOLDEN["parse"]["texts"][name]
    want = GOLDEN["parse"]["results"][key]
    if want[0] == "ok":
        g = P.parse_edge_list(text, bool(int(directed)))
        assert g.n == want[1] and h(g.adj) == want[2]
    else:
        with pytest.raises(P.ParseError) as ei:
            P.parse_edge_list(text, bool(int(directed)))
        assert ei.value.line == want[1]
        assert str(ei.value) == want[2]


def test_parse_edge_list_four_vertex(ref):
    text = "4 5\n0 1 2\n0 2 4\n1 2 1\n1 3 3\n2 3 5\n"
    for directed in (False, True):
        st, n, adj = ref.parse(text, directed)
        assert st == "ok"
        assert np.array_equal(P.parse_edge_list(text, directed).adj, adj)


def _random_edge_text(rng, n, m, corrupt):
    lines = []
    if rng.random() < 0.3:
        lines.append("# comment")
    lines.append(f"{n} {m}")
    for i in range(m + (1 if corrupt == "extra" else 0) - (1 if corrupt == "fewer" else 0)):
        u, v = int(rng.integers(0, n)), int(rng.integers(0, n))
        if u == v:
            v = (u + 1) % n
        w = int(rng.integers(0, 1000))
        sep = "\t" if rng.random() < 0.2 else " "
        lines.append(f"{u}{sep}{v} {w}" + ("\r" if rng.random() < 0.2 else ""))
        if rng.random() < 0.1:
            lines.append("" if rng.random() < 0.5 else "   # note")
    if corrupt in ("token", "range", "self", "neg", "fields", "big"):
        k = int(rng.integers(1, len(lines)))
        lines[k] = {"token": "1 x 3", "range": f"0 {n} 1", "self": "2 2 5", "neg": "0 1 -3",
                    "fields": "0 1", "big": "0 1 4294967296"}[corrupt]
    return "\n".join(lines) + ("\n" if rng.random() < 0.7 else "")


@pytest.mark.parametrize("seed", range(4))
def test_native_parser_matches_reference(ref, seed):
    # sssp_parse_edge_list splits the body over all host threads; the first
    # error (line, message) and the matrix must equal the sequential reference
    rng = np.random.default_rng(900 + seed)
    kinds = [None, "extra", "fewer", "token", "range", "self", "neg", "fields", "big"]
    for i in range(60):
        n = int(rng.integers(3, 40))
        m = int(rng.integers(0, 300))
        text = _random_edge_text(rng, n, m, kinds[i % len(kinds)])
        for directed in (False, True):
            want = ref.parse(text, directed)
            if want[0] == "ok":
                g = P.parse_edge_list(text, directed)
                assert g.n == want[1] and np.array_equal(g.adj, want[2]), (i, directed)
            else:
                with pytest.raises(P.ParseError) as ei:
                    P.parse_edge_list(text, directed)
                assert ei.value.line == want[1] and str(ei.value) == want[2], (i, text)


def test_header_m_not_backed_by_body_fails_before_allocation(ref):
    # A header whose m the body does not back must give the reference's
    # ParseError from the header-only call (graph.hpp:166-168), before the
    # caller sizes a 3*m buffer (here 24 GB).
    text = "3 1000000000\n0 1 5\n1 2 6\n"
    want = ref.parse(text, False)
    assert want[0] != "ok"
    n, m, line = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    err = ctypes.create_string_buffer(256)
    data = text.encode()
    rc = P.lib.sssp_parse_edge_list(data, len(data), ctypes.byref(n), ctypes.byref(m), None, 0,
                                    ctypes.byref(line), err, len(err))
    assert rc != 0 and line.value == want[1]
    with pytest.raises(P.ParseError) as ei:
        P.parse_edge_list(text, False)
    assert ei.value.line == want[1] and str(ei.value) == want[2]
    # a body line error after a short body: the first error wins, as in the reference
    text2 = "3 5\n0 1 5\n1 1 6\n"
    want2 = ref.parse(text2, True)
    with pytest.raises(P.ParseError) as ei:
        P.parse_edge_list(text2, True)
    assert ei.value.line == want2[1] and str(ei.value) == want2[2]
