"""Regenerates tests/golden/* from the REFERENCE's own code (oracle/_ref, the
unmodified /root/reference/proj/include headers behind oracle/ref_shim.cpp).
Run in the build container: python tests/golden/make_golden.py"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

INF = 0xFFFFFFFFFFFFFFFF


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.uint64).tobytes()).hexdigest()


def main():
    R = oracle.REF()
    C = oracle.C()  # only for its mt19937_64 stream (rng), pinned in tests/test_oracle.py
    out = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref/libref_sssp.so",
           "cases": []}

    def case(name, adj, n, source, directed, keep_arrays=True):
        d, p, vo, ct = R.serial(adj, n, source, visit_order=True, counters=True)
        c = {"name": name, "n": n, "source": source, "directed": directed,
             "adj_sha256": h(adj), "dist_sha256": h(d), "pred_sha256": h(p),
             "visit_order_sha256": h(vo), "counters": [int(x) for x in ct]}
        if keep_arrays:
            c["dist"] = [int(x) for x in d]
            c["pred"] = [int(x) for x in p]
            c["visit_order"] = [int(x) for x in vo]
        out["cases"].append(c)

    four = [(0, 1, 2), (0, 2, 4), (1, 2, 1), (1, 3, 3), (2, 3, 5)]
    case("four_vertex_undirected_s0", R.from_edges(4, four, False), 4, 0, False)   # test_serial.cpp:11-19
    case("four_vertex_directed_s3", R.from_edges(4, four, True), 4, 3, True)        # test_serial.cpp:21-26
    case("single_vertex", np.zeros(1, np.uint64), 1, 0, False)                      # test_serial.cpp:28-33
    zw = [(2, 0, 5), (2, 1, 5), (0, 1, 0), (1, 3, 2)]
    case("zero_weight_tie_s2", R.from_edges(4, zw, False), 4, 2, False)              # test_dataparallel.cpp:144-154
    for kind in ("sparse", "dense"):                                                 # BASELINE config 1
        adj = R.dense(1000, 42) if kind == "dense" else R.from_edges(1000, R.sparse_edges(1000, 42), False)
        case(f"config1_{kind}_n1000_seed42", adj, 1000, 0, False)
    # acceptance.cpp:42-80 sweep: rng 20240601, 400 graphs, hashes only
    rng = C.rng(20240601)
    sweep = []
    for dense in (False, True):
        for directed in (False, True):
            for _ in range(100):
                n = 7 + rng() % 194
                seed = rng()
                adj = R.dense(n, seed, directed) if dense else R.from_edges(n, R.sparse_edges(n, seed), directed)
                s = rng() % n
                d, p = R.serial(adj, n, s)
                sweep.append([n, int(seed), int(s), int(dense), int(directed), h(adj), h(d), h(p)])
    out["acceptance_sweep"] = sweep
    # generator goldens (generate.hpp): edge lists of small graphs
    out["generate_sparse_edges"] = {f"{n}:{s}": h(R.sparse_edges(n, s)) for n, s in [(7, 1), (10, 2), (100, 5), (1000, 42)]}
    out["generate_dense_matrix"] = {f"{n}:{s}": h(R.dense(n, s)) for n, s in [(2, 1), (10, 2), (100, 5), (1000, 42)]}
    # parse_edge_list (graph.hpp:126-174) error cases: line numbers reported by the reference
    texts = {
        "ok_crlf_comments": "# c\n4 2\r\n0 1 5\r\n\n2 3 7 \n",
        "missing_header": "# only comments\n\n",
        "bad_header": "4\n",
        "too_many_edges": "3 1\n0 1 1\n1 2 1\n",
        "too_few_edges": "3 2\n0 1 1\n",
        "self_loop": "3 1\n1 1 4\n",
        "out_of_range": "3 1\n0 3 4\n",
        "negative_weight": "3 1\n0 1 -4\n",
        "weight_range": "3 1\n0 1 4294967296\n",
        "malformed": "3 1\n0 x 4\n",
        "plus_sign": "3 1\n0 +1 4\n",
        "dup_min": "3 3\n0 1 9\n1 0 4\n0 1 6\n",
    }
    parse = {}
    for k, t in texts.items():
        for directed in (0, 1):
            r = R.parse(t, directed)
            parse[f"{k}:{directed}"] = [r[0], r[1], r[2]] if r[0] != "ok" else ["ok", r[1], h(r[2])]
    out["parse"] = {"texts": texts, "results": parse}
    # dijkstra_dataparallel (dataparallel.hpp:302-327): dist, reconstructed pred, rounds
    dp = []

    def dpcase(name, adj, n, source, keep_arrays=True, **extra):
        d, p, r = R.dataparallel(adj, n, source, 1)
        c = {"name": name, "n": n, "source": source, "rounds": r, **extra}
        if keep_arrays:
            c.update(adj=[int(x) for x in adj], dist=[int(x) for x in d], pred=[int(x) for x in p])
        else:
            c.update(dist_sha=h(d), pred_sha=h(p))
        dp.append(c)

    dpcase("four_vertex_undirected_s0", R.from_edges(4, four, False), 4, 0)       # test_dataparallel.cpp:60-66
    dpcase("single_vertex", np.zeros(1, np.uint64), 1, 0)                         # :68-73
    dpcase("zero_weight_tie_s2", R.from_edges(4, zw, False), 4, 2)                # :144-154
    zw2 = [(0, 1, 0), (1, 2, 0), (2, 0, 0), (3, 1, 0), (3, 4, 1), (4, 2, 0), (5, 3, 2), (0, 5, 2)]
    dpcase("zero_weight_cycle_s5", R.from_edges(6, zw2, True), 6, 5)              # multi-pass attach
    dpcase("config1_dense_n1000_seed42", R.dense(1000, 42), 1000, 0, keep_arrays=False, seed=42)
    out["dataparallel"] = dp
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
