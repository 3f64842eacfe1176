"""All five BASELINE.json configs on ONE B200 with parity against the
reference's serial CPU path (oracle/_ref) -- one JSON line per config.

  1  n=1000 generate_{sparse,dense}(1000,42) undirected, source 0
  2  n=16384 Bernoulli(0.5) undirected, seed 16384, source 0
  3  n=32768 generate_dense(32768,32768) undirected, source 0
  4  n=65536 Bernoulli(0.001) DIRECTED ('-w'), seed 65536, source 0 (1 GPU here; 8 in BASELINE)
  5  64 sources 256*k on the config-2 graph (batched; 8 GPUs in BASELINE)

Usage: python tools/configs_bench.py [--configs 1,2,3,4,5]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker + CPU baseline)
import paper_2504_03667_b200 as P  # noqa: E402


def timed(dg, sources, reps=5):
    dg.enqueue(sources)
    dg.finish()
    best = None
    for _ in range(reps):
        dg.enqueue(sources)
        st = dg.finish()
        best = st if best is None or st["rounds_s"] < best["rounds_s"] else best
    return best


def run(name, g, sources, R, engines=("auto", "cluster")):
    out = {"config": name, "n": g.n, "directed": g.directed, "sources": len(sources)}
    hg = R.graph(g.adj, g.n, int(g.directed))
    t = time.perf_counter()
    want = [R.graph_serial(hg, g.n, s)[:2] for s in sources[:2]]
    out["cpu_serial_ms_per_source"] = round(1e3 * (time.perf_counter() - t) / len(want), 2)
    R.graph_free(hg)
    for eng in engines:
        with P.DeviceGraph(g, engine=eng) as dg:
            st = timed(dg, sources if len(sources) > 1 else sources, reps=3 if eng != "auto" else 5)
            res = dg.solve_batch(sources[:2])
            ok = all(np.array_equal(r.dist, d) and np.array_equal(r.pred, p)
                     for r, (d, p) in zip(res, want))
            info = dg.info()
        key = {"auto": ["grid", "cluster", "bucket"][st["engine"] - 1]}.get(eng, eng)
        out[key] = {"ms_per_launch": round(st["rounds_s"] * 1e3, 4),
                    "ms_per_source": round(st["rounds_s"] * 1e3 / len(sources), 4),
                    "classes": st["classes"], "rows_read": st["rows_read"],
                    "weight_bytes": info["weight_bytes"], "parity": bool(ok)}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    a = ap.parse_args()
    R = oracle.REF()
    cfgs = set(a.configs.split(","))
    if "1" in cfgs:
        run("1-sparse", P.generate_sparse(1000, 42), [0], R)
        run("1-dense", P.generate_dense(1000, 42), [0], R)
    g2 = None
    if "2" in cfgs or "5" in cfgs:
        g2 = P.generate_bernoulli(16384, 0.5, 16384)
    if "2" in cfgs:
        run("2", g2, [0], R)
    if "3" in cfgs:
        run("3", P.generate_dense(32768, 32768), [0], R)
    if "4" in cfgs:
        run("4", P.generate_bernoulli(65536, 0.001, 65536, directed=True), [0], R,
            engines=("auto",))
    if "5" in cfgs:
        run("5", g2, [256 * k for k in range(64)], R)


if __name__ == "__main__":
    main()
