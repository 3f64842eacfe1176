"""The paper's data-parallel engine (sssp_solve_dataparallel) on BASELINE
configs 1-3: device ms (CUDA events), rounds, rows streamed, achieved HBM
GB/s, parity with the oracle restatement, and the reference's own
dijkstra_dataparallel (oracle/_ref, threaded lanes) timed on the host.
Usage: python tools/dp_bench.py [--configs 1,2,3] [--ref]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker + CPU baseline)
import paper_2504_03667_b200 as P  # noqa: E402


def run(name, g, ref, reps=5):
    out = {"config": name, "n": g.n, "engine": "dataparallel"}
    with P.DeviceGraph(g) as dg:
        r = dg.solve_dataparallel(0)
        best = None
        for _ in range(reps):
            x = dg.solve_dataparallel(0)
            best = x if best is None or x.stats["rounds_s"] < best.stats["rounds_s"] else best
        wb = dg.info()["weight_bytes"]
    st = best.stats
    rs = P.pad_vertex_count(g.n, 1)
    out.update(ms=round(st["rounds_s"] * 1e3, 4), rounds=st["rounds"], rows_read=st["rows_read"],
               pass_sweeps=st["classes"], weight_bytes=wb)
    out["achieved_gbs"] = round(st["rows_read"] * g.n * wb / st["rounds_s"] / 1e9, 1)
    t = time.perf_counter()
    d, p, rounds = oracle.C().dataparallel(g.adj, g.n, 0)
    out["oracle_s"] = round(time.perf_counter() - t, 2)
    out["parity"] = bool(np.array_equal(r.dist, d) and np.array_equal(r.pred, p)
                         and r.stats["rounds"] == rounds)
    if ref is not None:
        t = time.perf_counter()
        ref.dataparallel(g.adj, g.n, 0, 0)
        out["reference_dataparallel_threaded_s"] = round(time.perf_counter() - t, 3)
        out["host_threads"] = os.cpu_count()
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--ref", action="store_true")
    a = ap.parse_args()
    ref = oracle.REF() if a.ref else None
    c = set(a.configs.split(","))
    if "1" in c:
        run("1-sparse", P.generate_sparse(1000, 42), ref)
        run("1-dense", P.generate_dense(1000, 42), ref)
    if "2" in c:
        run("2", P.generate_bernoulli(16384, 0.5, 16384), ref)
    if "3" in c:
        run("3", P.generate_dense(32768, 32768), ref)


if __name__ == "__main__":
    main()
