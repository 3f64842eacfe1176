"""Bucket-engine solve time per config with the L2 flushed before every solve
(per-solve CUDA events on the library's stream; a 256 MiB write between
solves evicts the 126 MB L2), plus parity vs the reference serial solve.

  python tools/bucket_time.py [--configs 1s,1d,2,3,4] [--reps 20] [--trace]
SSSP_BUCKET_TRACE=1 prints the per-barrier %globaltimer trace of CTA 0."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2504_03667_b200 as P  # noqa: E402


def graphs(which):
    if "1s" in which:
        yield "1-sparse", P.generate_sparse(1000, 42)
    if "1d" in which:
        yield "1-dense", P.generate_dense(1000, 42)
    if "2" in which:
        yield "2", P.generate_bernoulli(16384, 0.5, 16384)
    if "3" in which:
        yield "3", P.generate_dense(32768, 32768)
    if "4" in which:
        yield "4", P.generate_bernoulli(65536, 0.001, 65536, directed=True)


def time_solves(dg, sources, reps, flush):
    stream = torch.cuda.ExternalStream(dg.stream_ptr())
    ts = []
    for i in range(reps + 3):
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xFF)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        dg.enqueue([sources[i % len(sources)]])
        e1.record(stream)
        st = dg.finish()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    return np.array(ts), st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1s,1d,2,3")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--engine", default="bucket")
    a = ap.parse_args()
    R = oracle.REF()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name, g in graphs(a.configs.split(",")):
        hg = R.graph(g.adj, g.n, int(g.directed))
        d, p = R.graph_serial(hg, g.n, 0)[:2]
        R.graph_free(hg)
        with P.DeviceGraph(g, engine=a.engine) as dg:
            r = dg.solve(0)
            ok = bool(np.array_equal(r.dist, d) and np.array_equal(r.pred, p))
            ts, st = time_solves(dg, [0], a.reps, flush)
            info = dg.info()
        rows = st["rows_read"]
        nb = st["bytes_read"]
        print(json.dumps({"config": name, "n": g.n, "parity": ok, "engine": st["engine"],
                          "ms_mean": round(float(ts.mean()), 4), "ms_min": round(float(ts.min()), 4),
                          "ms_p50": round(float(np.median(ts)), 4),
                          "lib_kernel_ms": round(st["rounds_s"] * 1e3, 4),
                          "classes": st["classes"], "rows_read": rows, "bytes": nb,
                          "gbs_at_mean": round(nb / (ts.mean() * 1e-3) / 1e9, 1)}), flush=True)
        del g


if __name__ == "__main__":
    main()
