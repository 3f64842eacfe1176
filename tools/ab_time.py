"""Back-to-back solve time (rotating sources, CUDA events on the library
stream) for A/B switches given by environment variables:
  SSSP_BUCKET_POLL=1 python tools/ab_time.py [configs: 1d,2,3,4] [steps]"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2504_03667_b200 as P

which = sys.argv[1] if len(sys.argv) > 1 else "2,3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
tag = {k: v for k, v in os.environ.items() if k.startswith("SSSP_") and k != "SSSP_BUCKET_TRACE"}
G = {"1d": lambda: P.generate_dense(1000, 42), "1s": lambda: P.generate_sparse(1000, 42),
     "2": lambda: P.generate_bernoulli(16384, 0.5, 16384), "3": lambda: P.generate_dense(32768, 32768),
     "4": lambda: P.generate_bernoulli(65536, 0.001, 65536, directed=True)}
def batch5():
    g = P.generate_bernoulli(16384, 0.5, 16384)
    srcs = [256 * k for k in range(64)]
    with P.DeviceGraph(g) as dg:
        stream = torch.cuda.ExternalStream(dg.stream_ptr())
        for _ in range(2):
            dg.enqueue(srcs); dg.finish()
        res = []
        for rep in range(3):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dg.enqueue(srcs)
            e1.record(stream)
            dg.finish()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1))
        bad = sum(int(dg.validate(r) != 0) for r in dg.solve_batch(srcs))
    print(json.dumps({"config": "5", "env": tag, "ms_64": round(min(res), 4), "invalid": bad}), flush=True)


for c in which.split(","):
    if c == "5":
        batch5()
        continue
    g = G[c]()
    dg = P.DeviceGraph(g)
    srcs = [(7919 * i) % g.n for i in range(steps)]
    stream = torch.cuda.ExternalStream(dg.stream_ptr())
    for s in srcs[:5]:
        dg.enqueue([s]); dg.finish()
    res, host = [], []
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        for s in srcs:
            dg.enqueue([s])
        h1 = time.perf_counter()
        e1.record(stream)
        st = dg.finish()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / steps)
        host.append((h1 - h0) * 1e3 / steps)
    bad = sum(dg.validate(dg.solve(s)) != 0 for s in srcs[:8])
    print(json.dumps({"config": c, "env": tag, "ms": round(min(res), 5), "ms_all": [round(x, 5) for x in res], "host_ms_per_enqueue": round(min(host), 5),
                      "engine": st["engine"], "classes": st["classes"], "barriers": st["barriers"],
                      "invalid": int(bad)}), flush=True)
    dg.close() if hasattr(dg, "close") else None
