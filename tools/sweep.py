"""Dev sweep: solve time and t_sync per round across launch shapes (one GPU).
Usage: python tools/sweep.py --n 32768 [--ctas 32,64,128] [--replicas 1,4,8,16]"""
import argparse, itertools, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2504_03667_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--seed", type=int, default=32768)
ap.add_argument("--graph", default="dense")
ap.add_argument("--ctas", default="0")
ap.add_argument("--replicas", default="0")
ap.add_argument("--flags", default="3")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--engine", default="cluster")
ap.add_argument("--warps", default="8")
a = ap.parse_args()
t = time.time()
g = P.generate_dense(a.n, a.seed) if a.graph == "dense" else P.generate_bernoulli(a.n, 0.5, a.seed)
print(f"# built n={a.n} in {time.time()-t:.1f}s", flush=True)
ref = None
for engine in a.engine.split(","):
  for ctas, rep, flags, warps in itertools.product(*[[int(x) for x in s.split(",")] for s in (a.ctas, a.replicas, a.flags, a.warps)]):
    try:
        dg = P.DeviceGraph(g, flags=flags, ctas=ctas, replicas=rep, engine=engine, warps=warps)
    except Exception as e:
        print(json.dumps({"engine": engine, "ctas": ctas, "warps": warps, "error": str(e)}), flush=True)
        continue
    info = dg.info()
    ts = dg.probe_sync(20000)
    times = []
    for _ in range(a.reps + 1):
        r = dg.solve(0)
        times.append(r.stats["rounds_s"])
    if ref is None:
        ref = r
    ok = (r == ref)
    print(json.dumps({"engine": engine, "ctas": info["ctas"], "warps": warps, "rep": rep, "flags": flags, "ms": round(1e3 * min(times[1:]), 3),
                      "us_per_round": round(1e6 * min(times[1:]) / r.stats["iterations"], 3),
                      "t_sync_us": round(ts * 1e6, 3), "mis": r.stats["mispredicts"], "same": ok}), flush=True)
    dg.close()
