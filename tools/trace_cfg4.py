"""Phase trace of the bucket kernel on BASELINE config 4 (n=65536 Bernoulli
0.1 % directed, seed 65536): SSSP_BUCKET_TRACE=1 python tools/trace_cfg4.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03667_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
g = P.generate_bernoulli(n, 0.001, n, directed=True)
with P.DeviceGraph(g, engine="bucket") as dg:
    for _ in range(3):
        r = dg.solve(0)
        st = r.stats
        print("ms %.3f classes %d rows %d" % (st["rounds_s"] * 1e3, st["classes"], st["rows_read"]), flush=True)
