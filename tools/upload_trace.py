"""Dev: graph-create (upload) breakdown.  SSSP_UPLOAD_TRACE=1 python tools/upload_trace.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2504_03667_b200 as P
g = P.generate_dense(32768, 32768)
for i in range(5):
    t = time.perf_counter()
    dg = P.DeviceGraph(g)
    t1 = time.perf_counter()
    r = dg.solve(0)
    t2 = time.perf_counter()
    dg.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t):.1f} ms  solve {1e3*(t2-t1):.2f} ms  close {1e3*(t3-t2):.1f} ms", flush=True)
t = time.perf_counter(); s = int(g.adj.sum(dtype=np.uint64)); print(f"numpy 1-thread read of 8 GiB: {1e3*(time.perf_counter()-t):.0f} ms")
