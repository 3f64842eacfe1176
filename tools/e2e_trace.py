"""Dev: where the e2e time of dijkstra(G, s) goes (SSSP_UPLOAD_TRACE=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03667_b200 as P
g = P.generate_dense(32768, 32768)
for i in range(4):
    t0 = time.perf_counter()
    dg = P.DeviceGraph(g)
    t1 = time.perf_counter()
    r = dg.solve(0)
    t2 = time.perf_counter()
    dg.close()
    t3 = time.perf_counter()
    r2 = P.dijkstra(g, 0)
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f}  solve {1e3*(t2-t1):.2f}  close {1e3*(t3-t2):.1f}  dijkstra() {1e3*(t4-t3):.1f} ms", flush=True)
