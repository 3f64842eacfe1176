"""Per-phase %globaltimer trace of the bucket kernel (CTA 0), for profiling:
SSSP_BUCKET_TRACE=1 python tools/trace_bucket.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03667_b200 as P
g = P.generate_dense(32768, 32768)
dg = P.DeviceGraph(g, engine="bucket")
for i in range(3):
    r = dg.solve(0)
    print(r.stats['rounds_s']*1e3, r.stats['classes'], r.stats['rows_read'], flush=True)
g2 = P.generate_bernoulli(16384, 0.5, 16384)
dg2 = P.DeviceGraph(g2, engine="bucket")
for i in range(2):
    r = dg2.solve(0)
    print(r.stats['rounds_s']*1e3, r.stats['classes'], r.stats['rows_read'], flush=True)
g3 = P.generate_sparse(16384, 3)
dg3 = P.DeviceGraph(g3, engine="bucket")
r = dg3.solve(0); print('sparse', r.stats['rounds_s']*1e3, r.stats['classes'], r.stats['rows_read'], flush=True)
