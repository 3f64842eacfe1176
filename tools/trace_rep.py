"""Bucket-kernel phase traces (CTA 0, %globaltimer) for config 3: source 0 warm,
then rotating sources; with SSSP_BUCKET_REPS=k the launch runs the solve k
times (warm-code timing of the later repeats).
SSSP_BUCKET_TRACE=1 [SSSP_BUCKET_REPS=2] python tools/trace_rep.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03667_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
g = P.generate_dense(n, 32768) if n != 16384 else P.generate_bernoulli(16384, 0.5, 16384)
dg = P.DeviceGraph(g, engine="bucket")
for i in range(3):
    r = dg.solve(0)
    print("src 0", round(r.stats['rounds_s'] * 1e3, 4), r.stats['classes'], r.stats['rows_read'], flush=True)
for s in (7919, 15838, 23757):
    r = dg.solve(s % n)
    print("src", s % n, round(r.stats['rounds_s'] * 1e3, 4), r.stats['classes'], r.stats['rows_read'], flush=True)
