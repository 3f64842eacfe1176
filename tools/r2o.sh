SSSP_BUCKET_TRACE=1 python tools/trace_rep.py 2>&1 | head -8
python tools/ab_time.py 1d,2,3 40
