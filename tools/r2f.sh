nvidia-smi --query-gpu=clocks.sm,clocks.mem --format=csv,noheader
SSSP_BUCKET_TRACE=1 python tools/trace_bucket.py 2>&1 | head -6
python tools/bucket_time.py --configs 1d,2,3 --reps 30
