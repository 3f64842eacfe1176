python -m pytest tests/test_gpu_bucket.py -x -q > gpurun_out/pytest_bucket.log 2>&1; tail -2 gpurun_out/pytest_bucket.log
SSSP_BUCKET_TRACE=1 python tools/trace_bucket.py 2>&1 | head -6
python tools/bucket_time.py --configs 1d,2,3 --reps 30
SSSP_OWNER_PULL_COLS=0 python tools/bucket_time.py --configs 2,3 --reps 30
