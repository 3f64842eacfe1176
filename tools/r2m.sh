timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py tests/test_gpu_serialized.py -x -q > gpurun_out/pytest_m.log 2>&1; tail -3 gpurun_out/pytest_m.log
SSSP_BUCKET_TRACE=1 python tools/trace_rep.py 2>&1 | head -8
SSSP_BUCKET_TRACE=1 python tools/trace_rep.py 16384 2>&1 | head -4
python tools/bucket_time.py --configs 1d,2,3 --reps 30
SSSP_BUCKET_TAGX=0 python tools/bucket_time.py --configs 1d,2,3 --reps 30
