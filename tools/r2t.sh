timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py -x -q > gpurun_out/pytest_t.log 2>&1; tail -2 gpurun_out/pytest_t.log
SSSP_BUCKET_TRACE=1 python tools/trace_rep.py 2>&1 | sed -n 3,4p
python tools/ab_time.py 1d,2,3,5 40
