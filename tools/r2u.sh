timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_u.log 2>&1; tail -2 gpurun_out/pytest_u.log
SSSP_BUCKET_TRACE=1 python tools/trace_rep.py 2>&1 | sed -n 3,4p
python tools/ab_time.py 1d,2,3,4,5 40
SSSP_BUCKET_LISTS=0 python tools/ab_time.py 3 40
