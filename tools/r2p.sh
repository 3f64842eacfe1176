timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_p.log 2>&1; tail -3 gpurun_out/pytest_p.log
SSSP_BUCKET_TRACE=1 python tools/trace_rep.py 2>&1 | head -8
python tools/ab_time.py 1d,1s,2,3,5 40
SSSP_BUCKET_LOCAL1=0 python tools/ab_time.py 1d,2,3,5 40
