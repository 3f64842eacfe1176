# Session 5: u8 push rows paired through VIMNMX3: timing (configs 1d/2/3/4 + batch 5) and parity tests.
python tools/ab_time.py 1d,2,3,4,5 20 > gpurun_out/ab_i.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_i.log 2>&1; tail -2 gpurun_out/pytest_i.log
