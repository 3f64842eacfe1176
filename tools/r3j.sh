# Session 5: VIMNMX3 push with a 2-input tail (no dummy rows): timing, twice.
python tools/ab_time.py 1d,2,3,4,5 20 > gpurun_out/ab_j.jsonl 2>&1
python tools/ab_time.py 1d,2,3,4,5 20 >> gpurun_out/ab_j.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py -x -q > gpurun_out/pytest_j.log 2>&1; tail -2 gpurun_out/pytest_j.log
