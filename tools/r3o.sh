# Session 6: row-split sparse push (classes >= 2048 rows) + tile-local sparse push; tests, A/B, trace
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py -x -q > gpurun_out/pytest_o.log 2>&1; tail -3 gpurun_out/pytest_o.log
timeout 300 python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_o.jsonl 2>&1
SSSP_SPLIT_ROWS=0 timeout 300 python tools/ab_time.py 4 20 >> gpurun_out/ab_o.jsonl 2>&1
SSSP_SPLIT_ROWS=512 timeout 300 python tools/ab_time.py 4 20 >> gpurun_out/ab_o.jsonl 2>&1
SSSP_SPLIT_ROWS=8192 timeout 300 python tools/ab_time.py 4 20 >> gpurun_out/ab_o.jsonl 2>&1
SSSP_BUCKET_TRACE=1 timeout 300 python tools/trace_cfg4.py > gpurun_out/trace_o.txt 2>&1
