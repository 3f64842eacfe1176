python -m pytest tests/test_gpu_bucket.py tests/test_gpu_parity.py tests/test_gpu_serialized.py -x -q > gpurun_out/pytest_bucket.log 2>&1; tail -3 gpurun_out/pytest_bucket.log
python tools/bucket_time.py --configs 1s,1d,2,3 > gpurun_out/bucket_time.jsonl 2>&1; cat gpurun_out/bucket_time.jsonl
SSSP_BUCKET_TRACE=1 python tools/trace_bucket.py > gpurun_out/trace.txt 2>&1; head -60 gpurun_out/trace.txt
