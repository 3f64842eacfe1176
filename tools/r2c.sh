python -m pytest tests/test_gpu_bucket.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_bucket.log 2>&1; tail -3 gpurun_out/pytest_bucket.log
echo "== default"; python tools/bucket_time.py --configs 1s,1d,2,3
echo "== push_ldg"; SSSP_PUSH_LDG=1 python tools/bucket_time.py --configs 1d,2,3
echo "== owner off"; SSSP_OWNER_PULL_BYTES=0 python tools/bucket_time.py --configs 1d,2,3
SSSP_BUCKET_TRACE=1 python tools/trace_bucket.py 2>&1 | head -12
