python -m pytest tests/test_gpu_bucket.py -x -q > gpurun_out/pytest_bucket.log 2>&1; tail -2 gpurun_out/pytest_bucket.log
for v in "SSSP_PUSH_DEPTH16=0 SSSP_OWNER_PULL_BYTES=0" "SSSP_OWNER_PULL_BYTES=0" "SSSP_OWNER_PULL_BYTES=32768" "SSSP_OWNER_PULL_BYTES=65536" "SSSP_OWNER_PULL_BYTES=131072" "SSSP_PUSH_BULK=1"; do
echo "== $v"; env $v python tools/bucket_time.py --configs 1d,2,3 --reps 30
done
SSSP_BUCKET_TRACE=1 python tools/trace_bucket.py 2>&1 | head -8
