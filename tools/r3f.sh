# Session 5: class-1 id list prefetched at kernel start (cp.async) + push row groups folded by
# warp shuffles: timing vs r3e's default, phase trace, bucket/config parity tests.
python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_f_default.jsonl 2>&1
SSSP_BUCKET_TRACE=1 python tools/trace_rep.py > gpurun_out/trace_f.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_f.log 2>&1; tail -2 gpurun_out/pytest_f.log
