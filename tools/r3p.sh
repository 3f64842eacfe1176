# Session 6: bitmap-walk row-split push; A/B vs e012c37 (build_old) on configs 1d/2/3/4/5, interleaved; tests
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py -x -q > gpurun_out/pytest_p.log 2>&1; tail -3 gpurun_out/pytest_p.log
for rep in 1 2; do
SSSP_LIB=build_old/libsssp_cuda.so timeout 300 python tools/ab_time.py 1d,2,3,4,5 20 >> gpurun_out/ab_p_old.jsonl 2>&1
timeout 300 python tools/ab_time.py 1d,2,3,4,5 20 >> gpurun_out/ab_p_new.jsonl 2>&1
done
SSSP_SPLIT_ROWS=512 timeout 300 python tools/ab_time.py 4 20 >> gpurun_out/ab_p_new.jsonl 2>&1
SSSP_SPLIT_ROWS=256 timeout 300 python tools/ab_time.py 4 20 >> gpurun_out/ab_p_new.jsonl 2>&1
SSSP_BUCKET_TRACE=1 timeout 300 python tools/trace_cfg4.py > gpurun_out/trace_p.txt 2>&1
