# Session 6: tile-local sparse push walks the B_d bitmap (no id enumeration); A/B vs cfdda3b+split512 (build_prev); tests
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py -x -q > gpurun_out/pytest_s.log 2>&1; tail -2 gpurun_out/pytest_s.log
for rep in 1 2; do
SSSP_LIB=build_prev/libsssp_cuda.so timeout 300 python tools/ab_time.py 3,4 20 >> gpurun_out/ab_s_prev.jsonl 2>&1
timeout 300 python tools/ab_time.py 3,4 20 >> gpurun_out/ab_s_new.jsonl 2>&1
done
