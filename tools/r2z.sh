# PDL launch microbenchmark; kernel-level A/B of the bulk-copy (TMA engine) push; bucket tests.
./tools/ubench_launch2 > gpurun_out/ubench_launch3.jsonl 2>&1; head -8 gpurun_out/ubench_launch3.jsonl
SSSP_LIB=build_ab/libsssp_cuda.so python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_push_ldg.jsonl 2>&1; cat gpurun_out/ab_push_ldg.jsonl
SSSP_LIB=build_ab/libsssp_cuda.so SSSP_PUSH_BULK=1 python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_push_bulk.jsonl 2>&1; cat gpurun_out/ab_push_bulk.jsonl
python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_default.jsonl 2>&1; cat gpurun_out/ab_default.jsonl
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_z.log 2>&1; tail -2 gpurun_out/pytest_z.log
