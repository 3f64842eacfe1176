# Session 5: software-pipelined push (two alternating half batches of 4 rows) vs the previous
# 8-deep batches (build_old = f079202's library), configs 1d/2/3/4/5; parity tests.
SSSP_LIB=build_old/libsssp_cuda.so python tools/ab_time.py 1d,2,3,4,5 20 > gpurun_out/ab_l_old.jsonl 2>&1
python tools/ab_time.py 1d,2,3,4,5 20 > gpurun_out/ab_l_new.jsonl 2>&1
SSSP_LIB=build_old/libsssp_cuda.so python tools/ab_time.py 1d,2,3,4,5 20 >> gpurun_out/ab_l_old.jsonl 2>&1
python tools/ab_time.py 1d,2,3,4,5 20 >> gpurun_out/ab_l_new.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_l.log 2>&1; tail -2 gpurun_out/pytest_l.log
