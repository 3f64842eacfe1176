# Session 6: sparse lists as their own kernel instance (dense instances = e012c37 SASS);
# full GPU suite, A/B vs e012c37, bench, config-4 ncu of the sparse instance
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; tail -3 gpurun_out/pytest_q.log
SSSP_LIB=build_old/libsssp_cuda.so timeout 300 python tools/ab_time.py 1d,2,3,4 20 >> gpurun_out/ab_q_old.jsonl 2>&1
timeout 300 python tools/ab_time.py 1d,2,3,4 20 >> gpurun_out/ab_q_new.jsonl 2>&1
SSSP_SPLIT_ROWS=512 timeout 300 python tools/ab_time.py 4 20 >> gpurun_out/ab_q_new.jsonl 2>&1
SSSP_SPLIT_ROWS=1024 timeout 300 python tools/ab_time.py 4 20 >> gpurun_out/ab_q_new.jsonl 2>&1
timeout 600 python bench.py > gpurun_out/bench_q.jsonl 2> gpurun_out/bench_q.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bucket_kernel -s 1 -c 1 -o gpurun_out/ncu_cfg4_sparse -f python tools/prof_cfg4.py > gpurun_out/ncu_q.log 2>&1
ncu -i gpurun_out/ncu_cfg4_sparse.ncu-rep --page raw --csv > gpurun_out/ncu_cfg4_sparse_raw.csv 2>/dev/null
