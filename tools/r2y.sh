# Vectorised upload kernels (row summary / list, symmetric check): parity, kernel times, e2e.
timeout 1200 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_y.log 2>&1; tail -2 gpurun_out/pytest_y.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:'row_|symmetric|transpose' --csv --log-file gpurun_out/upload_y.csv python tools/prof_one.py 32768 bucket > /dev/null 2>&1
python tools/ab_time.py 2,3,4 20 2>&1 | tail -3
SSSP_BUCKET_TRACE=1 python tools/trace_rep.py 2>&1 | head -12
python bench.py > gpurun_out/bench_y.log 2>&1; tail -1 gpurun_out/bench_y.log | cut -c1-200
SSSP_UPLOAD_TRACE=1 python tools/upload_trace.py 2>&1 | tail -8
