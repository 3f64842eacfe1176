# Session-3 baseline at HEAD: GPU tests, smoke (plain, serialized, under ncu), bench, bucket trace.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_full.log 2>&1; tail -3 gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_blocking.log 2>&1; echo blocking rc=$?; tail -2 gpurun_out/smoke_blocking.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo ncu-smoke rc=$?; tail -2 gpurun_out/smoke_ncu.log
SSSP_BUCKET_TRACE=1 python tools/trace_bucket.py > gpurun_out/trace.txt 2>&1; head -8 gpurun_out/trace.txt
timeout 1500 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-400
