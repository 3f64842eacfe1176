# Round-2 re-entry validation at HEAD: GPU tests, smoke, bench, launch list, bucket ncu capture.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_x.log 2>&1; tail -2 gpurun_out/pytest_x.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_x.log 2>&1; tail -1 gpurun_out/smoke_x.log
python bench.py > gpurun_out/bench_x.log 2>&1; tail -1 gpurun_out/bench_x.log | cut -c1-400
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_x.csv python bench.py --steps 2 --warmup 3 > gpurun_out/bench_ncu_x.log 2>&1; tail -1 gpurun_out/bench_ncu_x.log | cut -c1-200
ncu --set full --clock-control none --import-source on -k regex:bucket_kernel -s 1 -c 1 -o gpurun_out/prof_bucket_r02x python tools/prof_one.py 32768 bucket > gpurun_out/ncu_x.log 2>&1; tail -1 gpurun_out/ncu_x.log
