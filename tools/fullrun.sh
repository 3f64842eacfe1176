set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_full.log 2>&1; tail -3 gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bucket -s 3 -c 1 -o gpurun_out/prof_bucket_r01b python tools/prof_one.py 32768 bucket 0 3 > gpurun_out/ncu_bucket.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:dp_ -s 2 -c 2 -o gpurun_out/prof_dp_r01b python tools/prof_dp.py > gpurun_out/ncu_dp.log 2>&1
python tools/configs_bench.py > gpurun_out/configs.log 2>&1
ls -la gpurun_out
