free -g | head -2; nproc; lscpu | grep "Model name"
timeout 1500 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo rc=$?; tail -5 gpurun_out/bench.err
tail -1 gpurun_out/bench.log > gpurun_out/bench_line.json
