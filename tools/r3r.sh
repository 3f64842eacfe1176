# Session 6 final validation at the split-512 default: full GPU suite, smoke, bench, bench launch list
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r.log 2>&1; tail -2 gpurun_out/pytest_r.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r.txt 2>&1; echo rc=$? >> gpurun_out/smoke_r.txt
timeout 600 python bench.py > gpurun_out/bench_r.jsonl 2> gpurun_out/bench_r.err; echo rc=$? >> gpurun_out/bench_r.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_r.log 2>&1
