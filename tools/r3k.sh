# Session 5: full validation at HEAD (smoke, pytest -m gpu, bench) + ncu capture of the config-4 bucket solve.
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_k.log 2>&1; tail -1 gpurun_out/smoke_k.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_k.log 2>&1; tail -2 gpurun_out/pytest_k.log
timeout 500 python bench.py > gpurun_out/bench_k.jsonl 2> gpurun_out/bench_k.err; tail -c 300 gpurun_out/bench_k.jsonl
ncu --set full --clock-control none --import-source on -k regex:bucket_kernel -s 1 -c 1 -o gpurun_out/prof_bucket_cfg4 python tools/prof_cfg4.py > gpurun_out/ncu_k.log 2>&1; tail -1 gpurun_out/ncu_k.log
