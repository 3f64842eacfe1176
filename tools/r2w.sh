timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_w.log 2>&1; tail -2 gpurun_out/pytest_w.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python tools/ab_time.py 1d,1s,2,3,4,5 30
