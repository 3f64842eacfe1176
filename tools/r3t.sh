# Session 6 closing check at HEAD: full GPU suite + smoke
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_t.log 2>&1; tail -2 gpurun_out/pytest_t.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_t.txt 2>&1; echo rc=$? >> gpurun_out/smoke_t.txt
