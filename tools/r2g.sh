python -m pytest tests/test_gpu_parity.py -x -q -k "kmax or beyond_32 or wide or counters or visit_order or four or cpp_dropin" > gpurun_out/pytest_wide.log 2>&1; tail -30 gpurun_out/pytest_wide.log
./oracle/_ref/test_dropin | tail -5
