python -m pytest tests/test_gpu_configs.py -x -q > gpurun_out/pytest_cfg.log 2>&1; tail -5 gpurun_out/pytest_cfg.log
ncu --set full --clock-control none --import-source on -k regex:bucket_kernel -s 1 -c 1 -o gpurun_out/prof_bucket_r02b python tools/prof_one.py 32768 bucket > gpurun_out/ncu_b.log 2>&1; tail -2 gpurun_out/ncu_b.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python tools/prof_one.py 32768 bucket > /dev/null 2>&1; echo launches rc=$?
