# Session 5: ncu capture of the bucket kernel at HEAD (config 3), launch list of the bench command,
# config-4 phase trace.
ncu --set full --clock-control none --import-source on -k regex:bucket_kernel -s 1 -c 1 -o gpurun_out/prof_bucket_r02s5 python tools/prof_one.py 32768 bucket > gpurun_out/ncu_g.log 2>&1; tail -1 gpurun_out/ncu_g.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_g.csv python bench.py --steps 2 --warmup 3 > gpurun_out/bench_ncu_g.log 2>&1; tail -1 gpurun_out/bench_ncu_g.log | cut -c1-200
SSSP_BUCKET_TRACE=1 python tools/trace_cfg4.py > gpurun_out/trace_cfg4_g.txt 2>&1
