# Session 5: config-4 phase trace with 512 stamps (all 39 classes).
SSSP_BUCKET_TRACE=1 python tools/trace_cfg4.py > gpurun_out/trace_cfg4_h.txt 2>&1
