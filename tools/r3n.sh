# Session 6: config-4 phase trace with sparse tile lists; upload trace (lists, no transpose)
SSSP_UPLOAD_TRACE=1 SSSP_BUCKET_TRACE=1 timeout 300 python tools/trace_cfg4.py > gpurun_out/trace_n.txt 2>&1
SSSP_BUCKET_SPARSE=0 SSSP_UPLOAD_TRACE=1 timeout 300 python tools/trace_cfg4.py > gpurun_out/trace_n_dense.txt 2>&1
timeout 300 python tools/ab_time.py 4 20 > gpurun_out/ab_n.jsonl 2>&1
