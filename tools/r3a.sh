# Session 5: phase trace of the bucket kernel at HEAD (config 3 and config 2), spans.
SSSP_BUCKET_TRACE=1 python tools/trace_rep.py > gpurun_out/trace_r3a.txt 2>&1
SSSP_BUCKET_TRACE=1 python tools/trace_rep.py 16384 > gpurun_out/trace_r3a_16k.txt 2>&1
SSSP_BUCKET_SPANS=1 python tools/trace_rep.py > gpurun_out/spans_r3a.txt 2>&1
