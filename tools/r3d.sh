# Session 5: why bench.py's back-to-back solve is slower than tools/ab_time.py's (spans, host enqueue).
SSSP_BENCH_DEBUG=1 SSSP_BUCKET_SPANS=1 timeout 300 python bench.py --no-configs --no-batch --no-cpu-baseline --no-host-driven > gpurun_out/bench_dbg.jsonl 2> gpurun_out/bench_dbg.err
SSSP_BUCKET_TILE_BYTES=64 python tools/ab_time.py 1d,2 20 > gpurun_out/ab_tile64.jsonl 2>&1
SSSP_BUCKET_TILE_BYTES=32 python tools/ab_time.py 1d,2 20 > gpurun_out/ab_tile32.jsonl 2>&1
SSSP_BUCKET_TILE_BYTES=64 SSSP_BUCKET_TRACE=1 python tools/trace_rep.py 16384 > gpurun_out/trace_tile64_16k.txt 2>&1
