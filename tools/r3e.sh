# Session 5: kernel-level A/B of the TMA bulk-copy push (UBLKCP + mbarrier) and the 16-deep
# register push against the default LDG push (build_ab, -DSSSP_BUCKET_AB=1); tile 256 B at
# config 3; bench with the pre-queued timed loop.
SSSP_LIB=build_ab/libsssp_cuda.so python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_e_ldg.jsonl 2>&1
SSSP_LIB=build_ab/libsssp_cuda.so SSSP_PUSH_BULK=1 python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_e_bulk.jsonl 2>&1
SSSP_LIB=build_ab/libsssp_cuda.so SSSP_PUSH_DEPTH16=1 python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_e_d16.jsonl 2>&1
python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_e_default.jsonl 2>&1
SSSP_BUCKET_TILE_BYTES=256 python tools/ab_time.py 3 20 > gpurun_out/ab_e_tile256.jsonl 2>&1
timeout 400 python bench.py > gpurun_out/bench_e.jsonl 2> gpurun_out/bench_e.err
