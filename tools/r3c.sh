# Session 5: PDL A/B on back-to-back bucket solves; the clock sampler's effect; bucket parity tests.
python tools/hostq.py 20 > gpurun_out/pdl_on.txt 2>&1
SSSP_BUCKET_PDL=0 python tools/hostq.py 20 > gpurun_out/pdl_off.txt 2>&1
HOSTQ_SAMPLER=1 python tools/hostq.py 20 > gpurun_out/pdl_on_sampler.txt 2>&1
SSSP_BUCKET_SPANS=1 python tools/hostq.py 60 > gpurun_out/spans_pdl.txt 2>&1
python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_pdl_on.jsonl 2>&1
SSSP_BUCKET_PDL=0 python tools/ab_time.py 1d,2,3,4 20 > gpurun_out/ab_pdl_off.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_configs.py tests/test_gpu_serialized.py tests/test_gpu_multiproc.py -x -q > gpurun_out/pytest_c.log 2>&1; tail -2 gpurun_out/pytest_c.log
timeout 400 python bench.py > gpurun_out/bench_pdl.jsonl 2> gpurun_out/bench_pdl.err
