# Session 6: sparse tile lists (config 4 push reads each class row's finite
# entries per tile instead of the dense 128 B slice) vs the dense push
# (SSSP_BUCKET_SPARSE=0), configs 1s/1d/2/4; parity tests first.
timeout 600 python -m pytest tests/test_gpu_bucket.py -x -q > gpurun_out/pytest_m.log 2>&1; tail -3 gpurun_out/pytest_m.log
SSSP_BUCKET_SPARSE=0 timeout 300 python tools/ab_time.py 1s,1d,2,4 20 > gpurun_out/ab_m_dense.jsonl 2>&1
timeout 300 python tools/ab_time.py 1s,1d,2,4 20 > gpurun_out/ab_m_sparse.jsonl 2>&1
SSSP_UPLOAD_TRACE=1 timeout 300 python tools/ab_time.py 4 5 > gpurun_out/ab_m_upload.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_m2.log 2>&1; tail -3 gpurun_out/pytest_m2.log
