# Session 5: host-bound check of the back-to-back loop; PDL launch microbenchmark; launch spans.
python tools/hostq.py 20 > gpurun_out/hostq.txt 2>&1
python tools/hostq.py 200 >> gpurun_out/hostq.txt 2>&1
./tools/ubench_launch2 > gpurun_out/ubench_launch3.jsonl 2>&1
SSSP_BUCKET_SPANS=1 python tools/hostq.py 60 > gpurun_out/spans_hostq.txt 2>&1
