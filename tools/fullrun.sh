# Round-end style validation on one B200: GPU tests, smoke, bench (both arms),
# all-config parity bench, data-parallel bench, two-rank bench on one GPU.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_full.log 2>&1; tail -3 gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
SSSP_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --vertices 4096 > gpurun_out/bench_2rank.log 2>&1; tail -2 gpurun_out/bench_2rank.log | cut -c1-400
python tools/configs_bench.py > gpurun_out/configs.log 2>&1
python tools/dp_bench.py --ref > gpurun_out/dp_bench.jsonl 2>&1
ls -la gpurun_out
