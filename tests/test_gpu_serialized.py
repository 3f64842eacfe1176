"""Shards on one GPU must not depend on CUDA co-scheduling two kernels.

Round-1 regression: P logical shards on one device ran as P separate
launches that spin on each other's barrier, so anything that serialises
kernels (ncu replay, CUDA_LAUNCH_BLOCKING=1, compute-sanitizer, MPS) hung
until the 60 s watchdog.  Now every device's shards are one cooperative
launch.  These tests run the partitioned solve (partitioned.hpp:184-225, the
multi-shard path) in a child process with CUDA_LAUNCH_BLOCKING=1 and a short
watchdog, for every engine and P = 2/4/8, and bench.py --gpus 2 (ranks
self-launched) with both ranks on the one GPU."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import oracle, paper_2504_03667_b200 as P
ok = []
for n, seed in [(1000, 3), (2048, 4)]:
    g = P.generate_sparse(n, seed) if seed % 2 else P.generate_dense(n, seed)
    d, p = oracle.C().serial(g.adj, g.n, 5)
    for engine in ("bucket", "cluster", "grid"):
        if engine == "bucket" and seed % 2:
            continue
        for shards in (2, 4, 8):
            with P.DeviceGraph(g, [0] * shards, engine=engine, timeout_ms=20000) as dg:
                r = dg.solve(5)
                r2 = dg.solve_batch([5, 0])
            same = (np.array_equal(r.dist, d) and np.array_equal(r.pred, p)
                    and r2[0] == r)
            ok.append((engine, shards, n, bool(same)))
print("RESULT", ok)
"""


def test_logical_shards_with_launch_blocking(gpu):
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
    p = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")][0]
    res = eval(line[len("RESULT "):])
    assert res and all(r[3] for r in res), res


def test_smoke_with_launch_blocking(gpu):
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
    p = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], env=env,
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    assert "smoke ok" in p.stdout


def test_bench_self_launches_ranks(gpu):
    """`bench.py --gpus 2` without torchrun starts its 2 ranks itself and
    reports n_gpus 2 (both ranks on GPU 0 over gloo: SSSP_BENCH_ONE_GPU)."""
    env = dict(os.environ, SSSP_BENCH_ONE_GPU="1")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--vertices", "256", "--no-cpu-baseline", "--no-batch", "--e2e-steps", "1",
                        "--no-configs"],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
