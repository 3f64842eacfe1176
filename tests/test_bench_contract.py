"""bench.py's reference arm on CPU: the JSON line the driver reads (keys,
types, reference-arm e2e with zero copies) at a small n, and the N>1 rule that
only rank 0 runs it."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra, *args):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, "bench.py", "--impl", "reference", *args], cwd=ROOT,
                          env=env, capture_output=True, text=True, timeout=300)


def test_reference_arm_line(ref):
    p = _run({}, "--vertices", "384", "--steps", "2", "--warmup", "3")
    assert p.returncode == 0, p.stderr
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "ms" and d["higher_is_better"] is False
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "ms", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["n"] == 384


def test_reference_arm_nonzero_rank_is_silent(ref):
    p = _run({"RANK": "1", "WORLD_SIZE": "2"}, "--vertices", "384", "--steps", "1")
    assert p.returncode == 0, p.stderr
    assert p.stdout.strip() == ""


def test_our_arm_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a CUDA device")
    env = dict(os.environ)
    p = subprocess.run([sys.executable, "bench.py", "--steps", "1"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode != 0
    assert "needs a CUDA device" in p.stderr
