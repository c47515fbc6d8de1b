"""bench.py contract on the GPU: one short run of each arm prints one JSON line
with the keys the driver reads (value, e2e, roofline, clocks, gpu_launches).
Guards the bench against C-ABI signature drift (it calls a few entry points
directly)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    env = dict(os.environ)
    env.setdefault("MASTER_ADDR", "127.0.0.1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_line():
    j = _run("--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-model-cpu")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "e2e", "roofline",
                "clocks", "gpu_launches"):
        assert key in j, key
    assert j["n_gpus"] == 1 and j["steps"] == 2 and j["warmup"] == 3
    assert j["value"] > 0 and j["gpu_launches"] > 0
    assert j["e2e"]["value"] > 0 and j["e2e"]["h2d_bytes_per_step"] > 0
    assert 0 < j["roofline"]["frac"] <= 1.5


@pytest.mark.gpu
def test_bench_dist_line():
    j = _run("--dist", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-model-cpu")
    assert j["value"] > 0 and j["gpu_launches"] > 0
    assert j["e2e"]["value"] > 0
