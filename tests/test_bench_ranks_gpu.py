"""The bench's own multi-rank path on the GPU box: ``bench.py --gpus 2`` self-
spawns two ranks (torch.distributed.run, 127.0.0.1).  With one GPU the two ranks
share it (FLAME_SHARE_GPU=1: round-robin devices, gloo plumbing); each rank
scores its own requests and rank 0 prints one line whose value is the
whole-job aggregate over the max-over-ranks device time."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("workload", ["cfg2", "cfg4"])
def test_bench_two_ranks(gpu, workload):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FLAME_SHARE_GPU="1")
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--workload", workload, "--steps", "4", "--warmup", "3",
           "--no-fp32-line", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
