"""bench.py's multi-GPU arm (bench_dist) run for real on one GPU: two ranks
under torchrun share cuda:0 (FC_BENCH_SHARED_GPU=1: gloo for the IPC handle
exchange, the NCCL leg skipped), so the code the driver runs at --gpus N is
known to execute before an 8-GPU node is available."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_dist_dry_run_two_ranks_one_gpu():
    env = dict(os.environ, FC_BENCH_SHARED_GPU="1")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c1",
                        "--steps", "3", "--warmup", "3"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-4000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["tp"] == 2
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["roofline"]["peak"] in (900.0, d["roofline"]["peak"]) and 0 < d["roofline"]["frac"]
    assert d["gpu_launches"] >= d["steps"]
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 1024 * 8192
    assert len(d["sweep"]) >= 3 and all(r["int4_us"] > 0 for r in d["sweep"])
