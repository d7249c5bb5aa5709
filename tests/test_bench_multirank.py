"""bench.py's N > 1 step (the measured multi-GPU path: sliced all-to-all
merge in rank order, redundant fold, rank-local scores and sorts, global "dec"
order merged from the sorted runs on rank 0 inside the timed region) run
with 2-3 ranks on one GPU (LVSK_BENCH_SHARE_GPU=1: gloo, host-staged
collectives, never a measurement) and checked by bench.py --verify against
the CPU oracle: merged sketch bit-exact (hashed) / within 1e-4 (SRHT,
Gaussian), scores within tolerance, the order the stable argsort of the
gathered probabilities.  Reference: dist.py:82-151."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("config,rows,world", [("c2", 20_000, 2), ("c2", 7_000, 3), ("c4", 4_000, 2),
                                               ("c3", 20_480, 2), ("c5", 30_001, 3), ("c1", 0, 2)])
def test_bench_multirank_step_matches_oracle(config, rows, world):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, LVSK_BENCH_SHARE_GPU="1", PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", str(world), "--config", config, "--steps", "2", "--warmup", "3", "--no-e2e", "--verify"]
    if rows:
        cmd += ["--rows", str(rows)]
    p = subprocess.run(cmd, cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    lines = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    ver = [ln for ln in lines if ln.get("verify") == "ok"]
    assert ver and ver[0]["world"] == world, out[-4000:]
    bench = [ln for ln in lines if "metric" in ln]
    assert bench and bench[0]["n_gpus"] == world and bench[0]["value"] > 0


@pytest.mark.parametrize("config,rows", [("c2", 20_000), ("c3", 20_480), ("c5", 30_001), ("c1", 0)])
def test_bench_single_gpu_pipelined_matches_oracle(config, rows):
    """N = 1 default: two independent passes in flight (BatchRunner); the
    last pass is checked against the oracle by --verify and the line carries
    the single-pass latency next to the pipelined ms_per_step."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    cmd = [sys.executable, str(ROOT / "bench.py"), "--config", config, "--steps", "4", "--warmup", "3",
           "--no-e2e", "--no-cpu", "--verify"]
    if rows:
        cmd += ["--rows", str(rows)]
    p = subprocess.run(cmd, cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    lines = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert [ln for ln in lines if ln.get("verify") == "ok"], out[-4000:]
    bench = [ln for ln in lines if "metric" in ln]
    assert bench and bench[0]["config"]["passes_in_flight"] == 2, out[-4000:]
    assert bench[0]["latency_ms_per_pass"] > 0 and bench[0]["ms_per_step"] > 0
