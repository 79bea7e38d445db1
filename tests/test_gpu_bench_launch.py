"""The bench contract under torchrun (the driver's N>1 launch), with every
rank on the one GPU of the test box and gloo instead of NCCL
(ZO_BENCH_SHARE_GPU / ZO_DIST_BACKEND): rank 0 prints exactly one JSON line
with the contract's keys, the other ranks print nothing; the reference arm
runs on rank 0 only."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "gpu_launches", "e2e"}


def _run(n, *extra):
    from tests.dist_helpers import free_port

    env = dict(os.environ, ZO_BENCH_SHARE_GPU="1", ZO_DIST_BACKEND="gloo", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(n), "--steps", "2", "--warmup", "3", "--model", "opt-125m", "--seq", "128",
           *extra]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [2, 4])
def test_bench_multi_rank_line(n):
    d = _run(n)
    assert KEYS <= set(d) and d["n_gpus"] == n and d["scaling"] == "weak"
    assert d["config"]["global_batch"] == 4 * (n // 2)
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


def test_reference_arm_multi_rank():
    d = _run(2, "--impl", "reference")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
