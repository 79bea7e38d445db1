"""The bench contract under torchrun (the driver's N>1 launch), with every
rank on the one GPU of the test box and gloo instead of NCCL
(ZO_BENCH_SHARE_GPU / ZO_DIST_BACKEND): rank 0 prints exactly one JSON line
with the contract's keys, the other ranks print nothing; the reference arm
runs on rank 0 only.  The offload leg (the north-star offload target) runs at
a small shape and must report its object at N = 1 (the ZO2 baseline) and
N > 1 (the sliced mesh)."""

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
           "--offload-model", "opt-125m", "--offload-seq", "128", "--offload-steps", "2", "--no-cpu-full", *extra]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [2, 4])
def test_bench_multi_rank_line(n):
    d = _run(n)
    assert KEYS <= set(d) and d["n_gpus"] == n and d["scaling"] == "weak"
    assert d["config"]["global_batch"] == 8 * (n // 2)       # 8 sequences per PertP group: weak scaling
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    _check_offload(d["offload"], n)


OFFLOAD_KEYS = {"workload", "schedule", "n_gpus", "tokens_per_s", "ms_per_step", "h2d_gbs_per_rank",
                "d2h_gbs_per_rank", "nvlink_rx_gbs_per_rank", "per_block_ms", "t_comm_model_ms",
                "pcie_bytes_per_step_per_rank"}


def _check_offload(o, n):
    assert OFFLOAD_KEYS <= set(o) and o["n_gpus"] == n
    assert o["tokens_per_s"] > 0 and o["h2d_gbs_per_rank"] > 0 and o["d2h_gbs_per_rank"] > 0
    assert o["per_block_ms"]["compute"] > 0 and o["t_comm_model_ms"] > 0
    if n == 1:
        assert o["nvlink_rx_gbs_per_rank"] is None and o["compress"] == "none"
    else:
        assert o["nvlink_rx_gbs_per_rank"] > 0 and o["compress"] == "split16"
        assert o["per_block_ms"]["nvlink_exchange"] > 0


def test_bench_single_gpu_line_with_offload_and_cpu_baseline():
    """`bench.py --gpus 1` (no torchrun): the headline line with the roofline
    rows, the offload object of the 1-GPU ZO2 schedule and the CPU baseline."""
    env = dict(os.environ, PYTHONPATH=ROOT)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "2", "--warmup", "3",
           "--model", "opt-125m", "--seq", "128", "--offload-model", "opt-125m", "--offload-seq", "128",
           "--offload-steps", "2", "--no-cpu-full"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["config"]["global_batch"] == 4
    for k in ("perturb", "gemm", "attention", "layernorm"):
        r = d["roofline_other"][k]
        assert r["achieved"] > 0 and 0 < r["frac"] and r["share_of_step"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["extrapolated"] is True
    _check_offload(d["offload"], 1)


def test_reference_arm_multi_rank():
    d = _run(2, "--impl", "reference")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
