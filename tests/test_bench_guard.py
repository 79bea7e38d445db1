"""bench.py's offload leg cannot cost the headline line (CPU: the leg is
replaced by a stub that raises or hangs)."""

import json
import os
import subprocess
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_offload_exception_becomes_an_error_field(monkeypatch):
    def boom(*a, **k):
        raise RuntimeError("NCCL peer vanished")

    monkeypatch.setattr(bench, "offload_leg", boom)
    args = types.SimpleNamespace(offload_timeout=30.0)
    out = bench._guarded_offload(args, 0, 2, 0, {"metric": "m"})
    assert out["error"].startswith("RuntimeError: NCCL peer vanished")


def test_hung_offload_prints_the_line_and_exits_zero():
    code = (
        "import sys, time, types; sys.path.insert(0, %r); import bench\n"
        "bench.offload_leg = lambda *a, **k: time.sleep(60)\n"
        "line = {'metric': 'm', 'value': 1.0}\n"
        "bench._guarded_offload(types.SimpleNamespace(offload_timeout=0.5), 0, 2, 0, line)\n"
        "print('not reached')\n" % ROOT
    )
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=60)
    assert p.returncode == 0, p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and "not reached" not in p.stdout
    d = json.loads(lines[0])
    assert d["value"] == 1.0 and "did not finish" in d["offload"]["error"]
