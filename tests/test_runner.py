"""Run driver + artefacts (src/zosim/bench.py:53-227, 337-346).

CPU: RunConfig validation mirrors the reference's checks; throughput drops
the first two steps like bench.py:194-197.  GPU: ``run`` writes
report.json / steps.jsonl / timeline.json in the reference's format, and the
eager (mezo) and offloaded (zo2) strategies end on the same master.
"""

import json

import pytest

from paper_2507_03211_b200.errors import ConfigurationError
from paper_2507_03211_b200.model import ModelConfig
from paper_2507_03211_b200.runner import MeshConfig, RunConfig, throughput
from paper_2507_03211_b200.zo import ZoHyper

TINY = ModelConfig(16, 16, 2, 2, 8, "f32")
REPORT_KEYS = {"config", "strategy", "workers", "tokens_per_sec", "tokens_per_sec_total", "wall_time",
               "peak_device_bytes", "peak_by_tag", "comm_bytes", "final_checksum", "steps"}


def _rc(**kw):
    base = dict(model=TINY, hyper=ZoHyper(1e-3, 1e-2, 4))
    base.update(kw)
    return RunConfig(**base)


@pytest.mark.parametrize("kw,msg", [
    (dict(strategy="sgd"), "strategy must be one of"),
    (dict(strategy="mezo", mesh=MeshConfig(workers=2)), "runs on 1 worker"),
    (dict(strategy="pertp", mesh=MeshConfig(workers=4)), "exactly 2 workers"),
    (dict(strategy="ddp", mesh=MeshConfig(workers=3)), "not divisible by 3 workers"),
    (dict(strategy="2d", mesh=MeshConfig(workers=4, n_b=2, n_p=3)), "fixed at 2"),
    (dict(strategy="2d", mesh=MeshConfig(workers=6, n_b=2)), "workers = n_b x 2"),
    (dict(strategy="2d", batch_size=3, mesh=MeshConfig(workers=4, n_b=2)), "not divisible by 2 groups"),
    (dict(mesh=MeshConfig(ordering="zigzag")), "ordering must be one of"),
    (dict(batch_size=0), "batch_size must be >= 1"),
])
def test_validate(kw, msg):
    with pytest.raises(ConfigurationError, match=msg):
        _rc(**kw).validate()


def test_from_dict_roundtrip(tmp_path):
    rc = _rc(strategy="2d", batch_size=4, mesh=MeshConfig(workers=4, n_b=2)).validate()
    d = rc.to_dict()
    d["topology"] = {"host_bw": 1e9}          # simulator knob: accepted and ignored
    p = tmp_path / "run.json"
    p.write_text(json.dumps(d))
    back = RunConfig.from_file(p, {"hyper": {"steps": 7}})
    assert back.hyper.steps == 7 and back.mesh == rc.mesh and back.model == rc.model
    with pytest.raises(ConfigurationError, match="not valid JSON"):
        (tmp_path / "bad.json").write_text("{")
        RunConfig.from_file(tmp_path / "bad.json")


def test_throughput_drops_two_warmups():
    assert throughput([9.0, 9.0, 1.0, 1.0], 10) == 10.0
    assert throughput([2.0, 1.0, 1.0], 10) == 10.0       # <= 3 steps: all kept


@pytest.mark.gpu
def test_run_outputs_and_mezo_equals_zo2(tmp_path):
    from paper_2507_03211_b200.runner import run

    reps = {}
    for strat in ("mezo", "zo2"):
        out = tmp_path / strat
        rep = run(_rc(strategy=strat, report_dir=str(out)))
        reps[strat] = rep
        report = json.loads((out / "report.json").read_text())
        assert set(report) == REPORT_KEYS and report["strategy"] == strat and report["steps"] == 4
        lines = (out / "steps.jsonl").read_text().splitlines()
        assert [json.loads(x)["iter"] for x in lines] == [1, 2, 3, 4]
        assert set(json.loads(lines[0])) == {"iter", "seed", "loss_pos", "loss_neg", "g"}
        tl = json.loads((out / "timeline.json").read_text())
        if strat == "zo2":
            assert {e["op"] for e in tl} == {"upload", "compute", "offload"}
            assert report["comm_bytes"]["host_upload_bytes"] > 0
        else:
            assert tl == []
        assert rep.peak_device_bytes > 0 and rep.tokens_per_sec > 0
    # the capacity knob: part of the model resident, same trajectory
    out = tmp_path / "zo2cap"
    rep = run(_rc(strategy="zo2", report_dir=str(out), device_capacity_blocks=3.0))
    reps["zo2cap"] = rep
    assert rep.final_checksum == reps["zo2"].final_checksum
    # transfer compression: same trajectory, half the PCIe bytes
    rep = run(_rc(strategy="zo2", report_dir=str(tmp_path / "zo2c"), offload_compress="split16"))
    assert rep.final_checksum == reps["zo2"].final_checksum
    assert 2 * rep.comm_bytes["host_upload_bytes"] == reps["zo2"].comm_bytes["host_upload_bytes"]
    a, b = reps["mezo"], reps["zo2"]
    assert [(s.loss_pos, s.loss_neg, s.g) for s in a.steps] == [(s.loss_pos, s.loss_neg, s.g) for s in b.steps]
    assert a.final_checksum == b.final_checksum


def test_hyper_validation():
    """pkg/tests/test_zo_core.py:328-334."""
    from paper_2507_03211_b200.errors import NumericError

    with pytest.raises(NumericError):
        ZoHyper(epsilon=0.0, lr=1e-2).validate()
    with pytest.raises(NumericError):
        ZoHyper(epsilon=1e-3, lr=0.0).validate()
    with pytest.raises(NumericError):
        ZoHyper(epsilon=1e-3, lr=1e-2, steps=0).validate()
