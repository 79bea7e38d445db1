"""The distributed strategies on the GPU: 2-4 ranks share cuda:0 with gloo
collectives (the box has one GPU), running the same kernels and the same
device reductions the NCCL path uses.  Mirrors the reference's equivalence
lattice (pkg/tests/test_strategies.py:71-96, 164-197, 235-318)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import zo_oracle as O  # noqa: E402
from tests import dist_helpers as H  # noqa: E402


def _single(name, steps):
    import torch

    from paper_2507_03211_b200 import ops, zo
    from paper_2507_03211_b200.engine import DeviceStore
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import iteration_seeds

    v, d, h, n, t, bsz = {"tiny": (16, 16, 2, 2, 8, 4), "mid": (64, 32, 4, 2, 16, 4)}[name]
    cfg = ModelConfig(v, d, h, n, t, "f32")
    store = DeviceStore(cfg, init_seed=7)
    hyper = zo.ZoHyper(1e-3, 1e-2)
    recs = []
    for j, s in enumerate(iteration_seeds(5, steps), 1):
        r = zo.mezo_step(store, make_batch(cfg, bsz, 200 + j), hyper, s, iteration=j)
        recs.append((r.loss_pos, r.loss_neg, r.g))
    return recs, int(ops.hash_u64(store.theta).item()), store.theta.cpu().numpy()


def test_pertp_equals_mezo_bit_exact():
    res = H.run(H.gpu_strategy_worker, 2, "pertp", "mid", 3, False)
    recs, hsh, theta = _single("mid", 3)
    for r in res:
        assert r[1] == recs            # both ranks see the identical records
        assert r[2] == hsh             # replicas identical, and equal to the 1-GPU path
    assert np.array_equal(res[0][3], theta)
    assert set(res[0][5]) <= {"seed", "loss", "grad", "checksum"}   # no parameter traffic


def test_2d_one_group_equals_pertp_and_two_groups_equals_ddp():
    p = H.run(H.gpu_strategy_worker, 2, "2d", "tiny", 3, False)
    q = H.run(H.gpu_strategy_worker, 2, "pertp", "tiny", 3, False)
    assert p[0][1] == q[0][1] and p[0][2] == q[0][2]
    d4 = H.run(H.gpu_strategy_worker, 4, "2d:pertp_inner", "tiny", 2, False)
    d4b = H.run(H.gpu_strategy_worker, 4, "2d:ddp_inner", "tiny", 2, False)
    dd = H.run(H.gpu_strategy_worker, 2, "ddp", "tiny", 2, False)
    gs = [[r[2] for r in x[0][1]] for x in (d4, d4b, dd)]
    assert gs[0] == gs[1] == gs[2]                 # identical g sequence
    assert len({x[2] for x in d4 + d4b + dd}) == 1  # identical replicas everywhere
    # same numerics, different collective structure (test_strategies.py:293-318)
    assert d4[0][4] != d4b[0][4]


def test_pertp_oracle_mode_against_reference_fixture(golden):
    res = H.run(H.gpu_strategy_worker, 2, "pertp", "tiny", 3, True)
    ref = golden["dist/pertp"]
    for (lp, ln, g), (rlp, rln, rg) in zip(res[0][1], ref):
        assert abs(lp - rlp) <= 2e-3 and abs(ln - rln) <= 2e-3
        assert abs(g - rg) <= 2e-3 / 1e-3
    # the final weights track the reference within the K*lr*max|dg|*max|z| bound
    om = O.Model(16, 16, 2, 2, 8, init_seed=7)
    dg = max(abs(a[2] - b[2]) for a, b in zip(res[0][1], ref))
    for j, s in enumerate(O.iteration_seeds(5, 3), 1):
        ids, tg = O.synthetic_batch(16, 8, 4, 200 + j)
        O.mezo_step(om, ids, tg, 1e-3, 1e-2, s)
    zmax = max(float(np.abs(np.concatenate(O.z_stream(s, om.sizes))).max()) for s in O.iteration_seeds(5, 3))
    diff = np.abs(res[0][3].astype(np.float64) - np.concatenate(om.blocks)).max()
    assert diff <= 3 * 1e-2 * dg * zmax + 1e-6


def test_replica_divergence_is_detected():
    """test_strategies.py:121-140: a silently corrupted replica makes the
    post-step replica check raise ConsistencyError on every rank."""
    res = H.run(H.gpu_strategy_edge_worker, 2, "divergence")
    assert [r[1]["raised"] for r in res] == ["ConsistencyError", "ConsistencyError"]


def test_ddp_gradient_traffic_is_k_scalars_per_iteration():
    """test_strategies.py:200-215: only 8 B of g per rank per iteration move
    (plus the seed broadcast and the replica checksum); no parameter bytes."""
    res = H.run(H.gpu_strategy_edge_worker, 4, "traffic")
    assert sum(r[1]["bytes"]["grad"] for r in res) == 3 * 4 * 8
    assert all(r[1]["bytes"].get("param", 0) == 0 for r in res)


def test_ddp_k1_equals_eager():
    """test_strategies.py:218-226."""
    res = H.run(H.gpu_strategy_edge_worker, 1, "k1")
    assert res[0][1]["same"]


def test_wrong_worker_counts_are_configuration_errors():
    """test_strategies.py:114-118 and 321-326 (3 ranks)."""
    res = H.run(H.gpu_strategy_edge_worker, 3, "wrong_count")
    assert all(r[1] == {"pertp": "ConfigurationError", "twod": "ConfigurationError"} for r in res)


# ---------------------------------------------------------------------------
# the lazy mesh (MeshZo) against the REAL reference's recorded dist runs
# (tests/golden: zosim pertp_step / ddp_step / twod_step, strategies.py:92-222;
# properties at pkg/tests/test_strategies.py:164-197, 235-290)
# ---------------------------------------------------------------------------
_MESH_CASES = [("pertp", 2), ("ddp", 2), ("ddp", 4), ("2d:pertp_inner", 4), ("2d:ddp_inner", 4)]


def _golden_path():
    import os

    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


@pytest.mark.parametrize("strategy,world", _MESH_CASES)
def test_mesh_oracle_f32_matches_reference_dist_records(strategy, world):
    """f32 parity mode + reference z: every rank's (L+, L-, g) per step
    within 1e-6 (losses) / 1e-4 relative (g) of the reference rank's record;
    the flushed replicas are identical on every rank and within
    K * lr * max|dg| * max|z| of the oracle's eager trajectory."""
    res = H.run(H.mesh_golden_worker, world, strategy, "f32", False, _golden_path())
    dg = 0.0
    for r in res:
        for (lp, ln, g), (rlp, rln, rg) in zip(r[1], r[2]):
            # (a PertP / 2D rank's record holds its group's L+ and L-, like the reference's)
            assert abs(lp - rlp) <= 1e-6 and abs(ln - rln) <= 1e-6, (strategy, r[0], lp, rlp, ln, rln)
            assert abs(g - rg) <= 1e-4 * max(1.0, abs(rg)), (strategy, r[0], g, rg)
            dg = max(dg, abs(g - rg))
    assert len({r[5].tobytes() for r in res}) == 1            # replicas bit-identical
    kind, ordering = (strategy.split(":") + ["pertp_inner"])[:2]
    om = O.Model(16, 16, 2, 2, 8, init_seed=7)
    seeds = O.iteration_seeds(5, 3)
    for j, s in enumerate(seeds, 1):
        ids, tg = O.synthetic_batch(16, 8, 4, 200 + j)
        if kind == "pertp":
            O.mezo_step(om, ids, tg, 1e-3, 1e-2, s)
        elif kind == "ddp":
            O.ddp_step(om, ids, tg, 1e-3, 1e-2, world, s)
        else:
            O.twod_step(om, ids, tg, 1e-3, 1e-2, world // 2, s, ordering)
    zmax = max(float(np.abs(np.concatenate(O.z_stream(s, om.sizes))).max()) for s in seeds)
    diff = np.abs(res[0][5].astype(np.float64) - np.concatenate(om.blocks)).max()
    assert diff <= 3 * 1e-2 * dg * zmax + 1e-6


@pytest.mark.parametrize("strategy,world", _MESH_CASES)
def test_mesh_teacher_forced_reproduces_reference_checksum(strategy, world):
    """Feeding each rank the reference's g as g_prev (what the reference's
    lazy executors apply), the flushed master of every rank has exactly the
    reference's SHA-256 (dist/*_sha): the lazy mesh's perturb / update
    arithmetic and z are the reference's bit for bit."""
    res = H.run(H.mesh_golden_worker, world, strategy, "f32", True, _golden_path())
    for r in res:
        assert r[3] == r[4], (strategy, r[0])


@pytest.mark.parametrize("strategy,world", [("pertp", 2), ("2d", 4)])
def test_mesh_fill_plan_equals_serial_plan(strategy, world):
    """MeshZo's fill plan (blocks 2.. perturbed on a low-priority stream under
    the forward) gives the serial plan's records and
    flushed master bit for bit on every rank."""
    fill = H.run(H.mesh_plan_worker, world, strategy, "fill", 3)
    ser = H.run(H.mesh_plan_worker, world, strategy, "none", 3)
    for a, b in zip(sorted(fill), sorted(ser)):
        assert a[1] == b[1] and a[2] == b[2], (a, b)
    assert len({r[2] for r in fill}) == 1          # identical replicas
