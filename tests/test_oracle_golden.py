"""Pin the CPU oracle (oracle/zo_oracle.py) to the reference's own outputs.

The fixtures in tests/golden/golden.npz were produced by running the real
reference (zosim) in the build container (tests/golden/make_golden.py).
Everything here is bit-exact: same numpy, same op order.
"""

import hashlib
import math

import numpy as np
import pytest

from oracle import zo_oracle as O

EPS, LR = 1e-3, 1e-2


def _case(golden, name):
    for c in golden["_meta"]["cases"]:
        if c["name"] == name:
            return c
    raise KeyError(name)


def _model(golden, c):
    dt = np.float32 if c["dtype"] == "f32" else np.float64
    return O.Model(c["vocab"], c["d"], c["heads"], c["n_blocks"], c["seq"], init_seed=7, dtype=dt)


def _sha(blocks):
    h = hashlib.sha256()
    for b in blocks:
        h.update(b.tobytes())
    return h.hexdigest()


CASES = ["tiny32", "tiny64", "ragged32", "mid32", "wide32"]


def test_numpy_version_matches_fixture(golden):
    # numpy's Generator streams are not promised stable across versions
    assert golden["_meta"]["numpy"] == np.__version__


@pytest.mark.parametrize("name", CASES)
def test_init_layout_and_z_stream(golden, name):
    c = _case(golden, name)
    m = _model(golden, c)
    assert sum(m.sizes) == O.param_count(c["vocab"], c["d"], c["n_blocks"], c["seq"])
    for i, b in enumerate(m.blocks):
        assert np.array_equal(b, golden[f"{name}/init/{i}"])
    seeds = O.iteration_seeds(17, c["steps"])
    assert seeds == [int(s) for s in golden[f"{name}/seeds"]]
    zs = O.z_stream(seeds[0], m.sizes)
    for i, z in enumerate(zs):
        assert np.array_equal(z, golden[f"{name}/z0/{i}"])


@pytest.mark.parametrize("name", CASES)
def test_forward_loss_and_mezo_trajectory_bit_exact(golden, name):
    c = _case(golden, name)
    m = _model(golden, c)
    seeds = O.iteration_seeds(17, c["steps"])
    recs = []
    for j, s in enumerate(seeds, 1):
        ids, tgt = O.synthetic_batch(c["vocab"], c["seq"], c["batch"], 100 + j)
        assert np.array_equal(ids, golden[f"{name}/ids/{j}"])
        assert np.array_equal(tgt, golden[f"{name}/tgt/{j}"])
        if j == 1:
            logits = m.forward(ids)
            assert np.array_equal(logits, golden[f"{name}/logits1"])
            assert O.cross_entropy(logits, tgt) == float(golden[f"{name}/loss1"])
        recs.append(O.mezo_step(m, ids, tgt, EPS, LR, s))
        if j == 1:
            for i, b in enumerate(m.blocks):
                assert np.array_equal(b, golden[f"{name}/after1/{i}"])
    assert np.array_equal(np.array(recs), golden[f"{name}/mezo"])
    for i, b in enumerate(m.blocks):
        assert np.array_equal(b, golden[f"{name}/final/{i}"])
    assert _sha(m.blocks) == str(golden[f"{name}/final_sha"])


@pytest.mark.parametrize("name", CASES)
def test_lazy_update_matches_streaming_and_offload(golden, name):
    c = _case(golden, name)
    m = _model(golden, c)
    lz = O.LazyZo(m, EPS, LR)
    recs = []
    for j, s in enumerate(O.iteration_seeds(17, c["steps"]), 1):
        ids, tgt = O.synthetic_batch(c["vocab"], c["seq"], c["batch"], 100 + j)
        recs.append(lz.step(ids, tgt, s))
    for i, b in enumerate(m.blocks):
        assert np.array_equal(b, golden[f"{name}/lazy_unflushed/{i}"])   # host lags one update
    lz.flush()
    assert np.array_equal(np.array(recs), golden[f"{name}/streaming"])
    assert np.array_equal(np.array(recs), golden[f"{name}/offload"])
    assert _sha(m.blocks) == str(golden[f"{name}/streaming_sha"])
    assert _sha(m.blocks) == str(golden[f"{name}/offload_sha"])
    assert _sha(m.blocks) == str(golden[f"{name}/final_sha"])
    with pytest.raises(RuntimeError):
        lz.flush()


def _tiny():
    return O.Model(16, 16, 2, 2, 8, init_seed=7, dtype=np.float32)


def test_pertp_is_mezo_and_matches_reference(golden):
    m = _tiny()
    recs = []
    for j, s in enumerate(O.iteration_seeds(5, 3), 1):
        ids, tgt = O.synthetic_batch(16, 8, 4, 200 + j)
        recs.append(O.mezo_step(m, ids, tgt, EPS, LR, s))
    assert np.array_equal(np.array(recs), golden["dist/pertp"])
    assert _sha(m.blocks) == str(golden["dist/pertp_sha"])


@pytest.mark.parametrize("k", [2, 4])
def test_ddp_matches_reference(golden, k):
    m = _tiny()
    ref = golden[f"dist/ddp{k}"]            # [rank, iter, (lp, ln, g)]
    for j, s in enumerate(O.iteration_seeds(5, 3), 1):
        ids, tgt = O.synthetic_batch(16, 8, 4, 200 + j)
        per, g = O.ddp_step(m, ids, tgt, EPS, LR, k, s)
        for r in range(k):
            assert (per[r][0], per[r][1]) == tuple(ref[r, j - 1, :2])
            assert g == ref[r, j - 1, 2]
    assert _sha(m.blocks) == str(golden[f"dist/ddp{k}_sha"])


@pytest.mark.parametrize("ordering", ["pertp_inner", "ddp_inner"])
def test_2d_matches_reference_and_ddp(golden, ordering):
    m = _tiny()
    ref = golden[f"dist/2d_{ordering}"]
    for j, s in enumerate(O.iteration_seeds(5, 3), 1):
        ids, tgt = O.synthetic_batch(16, 8, 4, 200 + j)
        per, g = O.twod_step(m, ids, tgt, EPS, LR, 2, s, ordering)
        for r in range(4):
            grp = r // 2
            assert (per[grp][0], per[grp][1]) == tuple(ref[r, j - 1, :2])
            assert g == ref[r, j - 1, 2]
    assert _sha(m.blocks) == str(golden[f"dist/2d_{ordering}_sha"])
    assert _sha(m.blocks) == str(golden["dist/ddp2_sha"])


def test_slice_layouts_and_tcomm(golden):
    for total, n, owner, off, ln in golden["comm/layouts"]:
        assert O.slice_layout(int(total), int(n))[int(owner)] == (owner, off, ln)
    for m, n, t in golden["comm/tcomm"]:
        assert O.sliced_upload_time(int(m), int(n), 4e8, 2.4e9) == t


def test_sliced_upload_offload_bytes():
    host = np.arange(1003, dtype=np.float32)
    for n in (1, 2, 3, 8):
        reps = O.sliced_upload(host, n)
        assert all(np.array_equal(r, host) for r in reps)
        back = np.zeros_like(host)
        O.sliced_offload(reps, back)
        assert np.array_equal(back, host)
    reps = O.sliced_upload(host, 2)
    reps[1][5] += 1
    with pytest.raises(ValueError):
        O.sliced_offload(reps, np.zeros_like(host))


def test_known_answers(golden):
    assert O.zo_grad(1.2, 0.8, 0.1) == golden["kat/zo_grad"][0]
    assert O.zo_grad(1.5, 1.5, 0.1) == 0.0
    assert O.cross_entropy(np.zeros((2, 3, 4)), np.zeros((2, 3), dtype=np.int64)) == float(golden["kat/ce_uniform4"])
    assert abs(float(golden["kat/ce_uniform4"]) - math.log(4.0)) < 1e-12
    assert O.iteration_seeds(1234, 8) == [int(s) for s in golden["kat/iteration_seeds_1234"]]


def test_perturb_restore_cycle_exact():
    m = _tiny()
    zs = O.z_stream(3, m.sizes)
    for b, z in zip(m.blocks, zs):
        assert np.array_equal(O.perturbed(b, 0.0, z), b)
        lo, hi = O.perturbed(b, -EPS, z), O.perturbed(b, +EPS, z)
        assert not np.array_equal(lo, hi)


def test_estimator_second_order_in_epsilon():
    """pkg/tests/test_zo_core.py:186-233 on the oracle (f64): the central
    difference's error against z . grad shrinks as eps^2 (empirical order in
    [1.8, 2.2])."""
    m = O.Model(7, 6, 2, 1, 6, init_seed=3, dtype=np.float64)
    ids, tg = O.synthetic_batch(7, 6, 2, 5)

    def loss_at(blocks):
        return O.cross_entropy(m.forward(ids, blocks), tg)

    h = 1e-5
    grad = []
    for bi, blk in enumerate(m.blocks):
        gb = np.empty(blk.size)
        for i in range(blk.size):
            orig = blk[i]
            blk[i] = orig + h
            lp = loss_at(m.blocks)
            blk[i] = orig - h
            lm = loss_at(m.blocks)
            blk[i] = orig
            gb[i] = (lp - lm) / (2 * h)
        grad.append(gb)
    grad = np.concatenate(grad)

    def g_at(eps, seed):
        zs = O.z_stream(seed, m.sizes)
        return O.zo_grad(m.loss_at(+eps, zs, ids, tg), m.loss_at(-eps, zs, ids, tg), eps)

    e_full, e_half = [], []
    for seed in range(10):
        zv = np.concatenate(O.z_stream(seed, m.sizes))
        proj = float(zv @ grad)
        e_full.append(abs(g_at(1e-3, seed) - proj))
        e_half.append(abs(g_at(5e-4, seed) - proj))
    order = math.log2(np.mean(e_full) / np.mean(e_half))
    assert 1.8 <= order <= 2.2, order
