"""GPU mirror of the reference's pkg/tests/test_zo_core.py: the same
properties, checked on the B200 path.  With a numpy Generator as the
direction source (oracle mode) the perturb / update arithmetic is the
reference's bit for bit, so "bit-exact" assertions carry over unchanged; the
forward is bf16 (tolerances as DESIGN.md states).

test_estimator_second_order_in_epsilon runs in the f32 parity mode at larger
eps than the reference's f64 version (tests/test_oracle_golden.py keeps the
f64 one on the oracle), so the eps^2 term dominates f32 loss rounding."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2507_03211_b200 import zo  # noqa: E402
from paper_2507_03211_b200.engine import PLUS, DeviceStore  # noqa: E402
from paper_2507_03211_b200.errors import NumericError, ProtocolError  # noqa: E402
from paper_2507_03211_b200.model import ModelConfig, make_batch  # noqa: E402
from paper_2507_03211_b200.rng import RngStateManager, iteration_seeds  # noqa: E402

TINY = ModelConfig(16, 16, 2, 2, 8, "f32")
HYPER = zo.ZoHyper(1e-3, 1e-2)


def _store(cfg=TINY, seed=7):
    return DeviceStore(cfg, init_seed=seed, device="cuda:0")


def _theta(store):
    return store.theta.cpu().numpy().copy()


def _oracle_gen(seed):
    mgr = RngStateManager("oracle")
    mgr.reset(seed)
    return mgr, mgr.generator(seed)


def test_perturb_restore_cycle_is_bit_exact():
    """test_zo_core.py:44-63: +eps, -2eps, +eps leaves the master untouched and
    the forward views back at the unperturbed values."""
    rng = np.random.default_rng(0)
    for trial in range(4):
        cfg = ModelConfig(int(rng.integers(4, 12)), int(rng.choice([4, 8, 12])), 2, int(rng.integers(1, 3)), 4,
                          "f32")
        store = _store(cfg, trial)
        before = _theta(store)
        seed = int(rng.integers(0, 2**31))
        mgr = RngStateManager("oracle")
        for scale in (HYPER.epsilon, -2 * HYPER.epsilon, HYPER.epsilon):
            mgr.reset(seed)
            zo.perturb_params(store, scale, mgr.generator(seed))
        assert np.array_equal(_theta(store), before)
        assert all(b.pert_scale == 0.0 for b in store.blocks)
        # closed cycle: the forward equals the unperturbed forward
        batch = make_batch(cfg, 2, 1)
        closed = zo.forward(store, batch.token_ids).cpu()
        fresh = zo.forward(_store(cfg, trial), batch.token_ids).cpu()
        assert torch.equal(closed, fresh)


def test_perturb_scale_zero_advances_rng_without_touching_values():
    """test_zo_core.py:66-76."""
    store = _store()
    before = _theta(store)
    mgr, gen = _oracle_gen(3)
    zo.perturb_params(store, 0.0, gen)
    assert np.array_equal(_theta(store), before)
    ref = np.random.Generator(np.random.PCG64(3))
    ref.standard_normal(store.total_params)
    assert gen.bit_generator.state == ref.bit_generator.state


def test_update_with_zero_gradient_is_value_noop():
    """test_zo_core.py:93-103."""
    store = _store()
    before = _theta(store)
    mgr, gen = _oracle_gen(9)
    zo.update_params(store, 0.0, 1e-2, gen)
    assert np.array_equal(_theta(store), before)
    ref = np.random.Generator(np.random.PCG64(9))
    ref.standard_normal(store.total_params)
    assert gen.bit_generator.state == ref.bit_generator.state


def test_update_matches_explicit_logged_z():
    """test_zo_core.py:106-116, bit-exact: theta' = f32(f64(theta) - (lr*g) z)."""
    store = _store()
    base = _theta(store).astype(np.float64)
    g, lr = 0.7, 1e-2
    _, gen = _oracle_gen(21)
    zo.update_params(store, g, lr, gen)
    z = np.random.Generator(np.random.PCG64(21))
    want = np.concatenate([(base[bl.key0:bl.key0 + bl.elem_count] - (lr * g) * z.standard_normal(bl.elem_count))
                           for bl in store.layouts]).astype(np.float32)
    assert np.array_equal(_theta(store), want)


def test_update_while_perturbed_is_protocol_error():
    """test_zo_core.py:119-126."""
    store = _store()
    mgr, gen = _oracle_gen(2)
    zo.perturb_params(store, 1e-3, gen)
    with pytest.raises(ProtocolError):
        zo.update_params(store, 1.0, 1e-2, mgr.generator(2))
    mgr.reset(2)
    zo.perturb_params(store, -1e-3, mgr.generator(2))


def test_mezo_step_deterministic():
    """test_zo_core.py:147-153 (Philox and oracle directions)."""
    for mode in ("philox", "oracle"):
        a, b = _store(), _store()
        batch = make_batch(TINY, 4, 3)
        ra = zo.mezo_step(a, batch, HYPER, 42, mgr=RngStateManager(mode))
        rb = zo.mezo_step(b, batch, HYPER, 42, mgr=RngStateManager(mode))
        assert a.equal(b)
        assert (ra.loss_pos, ra.loss_neg, ra.g) == (rb.loss_pos, rb.loss_neg, rb.g)


def test_mezo_update_matches_manual_composition():
    """test_zo_core.py:174-183: the eager step's update is exactly
    theta - (lr * g) z with the reference's z and the step's own g."""
    store = _store()
    base = _theta(store).astype(np.float64)
    step = zo.mezo_step(store, make_batch(TINY, 4, 3), HYPER, 99, mgr=RngStateManager("oracle"))
    z = np.random.Generator(np.random.PCG64(99))
    want = np.concatenate([(base[bl.key0:bl.key0 + bl.elem_count]
                            - (HYPER.lr * step.g) * z.standard_normal(bl.elem_count)) for bl in store.layouts])
    assert np.array_equal(_theta(store), want.astype(np.float32))


def test_mezo_losses_match_recomputed_forwards():
    """test_zo_core.py:156-171: L+/L- equal fresh forwards at theta +/- eps z
    (same kernels, so equal bit for bit)."""
    store = _store()
    batch = make_batch(TINY, 4, 3)
    step = zo.mezo_step(store, batch, HYPER, 13, mgr=RngStateManager("oracle"))
    probe = _store()
    for sign, want in ((+1, step.loss_pos), (-1, step.loss_neg)):
        mgr, gen = _oracle_gen(13)
        zo.perturb_params(probe, sign * HYPER.epsilon, gen)
        assert zo.loss(zo.forward(probe, batch.token_ids), batch) == pytest.approx(want, abs=2e-3)
        mgr.reset(13)
        zo.perturb_params(probe, -sign * HYPER.epsilon, mgr.generator(13))


def _dual_pass(store, hyper, seed, batch, mgr):
    mgr.reset(seed)
    rs = mgr.capture(seed)
    x_pos = x_neg = batch.token_ids
    lrs = None
    for block in store.blocks:
        x_pos, x_neg, rs, lrs = zo.dual_forward(block, hyper, seed, mgr, rs, lrs, 0.0, x_pos, x_neg,
                                                apply_pending=False)
    return x_pos, x_neg


def test_dual_forward_first_iteration_restores_parameters():
    """test_zo_core.py:236-249."""
    store = _store()
    before = _theta(store)
    batch = make_batch(TINY, 4, 5)
    x_pos, x_neg = _dual_pass(store, HYPER, 5, batch, RngStateManager("oracle"))
    assert np.array_equal(_theta(store), before)
    assert zo.loss(x_pos, batch) != zo.loss(x_neg, batch)


def test_dual_forward_zero_epsilon_equals_plain_forward():
    """test_zo_core.py:252-265."""
    store = _store()
    batch = make_batch(TINY, 4, 5)
    plain = zo.forward(store, batch.token_ids).cpu()
    x_pos, x_neg = _dual_pass(store, zo.ZoHyper(epsilon=0.0, lr=1e-2), 5, batch, RngStateManager("oracle"))
    assert torch.equal(x_pos.cpu(), plain) and torch.equal(x_neg.cpu(), plain)


def test_dual_forward_pending_without_state_is_protocol_error():
    """test_zo_core.py:268-276."""
    store = _store()
    batch = make_batch(TINY, 4, 5)
    mgr = RngStateManager("oracle")
    mgr.reset(5)
    with pytest.raises(ProtocolError):
        zo.dual_forward(store.blocks[0], HYPER, 5, mgr, mgr.capture(5), None, 0.5, batch.token_ids,
                        batch.token_ids, apply_pending=True)


@pytest.mark.parametrize("mode", ["philox", "oracle"])
def test_streaming_matches_eager_with_flush(mode):
    """test_zo_core.py:279-294, including the FIFO depth after each step."""
    eager, lazy = _store(), _store()
    sz = zo.StreamingZo(lazy, HYPER, mgr=RngStateManager(mode))
    emgr = RngStateManager(mode)
    for j, s in enumerate(iteration_seeds(17, 5), 1):
        batch = make_batch(TINY, 4, 100 + j)
        re = zo.mezo_step(eager, batch, HYPER, s, mgr=emgr, iteration=j)
        rl = sz.step(batch, s)
        assert (re.loss_pos, re.loss_neg, re.g) == (rl.loss_pos, rl.loss_neg, rl.g)
        assert sz.mgr.fifo_depth == 1
    assert not eager.equal(lazy)
    sz.flush()
    assert eager.equal(lazy)


def test_flush_with_zero_gradient_is_value_noop():
    """test_zo_core.py:297-305: flush applies the CURRENT g_prev."""
    store = _store()
    sz = zo.StreamingZo(store, HYPER)
    sz.step(make_batch(TINY, 4, 1), 3)
    sz.g_prev = 0.0
    before = _theta(store)
    sz.flush()
    assert np.array_equal(_theta(store), before)


def test_double_flush_raises_and_stepping_resumes_after_flush():
    """test_zo_core.py:308-325."""
    store = _store()
    sz = zo.StreamingZo(store, HYPER)
    sz.step(make_batch(TINY, 4, 1), 3)
    sz.flush()
    with pytest.raises(ProtocolError):
        sz.flush()
    sz.step(make_batch(TINY, 4, 2), 4)
    sz.flush()
    # == the eager path over the same two steps
    eager = _store()
    zo.mezo_step(eager, make_batch(TINY, 4, 1), HYPER, 3, iteration=1)
    zo.mezo_step(eager, make_batch(TINY, 4, 2), HYPER, 4, iteration=2)
    assert eager.equal(store)


def test_nonfinite_logits_raise_numeric_error():
    """test_model.py:151-155 on the device: a poisoned head turns the CE
    epilogue's error flag into NumericError."""
    store = _store()
    head = store.layouts[-1]
    store.theta[head.key("b_out")] = float("inf")
    with pytest.raises(NumericError):
        zo.mezo_step(store, make_batch(TINY, 4, 1), HYPER, 5)


def _bits(t):
    return t.view(torch.int32).cpu().numpy().copy()


@pytest.mark.parametrize("graph", [False, True])
def test_nonfinite_loss_never_reaches_the_master(graph):
    """A step with non-finite losses raises NumericError BEFORE any update
    touches the master (the reference raises in loss(), model.py:366-367):
    the device arms no deferred update for a non-finite g, so the eager
    update pass and the next fused pass are value no-ops, nothing is left
    pending, and stepping resumes from the last good weights."""
    store = _store()
    head = store.layouts[-1]
    k = head.key("b_out")
    store.theta[k] = float("nan")
    before = _bits(store.theta)
    with pytest.raises(NumericError):
        zo.mezo_step(store, make_batch(TINY, 4, 1), HYPER, 5)
    assert np.array_equal(_bits(store.theta), before)       # no theta -= NaN * z
    assert store.scalars()["pending"] == 0 and store.scalars()["lr_g_prev"] == 0.0
    # lazy: step 1 good, step 2 poisoned -> step 2's pass applied update 1 only
    good, lazy = _store(), _store()
    sz = zo.StreamingZo(lazy, HYPER, overlap=False, graph=graph)
    sz.step(make_batch(TINY, 4, 1), 3)
    zo.mezo_step(good, make_batch(TINY, 4, 1), HYPER, 3, iteration=1)
    lazy.theta[k] = float("nan")
    good.theta[k] = float("nan")
    with pytest.raises(NumericError):
        sz.step(make_batch(TINY, 4, 2), 4)
    a, b = _bits(lazy.theta), _bits(good.theta)
    a[k] = b[k] = 0                       # (NaN - lr g z is a NaN with other payload bits)
    assert np.array_equal(a, b) and bool(torch.isnan(lazy.theta[k]))
    with pytest.raises(ProtocolError):
        sz.flush()                                             # nothing pending
    lazy.theta[k] = 0.0                                        # repair, then resume
    good.theta[k] = 0.0
    r1 = sz.step(make_batch(TINY, 4, 3), 6)
    r2 = zo.mezo_step(good, make_batch(TINY, 4, 3), HYPER, 6, iteration=3)
    assert (r1.loss_pos, r1.loss_neg, r1.g) == (r2.loss_pos, r2.loss_neg, r2.g)
    sz.flush()
    assert lazy.equal(good)


def test_uniform_logits_loss_is_log_vocab():
    """test_model.py:137-140 through the fused CE head: zero head weights and
    bias give uniform logits, so both directional losses are ln V up to the
    bf16 perturbation of the head."""
    store = _store()
    head = store.layouts[-1]
    for name in ("w_out", "b_out"):
        k = head.key(name)
        store.theta[k:k + head.size(name)] = 0.0
    st = zo.mezo_step(store, make_batch(TINY, 4, 1), zo.ZoHyper(1e-6, 1e-2), 5)
    assert abs(st.loss_pos - np.log(TINY.vocab_size)) < 1e-3
    assert abs(st.loss_neg - np.log(TINY.vocab_size)) < 1e-3
    _ = PLUS


def test_store_copy_and_block_views():
    """model.py:140-200: copy equals the source, refuses mid-perturbation
    and with a deferred update outstanding; block views share the master."""
    store = _store()
    c = store.copy()
    assert c.equal(store) and c.checksum() == store.checksum()
    assert store.block(1).kind == "transformer" and len(store.transformer_blocks()) == TINY.n_blocks
    blk = store.block(1)
    blk.buf[0] = 1.5                              # the view writes through to the master
    assert float(store.theta[blk.key0]) == 1.5
    mgr, gen = _oracle_gen(4)
    zo.perturb_block(blk, 1e-3, gen)
    with pytest.raises(ProtocolError):
        store.copy()
    with pytest.raises(ProtocolError):
        blk.copy()
    mgr.reset(4)
    zo.perturb_block(blk, -1e-3, mgr.generator(4))
    sz = zo.StreamingZo(store, HYPER)
    sz.step(make_batch(TINY, 4, 1), 3)
    with pytest.raises(ProtocolError):
        store.copy()
    sz.flush()
    assert store.copy().equal(store)


def _block_ref_out(kind, buf, cfg, x):
    from oracle import zo_oracle as O

    return O.block_forward(kind, buf, cfg.vocab_size, cfg.d_model, cfg.seq_len, cfg.n_heads, x)


@pytest.mark.parametrize("precision,rtol", [("f32", 2e-5), ("bf16", 3e-2)])
def test_dual_forward_values_match_oracle_blocks(precision, rtol):
    """Alg. 2 per block (zo.py:181-224) against the oracle's pure block
    forward (model.py:298-346) on the reference's perturbed buffers: every
    block's +eps / -eps outputs, first without a pending update, then (next
    iteration) with the deferred update folded in -- the block's master then
    equals O.updated(base, g_prev, lr, z_prev) bit for bit and the outputs
    are the oracle's forward of O.perturbed(O.updated(...), +-eps, z).  Each
    block is fed the device's own input, so the error is per block.  f32
    parity mode to 2e-5 relative; the bf16 production kernels to the
    operand-rounding scale."""
    from oracle import zo_oracle as O

    cfg = ModelConfig(64, 32, 4, 2, 16, "f32")
    store = DeviceStore(cfg, init_seed=7, device="cuda:0", precision=precision)
    om = O.Model(64, 32, 4, 2, 16, init_seed=7)
    kinds = O.block_kinds(cfg.n_blocks)
    ids, _ = O.synthetic_batch(64, 16, 2, 77)
    seeds = iteration_seeds(23, 2)
    g_prev = 0.61803
    mgr = RngStateManager("oracle")
    base = [b.copy() for b in om.blocks]
    start_prev = None
    for it, seed in enumerate(seeds):
        mgr.reset(seed)
        rs = mgr.capture(seed)                  # this iteration's stream start (zo.py:264-266)
        lrs = start_prev if it == 1 else None   # the previous iteration's, for the deferred update
        start_prev = rs
        zs = O.z_stream(seed, om.sizes)
        zprev = O.z_stream(seeds[0], om.sizes) if it == 1 else None
        xp = xn = ids
        for bid, blk in enumerate(zo.store_blocks(store)):
            op, on, rs, lrs = zo.dual_forward(blk, HYPER, seed, mgr, rs, lrs, g_prev, xp, xn, it == 1)
            if it == 1:
                base[bid] = O.updated(base[bid], g_prev, HYPER.lr, zprev[bid])
            assert np.array_equal(blk.buf.cpu().numpy(), base[bid]), (it, bid)   # updated / restored exactly
            for out, x, sc in ((op, xp, +HYPER.epsilon), (on, xn, -HYPER.epsilon)):
                xin = x if kinds[bid] == "embedding" else x.cpu().numpy()
                want = _block_ref_out(kinds[bid], O.perturbed(base[bid], sc, zs[bid]), cfg, xin)
                got = out.cpu().numpy()
                scale = float(np.abs(want).max())
                assert float(np.abs(got - want).max()) <= rtol * scale, (precision, it, bid, sc)
            xp, xn = op, on


def test_estimator_second_order_in_epsilon_f32_mode():
    """pkg/tests/test_zo_core.py:185-229 on the GPU: the projected gradient of
    the f32 parity mode (reference z injected) converges to the directional
    derivative z . grad L as eps^2 -- the empirical order of the error between
    eps and eps/2, averaged over 10 directions, lies in [1.8, 2.2].  z . grad L
    is the oracle's f64 central difference at h = 1e-5 (O(h^2) ~ 1e-10).  The
    update is negligible (lr = 1e-30: only the zero-initialised biases move, by ~1e-30)."""
    import math

    from oracle import zo_oracle as O

    from paper_2507_03211_b200.model import Batch

    cfg = ModelConfig(16, 16, 2, 1, 8, "f32")
    store = DeviceStore(cfg, init_seed=3, precision="f32")
    o32 = O.Model(16, 16, 2, 1, 8, init_seed=3)
    assert np.array_equal(store.theta.cpu().numpy(), np.concatenate(o32.blocks))
    m64 = O.Model(16, 16, 2, 1, 8, dtype=np.float64, blocks=[b.astype(np.float64) for b in o32.blocks])
    ids, tg = O.synthetic_batch(16, 8, 2, 5)
    eps_full, h = 2e-3, 1e-5          # asymptotic regime: the f32 oracle gives order 1.99 here
    e_full, e_half = [], []
    for seed in range(10):
        zs = O.z_stream(seed, m64.sizes)
        proj = (m64.loss_at(+h, zs, ids, tg) - m64.loss_at(-h, zs, ids, tg)) / (2 * h)
        errs = []
        for eps in (eps_full, eps_full / 2):
            got = zo.mezo_step(store, Batch(ids, tg), zo.ZoHyper(eps, 1e-30), seed, mgr=RngStateManager("oracle"))
            errs.append(abs(got.g - proj))
        e_full.append(errs[0])
        e_half.append(errs[1])
    drift = np.abs(store.theta.cpu().numpy().astype(np.float64) - np.concatenate(o32.blocks)).max()
    assert drift < 1e-25, drift          # updates below an ulp of the weights (zero-init biases move by ~1e-30)
    order = math.log2(np.mean(e_full) / np.mean(e_half))
    assert 1.8 <= order <= 2.2, (order, e_full, e_half)


def test_graph_replay_with_changing_batch_shapes_matches_eager():
    """The public step replays one I/O-carrying graph per batch shape (its own
    pinned staging): alternating shapes, and coming back to an earlier one,
    gives the eager executor's records and master bit for bit."""
    cfg = ModelConfig(32, 32, 4, 2, 16, "f32")
    shapes = [(2, 16), (1, 8), (2, 16), (4, 8), (1, 8), (2, 16)]
    seeds = iteration_seeds(61, len(shapes))
    runs = []
    for graph in (True, False):
        store = _store(cfg)
        sz = zo.StreamingZo(store, HYPER, graph=graph)
        recs = []
        for j, ((b, t), s) in enumerate(zip(shapes, seeds), 1):
            full = make_batch(cfg, b, 80 + j)
            batch = type(full)(full.token_ids[:, :t], full.targets[:, :t])
            r = sz.step(batch, s)
            recs.append((r.loss_pos, r.loss_neg, r.g))
        sz.flush()
        runs.append((recs, _theta(store)))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])


def test_zo_sgd_reduces_the_loss_end_to_end():
    """End to end, the shipped path trains: ZO-SGD (lazy update, fill / graph
    replay) memorising one fixed batch on a small model lowers the mean of the
    two directional losses well below its start (ln V = 4.16; measured
    4.12 -> 2.93 over 3000 steps at this lr)."""
    cfg = ModelConfig(64, 64, 4, 2, 32, "f32")
    store = _store(cfg)
    sz = zo.StreamingZo(store, zo.ZoHyper(1e-3, 1e-3))
    batch = make_batch(cfg, 4, 123)
    losses = []
    for s in iteration_seeds(5, 1500):
        r = sz.step(batch, s)
        losses.append(0.5 * (r.loss_pos + r.loss_neg))
    sz.flush()
    first, last = float(np.mean(losses[:50])), float(np.mean(losses[-50:]))
    assert np.isfinite(losses).all()
    assert last < first - 0.3, (first, last)
