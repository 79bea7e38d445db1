"""Real OPT on the B200 path: ReLU FFN, tied bias-free
LM head (CE GEMM on the embedding's bf16 shadow as a K-major B operand),
positions with offset 2.

Checker: tests/opt_ref.py, a plain-torch fp32 OPT forward pinned to HF
transformers' OPTForCausalLM by tests/test_opt_cpu.py.  Tolerances (bf16
operands, fp32 accumulate): logits |d| <= 2e-2 * max|ref| + 1e-3, losses
|dL| <= 3e-3, projected gradient |dg| <= 3e-3 / eps; the update itself is
fp32 arithmetic on the master (checked to 1 ulp of the result + 1 ulp of the product)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2507_03211_b200 import checkpoint as CK  # noqa: E402
from paper_2507_03211_b200 import ops, opt, zo  # noqa: E402
from paper_2507_03211_b200.engine import DeviceStore  # noqa: E402
from paper_2507_03211_b200.model import Batch, OPTConfig  # noqa: E402
from paper_2507_03211_b200.rng import iteration_seeds  # noqa: E402
from paper_2507_03211_b200.scheduler import HostStore, OffloadedZo  # noqa: E402
from tests.opt_ref import ce_f64, opt_forward_ref, random_opt_state  # noqa: E402

CASES = {  # name: (vocab, d, heads, layers, seq, max_pos, batch)
    "tiny": (96, 64, 4, 2, 24, 32, 2),
    "hd64": (500, 128, 2, 2, 64, 64, 2),
    "hd128": (1000, 256, 2, 3, 128, 130, 2),
}


def _setup(name, seed=0):
    v, d, h, n, t, mp, b = CASES[name]
    cfg = OPTConfig(v, d, h, n, t, "f32", max_positions=mp).validate()
    sd = random_opt_state(v, d, h, n, mp, seed=seed)
    master = opt.master_from_hf(sd, cfg)
    store = DeviceStore(cfg, init_seed=0, device="cuda:0", init="none")
    store.theta.copy_(torch.from_numpy(master))
    g = np.random.default_rng(seed + 1)
    ids = g.integers(0, v, (b, t + 1))
    return cfg, sd, master, store, Batch(ids[:, :-1], ids[:, 1:])


def _ref_loss(master, cfg, batch):
    sd = opt.hf_from_master(master, cfg)
    logits = opt_forward_ref(sd, cfg.n_heads, torch.from_numpy(batch.token_ids))
    return ce_f64(logits, torch.from_numpy(batch.targets)), logits


@pytest.mark.parametrize("name", list(CASES))
def test_forward_matches_opt_reference(name):
    cfg, sd, master, store, batch = _setup(name)
    got = zo.forward(store, batch.token_ids).cpu()
    want = opt_forward_ref(sd, cfg.n_heads, torch.from_numpy(batch.token_ids))
    assert float((got - want).abs().max()) <= 2e-2 * float(want.abs().max()) + 1e-3
    assert abs(zo.loss(got.cuda(), batch) - ce_f64(want, torch.from_numpy(batch.targets))) <= 3e-3


@pytest.mark.parametrize("name", list(CASES))
def test_mezo_step_matches_reference_at_perturbed_weights(name):
    eps, lr = 1e-2, 1e-3
    cfg, sd, master, store, batch = _setup(name)
    seed = iteration_seeds(5, 1)[0]
    rec = zo.mezo_step(store, batch, zo.ZoHyper(eps, lr), seed)
    z = ops.philox_normals(seed, 0, master.size).cpu().numpy().astype(np.float64)
    lp, _ = _ref_loss((master + eps * z).astype(np.float32), cfg, batch)
    ln, _ = _ref_loss((master - eps * z).astype(np.float32), cfg, batch)
    assert abs(rec.loss_pos - lp) <= 3e-3 and abs(rec.loss_neg - ln) <= 3e-3
    assert abs(rec.g - (lp - ln) / (2 * eps)) <= 3e-3 / eps
    want = (master.astype(np.float64) - (lr * rec.g) * z).astype(np.float32)
    got = store.theta.cpu().numpy()
    # fp32 update: one rounding of the result plus the fp32 product (lr g) z
    tol = 1.5 * np.spacing(np.abs(want)) + 2.4e-7 * np.abs(lr * rec.g * z)
    assert np.all(np.abs(got - want) <= tol)


def test_lazy_equals_eager_and_offloaded_equals_resident():
    """The equivalence lattice holds for the OPT architecture too: lazy ==
    eager after flush, and the ZO2 offload runtime (embedding resident so
    the tied head reads it) == resident, bit-exact."""
    name = "hd64"
    h = zo.ZoHyper(1e-3, 1e-3)
    cfg, _, master, a, _ = _setup(name)
    b = DeviceStore(cfg, init_seed=0, device="cuda:0", init="none")
    b.theta.copy_(a.theta)
    host = HostStore(cfg, init_seed=0, init="none")
    host.theta.copy_(torch.from_numpy(master))
    sz = zo.StreamingZo(b, h)
    rt = OffloadedZo(host, h, batch=CASES[name][6])
    g = np.random.default_rng(3)
    for j, s in enumerate(iteration_seeds(7, 4), 1):
        ids = g.integers(0, cfg.vocab_size, (2, cfg.seq_len + 1))
        batch = Batch(ids[:, :-1], ids[:, 1:])
        ra = zo.mezo_step(a, batch, h, s, iteration=j)
        rb = sz.step(batch, s)
        rc = rt.step(batch, s)
        assert (ra.loss_pos, ra.loss_neg, ra.g) == (rb.loss_pos, rb.loss_neg, rb.g) == \
            (rc.loss_pos, rc.loss_neg, rc.g)
    sz.flush()
    rt.flush()
    assert torch.equal(a.theta, b.theta)
    assert np.array_equal(host.theta.numpy(), a.theta.cpu().numpy())


def test_save_and_load_pretrained_and_zopk(tmp_path):
    cfg, sd, master, store, batch = _setup("tiny")
    sz = zo.StreamingZo(store, zo.ZoHyper(1e-3, 1e-3))
    sz.step(batch, 11)
    sz.flush()
    opt.save_pretrained(store, str(tmp_path / "hf"))
    back = opt.load_pretrained(str(tmp_path / "hf"), seq_len=cfg.seq_len, device="cuda:0")
    assert back.config == cfg and torch.equal(back.theta, store.theta)
    CK.save_checkpoint(store, tmp_path / "ck.zopk")
    st2 = CK.load_checkpoint(tmp_path / "ck.zopk", device="cuda:0")
    assert st2.config == cfg and torch.equal(st2.theta, store.theta)
