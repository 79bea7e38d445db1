"""Size-independent properties at BASELINE's headline size (the OPT-1.3B
shape, T=512, B=4: 1.42 G parameters), where the oracle cannot run: the
equivalence lattice of the reference's own tests (pkg/tests/test_zo_core.py
lazy == eager, test_offload.py offloaded == resident) holds bit for bit on
the production path (stacked plan, CUDA-graph replay, tcgen05 kernels), and
the step is finite and deterministic."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2507_03211_b200 import ops, zo  # noqa: E402
from paper_2507_03211_b200.engine import DeviceStore  # noqa: E402
from paper_2507_03211_b200.model import make_batch, opt_config  # noqa: E402
from paper_2507_03211_b200.rng import iteration_seeds  # noqa: E402
from paper_2507_03211_b200.scheduler import HostStore, OffloadedZo  # noqa: E402

EPS, LR = 1e-3, 1e-7
CFG = opt_config("opt-1.3b", 512)
B = 4


def _batches(n):
    return [make_batch(CFG, B, 99 * 1_000_003 + j) for j in range(1, n + 1)]


def test_fullsize_lazy_graph_equals_eager_bit_exact():
    """StreamingZo (lazy update, stacked +-eps forwards, graph replay) vs the
    eager MeZO step at 1.42 G parameters: identical records every step and an
    identical master after flush."""
    steps = 3
    seeds = iteration_seeds(1234, steps)
    batches = _batches(steps)
    a = DeviceStore(CFG, 7, init="philox")
    recs = [zo.mezo_step(a, batches[j], zo.ZoHyper(EPS, LR), s, iteration=j + 1) for j, s in enumerate(seeds)]
    ha = int(ops.hash_u64(a.theta).item())
    del a
    torch.cuda.empty_cache()
    b = DeviceStore(CFG, 7, init="philox")
    sz = zo.StreamingZo(b, zo.ZoHyper(EPS, LR))
    for j, s in enumerate(seeds):
        r = sz.step(batches[j], s)
        assert (r.loss_pos, r.loss_neg, r.g) == (recs[j].loss_pos, recs[j].loss_neg, recs[j].g)
        assert np.isfinite([r.loss_pos, r.loss_neg, r.g]).all()
    sz.flush()
    assert int(ops.hash_u64(b.theta).item()) == ha


def test_fullsize_offloaded_equals_resident_bit_exact():
    """The ZO2 offload schedule (U/C/O streams, 3 slots, split16 transfer
    compression) at 1.42 G parameters equals the resident lazy step."""
    steps = 2
    seeds = iteration_seeds(77, steps)
    batches = _batches(steps)
    res = DeviceStore(CFG, 7, init="philox")
    sz = zo.StreamingZo(res, zo.ZoHyper(EPS, LR))
    recs = [sz.step(batches[j], s) for j, s in enumerate(seeds)]
    sz.flush()
    final = res.theta.cpu()
    del res, sz
    torch.cuda.empty_cache()
    host = HostStore(CFG, 7, init="philox")
    rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=B, compress="split16")
    for j, s in enumerate(seeds):
        r = rt.step(batches[j], s)
        assert (r.loss_pos, r.loss_neg, r.g) == (recs[j].loss_pos, recs[j].loss_neg, recs[j].g)
    rt.flush()
    assert torch.equal(host.theta, final)


def test_fullsize_long_run_is_finite_and_reproducible():
    """100 lazy steps at 1.42 G parameters (graph replay): every record is
    finite and two runs from the same seeds end on the same master bits."""
    steps = 100
    seeds = iteration_seeds(4321, steps)
    hashes, finals = [], []
    for _ in range(2):
        st = DeviceStore(CFG, 7, init="philox")
        sz = zo.StreamingZo(st, zo.ZoHyper(EPS, LR))
        recs = []
        for j, s in enumerate(seeds):
            recs.append(sz.step(make_batch(CFG, B, 7 * 1_000_003 + j), s))
        sz.flush()
        assert all(np.isfinite([r.loss_pos, r.loss_neg, r.g]).all() for r in recs)
        hashes.append(int(ops.hash_u64(st.theta).item()))
        finals.append([(r.loss_pos, r.loss_neg, r.g) for r in recs[-3:]])
        del st, sz
        torch.cuda.empty_cache()
    assert hashes[0] == hashes[1] and finals[0] == finals[1]


def test_fullsize_real_opt_lazy_graph_equals_eager_bit_exact():
    """The same lattice at the real OPT-1.3B architecture (ReLU FFN, tied
    bias-free LM head through the K-major B operand, positions + 2)."""
    from paper_2507_03211_b200.model import real_opt_config

    cfg = real_opt_config("opt-1.3b", 512)
    steps = 2
    seeds = iteration_seeds(99, steps)
    batches = [make_batch(cfg, B, 5 + j) for j in range(steps)]
    a = DeviceStore(cfg, 7, init="philox")
    recs = [zo.mezo_step(a, batches[j], zo.ZoHyper(EPS, LR), s, iteration=j + 1) for j, s in enumerate(seeds)]
    ha = int(ops.hash_u64(a.theta).item())
    del a
    torch.cuda.empty_cache()
    b = DeviceStore(cfg, 7, init="philox")
    sz = zo.StreamingZo(b, zo.ZoHyper(EPS, LR))
    for j, s in enumerate(seeds):
        r = sz.step(batches[j], s)
        assert (r.loss_pos, r.loss_neg, r.g) == (recs[j].loss_pos, recs[j].loss_neg, recs[j].g)
    sz.flush()
    assert int(ops.hash_u64(b.theta).item()) == ha


def test_fullsize_pertp_mesh_equals_single_gpu_mezo():
    """PertP (the 2D mesh with one group, two ranks sharing cuda:0 over gloo)
    at 1.42 G parameters: both ranks report the single-GPU lazy step's
    records and end on the single-GPU master bits (SPEC lattice PertP ==
    MeZO)."""
    from tests import dist_helpers as H

    steps = 2
    seeds = iteration_seeds(1234, steps)
    st = DeviceStore(CFG, 7, init="philox")
    sz = zo.StreamingZo(st, zo.ZoHyper(EPS, LR))
    want = []
    for j, s in enumerate(seeds):
        r = sz.step(make_batch(CFG, B, 99 * 1_000_003 + j + 1), s)
        want.append((r.loss_pos, r.loss_neg, r.g))
    sz.flush()
    h = int(ops.hash_u64(st.theta).item())
    del st, sz
    torch.cuda.empty_cache()
    res = H.run(H.fullsize_mesh_worker, 2, steps, timeout=600)
    for rank, recs, hr in res:
        assert recs == want, rank
        assert hr == h, rank


def test_13b_lazy_graph_equals_eager_bit_exact():
    """BASELINE config #3's model (OPT-13B shape, hd 128, T = 2048, B = 1;
    13.1 G parameters, ~105 GB on the device): lazy + graph == eager, one
    store at a time."""
    cfg = opt_config("opt-13b", 2048)
    seeds = iteration_seeds(5, 2)
    batches = [make_batch(cfg, 1, 11 + j) for j in range(2)]
    a = DeviceStore(cfg, 7, init="philox")
    recs = [zo.mezo_step(a, batches[j], zo.ZoHyper(EPS, LR), s, iteration=j + 1) for j, s in enumerate(seeds)]
    ha = int(ops.hash_u64(a.theta).item())
    del a
    torch.cuda.empty_cache()
    b = DeviceStore(cfg, 7, init="philox")
    sz = zo.StreamingZo(b, zo.ZoHyper(EPS, LR))
    for j, s in enumerate(seeds):
        r = sz.step(batches[j], s)
        assert (r.loss_pos, r.loss_neg, r.g) == (recs[j].loss_pos, recs[j].loss_neg, recs[j].g)
        assert np.isfinite([r.loss_pos, r.loss_neg, r.g]).all()
    sz.flush()
    assert int(ops.hash_u64(b.theta).item()) == ha
    del b, sz
    torch.cuda.empty_cache()
