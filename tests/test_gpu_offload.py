"""The ZO2 offload runtime on the GPU (mirror of pkg/tests/test_offload.py):
streamed == serial == resident, bit-exact; the host master lags one update;
U/C/O overlap; sliced upload/offload across ranks (gloo, one GPU) ==
resident."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2507_03211_b200 import zo  # noqa: E402
from paper_2507_03211_b200.engine import DeviceStore  # noqa: E402
from paper_2507_03211_b200.errors import ProtocolError  # noqa: E402
from paper_2507_03211_b200.model import ModelConfig, make_batch  # noqa: E402
from paper_2507_03211_b200.rng import iteration_seeds  # noqa: E402
from paper_2507_03211_b200.scheduler import HostStore, OffloadedZo  # noqa: E402
from tests import dist_helpers as H  # noqa: E402

EPS, LR = 1e-3, 1e-2
DEEP = ModelConfig(64, 32, 4, 5, 16, "f32")   # 5 streamed blocks through 3 slots


def _resident(cfg, steps, bsz=2, flush=True):
    st = DeviceStore(cfg, 7)
    sz = zo.StreamingZo(st, zo.ZoHyper(EPS, LR))
    recs, thetas = [], []
    for j, s in enumerate(iteration_seeds(9, steps), 1):
        r = sz.step(make_batch(cfg, bsz, 40 + j), s)
        recs.append((r.loss_pos, r.loss_neg, r.g))
        thetas.append(st.theta.cpu().numpy().copy())
    if flush:
        sz.flush()
    return recs, thetas, st.theta.cpu().numpy()


@pytest.mark.parametrize("mode", ["streams", "serial"])
def test_offloaded_equals_resident_bit_exact(mode):
    recs, thetas, final = _resident(DEEP, 4)
    host = HostStore(DEEP, 7)
    rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=2, mode=mode)
    layouts = host.layouts
    for j, s in enumerate(iteration_seeds(9, 4), 1):
        r = rt.step(make_batch(DEEP, 2, 40 + j), s)
        assert (r.loss_pos, r.loss_neg, r.g) == recs[j - 1]
        # host master of streamed blocks == resident master (both lag one update)
        for bl in layouts[1:-1]:
            assert np.array_equal(host.block_buf(bl.block_id).numpy(),
                                  thetas[j - 1][bl.key0:bl.key0 + bl.elem_count])
    rt.flush()
    assert np.array_equal(host.theta.numpy(), final)
    with pytest.raises(ProtocolError):
        rt.flush()


def test_uco_streams_overlap_and_timeline_schema():
    cfg = ModelConfig(1024, 512, 8, 8, 128, "f32")
    host = HostStore(cfg, 7)
    rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=4, mode="streams", trace=True)
    for j, s in enumerate(iteration_seeds(1, 3), 1):
        rt.step(make_batch(cfg, 4, j), s)
    tl = rt.last_timeline
    assert {e["op"] for e in tl} == {"upload", "compute", "offload"}
    assert all(set(e) == {"op", "block_id", "stream", "start", "end"} for e in tl)
    busy = sum(e["end"] - e["start"] for e in tl)
    assert rt.makespan() < busy            # ops on the three streams overlap in time
    rt.flush()


def test_sliced_offload_two_ranks_equals_resident():
    """Two ranks share one host master (shared memory); each uploads its
    slice + all-gathers the rest and writes back only its slice.  The result
    equals the resident ZO-DDP(2) path bit for bit."""
    res = H.run(H.sliced_offload_worker, 2, "mezo", 3)
    assert all(len(r[1]) == 3 for r in res)
    assert np.array_equal(res[0][2], res[1][2])
    ddp = H.run(H.gpu_strategy_worker_theta, 2, "ddp", 3)
    assert [r[2] for r in res[0][1]] == [r[2] for r in ddp[0][1]]
    assert np.array_equal(res[0][2], ddp[0][2])


@pytest.mark.parametrize("init_kind", ["host", "philox"])
def test_hbm_sharded_master_two_ranks_equals_resident(init_kind):
    """the fp32 master sharded over 2 ranks' HBM (each rank
    holds ceil(P_blk/2) of every block), blocks reassembled by all-gather,
    own slice written back: records and the final master equal the resident
    ZO-DDP(2) run bit for bit, and each rank holds half the master."""
    res = H.run(H.sharded_worker, 2, "mezo", 3, init_kind)
    want_init = DeviceStore(DEEP, 7, init=init_kind).theta.cpu().numpy()
    for r in res:
        assert np.array_equal(r[3], want_init)
        assert r[4] <= (want_init.size // 2 + 8 * len(DeviceStore(DEEP, 7).layouts)) * 4
    assert np.array_equal(res[0][2], res[1][2])
    if init_kind == "host":
        ddp = H.run(H.gpu_strategy_worker_theta, 2, "ddp", 3)
        assert [r[2] for r in res[0][1]] == [r[2] for r in ddp[0][1]]
        assert np.array_equal(res[0][2], ddp[0][2])


@pytest.mark.parametrize("world,sharded", [(2, False), (4, False), (4, True)])
def test_direction_aware_bf16_redistribution_equals_fp32(world, sharded):
    """SURVEY 8e direction-aware exchange: each rank updates and perturbs its
    own slice for both directions and receives only its direction's bf16
    slices.  Records and the final master equal the fp32 all-gather
    redistribution bit for bit (2D mesh, host or HBM-sharded master, slices
    that are not multiples of 4 and vectors split across ranks), with half
    the per-step parameter bytes received."""
    fp = H.run(H.sliced_dir_worker, world, "fp32", 3, sharded, "none", "2d")
    bf = H.run(H.sliced_dir_worker, world, "bf16", 3, sharded, "none", "2d")
    for a, b in zip(fp, bf):
        assert a[1] == b[1]
        assert np.array_equal(a[2], b[2])
    for r in range(world):
        assert [x[2] for x in fp[r][1]] == [x[2] for x in fp[0][1]]      # one g (losses are per group)
        assert np.array_equal(fp[r][2], fp[0][2])
        p32, p16 = fp[r][3]["param"], bf[r][3]["param"]
        assert p16 * 2 <= p32 * 1.01, (p16, p32)


def test_bf16_redistribution_needs_one_direction_per_rank():
    from paper_2507_03211_b200.errors import ConfigurationError

    host = HostStore(DEEP, 7)
    with pytest.raises(ConfigurationError):
        OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=2, redistribute="bf16")
    with pytest.raises(ConfigurationError):
        OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=2, redistribute="fp16")


@pytest.mark.parametrize("mode", ["streams", "serial"])
def test_split16_compressed_offload_equals_resident(mode):
    """the fp32 master of streamed blocks as hi / lo 16-bit
    planes (hi over PCIe, lo in HBM).  Records every step, the host master
    rebuilt by sync_host (lagging one update, like the uncompressed path) and
    the flushed master equal the resident run bit for bit; PCIe bytes halve."""
    recs, thetas, final = _resident(DEEP, 4)
    host = HostStore(DEEP, 7)
    rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=2, mode=mode, compress="split16")
    plain = OffloadedZo(HostStore(DEEP, 7), zo.ZoHyper(EPS, LR), batch=2, mode=mode)
    assert [2 * b for b in rt.pcie_bytes_per_step()] == list(plain.pcie_bytes_per_step())
    for j, s in enumerate(iteration_seeds(9, 4), 1):
        r = rt.step(make_batch(DEEP, 2, 40 + j), s)
        assert (r.loss_pos, r.loss_neg, r.g) == recs[j - 1]
        rt.sync_host()
        for bl in host.layouts[1:-1]:
            assert np.array_equal(host.block_buf(bl.block_id).numpy(),
                                  thetas[j - 1][bl.key0:bl.key0 + bl.elem_count])
    rt.flush()
    assert np.array_equal(host.theta.numpy(), final)


@pytest.mark.parametrize("world,redistribute,strategy", [(2, "fp32", "ddp"), (4, "bf16", "2d")])
def test_split16_sliced_offload_equals_uncompressed(world, redistribute, strategy):
    """Compression composes with the sliced schedule (each rank keeps the lo
    plane of its own slices) and with the bf16 exchange: bit-identical."""
    a = H.run(H.sliced_dir_worker, world, redistribute, 3, False, "none", strategy)
    b = H.run(H.sliced_dir_worker, world, redistribute, 3, False, "split16", strategy)
    for x, y in zip(a, b):
        assert x[1] == y[1]
        assert np.array_equal(x[2], y[2])
        assert [2 * v for v in y[3]["pcie"]] == list(x[3]["pcie"])


def test_split16_rejects_sharded_master_and_unknown_modes():
    from paper_2507_03211_b200.errors import ConfigurationError
    from paper_2507_03211_b200.sharded import ShardStore

    with pytest.raises(ConfigurationError):
        OffloadedZo(ShardStore(DEEP, None, 7), zo.ZoHyper(EPS, LR), batch=2, compress="split16")
    with pytest.raises(ConfigurationError):
        OffloadedZo(HostStore(DEEP, 7), zo.ZoHyper(EPS, LR), batch=2, compress="fp8")


def test_hbm_sharded_single_rank_equals_resident():
    from paper_2507_03211_b200.sharded import ShardStore

    recs, _, final = _resident(DEEP, 3)
    shards = ShardStore(DEEP, None, 7)
    rt = OffloadedZo(shards, zo.ZoHyper(EPS, LR), batch=2)
    for j, s in enumerate(iteration_seeds(9, 3), 1):
        r = rt.step(make_batch(DEEP, 2, 40 + j), s)
        assert (r.loss_pos, r.loss_neg, r.g) == recs[j - 1]
    rt.flush()
    assert np.array_equal(shards.gather_master(), final)


def test_offload_flush_then_continue_and_single_block():
    """test_offload.py: flush, keep stepping, flush again == resident; and a
    one-transformer-block model degenerates to a valid schedule."""
    for cfg in (DEEP, ModelConfig(64, 32, 4, 1, 16, "f32")):
        recs, _, final = _resident(cfg, 4, flush=False)
        st = DeviceStore(cfg, 7)
        sz = zo.StreamingZo(st, zo.ZoHyper(EPS, LR))
        host = HostStore(cfg, 7)
        rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=2)
        for j, s in enumerate(iteration_seeds(9, 4), 1):
            batch = make_batch(cfg, 2, 40 + j)
            a, b = sz.step(batch, s), rt.step(batch, s)
            assert (a.loss_pos, a.loss_neg, a.g) == (b.loss_pos, b.loss_neg, b.g) == recs[j - 1]
            if j == 2:
                sz.flush()
                rt.flush()
                assert np.array_equal(host.theta.numpy(), st.theta.cpu().numpy())
        sz.flush()
        rt.flush()
        assert np.array_equal(host.theta.numpy(), st.theta.cpu().numpy())


def test_streamed_peak_is_independent_of_depth():
    """test_offload.py:187-194 in bytes: the device footprint of the offload
    runtime is the persistent embedding / head + 3 block slots, so doubling
    the number of streamed blocks does not raise the allocation peak."""
    peaks = []
    for n in (4, 8):
        cfg = ModelConfig(256, 128, 4, n, 32, "f32")
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        rt = OffloadedZo(HostStore(cfg, 7), zo.ZoHyper(EPS, LR), batch=2)
        for j, s in enumerate(iteration_seeds(3, 2), 1):
            rt.step(make_batch(cfg, 2, j), s)
        rt.flush()
        peaks.append(torch.cuda.max_memory_allocated() - base)
        del rt
    blk = (12 * 128 * 128 + 13 * 128) * 4
    assert abs(peaks[1] - peaks[0]) < blk          # no growth with depth


@pytest.mark.parametrize("k", [2, 5])
def test_partially_resident_offload_equals_resident(k):
    """OffloadedZo(resident_blocks=k): the first k transformer blocks stay in
    HBM (uploaded once), only the rest stream -- records and the flushed host
    master equal the resident path bit for bit, and the streamed bytes drop."""
    recs, _, final = _resident(DEEP, 3)
    host = HostStore(DEEP, 7)
    rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=2, resident_blocks=k)
    for j, s in enumerate(iteration_seeds(9, 3), 1):
        r = rt.step(make_batch(DEEP, 2, 40 + j), s)
        assert (r.loss_pos, r.loss_neg, r.g) == recs[j - 1]
    assert rt.uploaded_params == 3 * sum(host.layouts[b].elem_count for b in rt.wids)
    rt.flush()
    assert np.array_equal(host.theta.numpy(), final)


def test_execute_sliced_upload_offload_bytes_and_divergence_guard():
    """pkg/tests/test_comm.py:188-207 on device replicas: every replica equals
    the host buffer after the two-phase upload, the offload reassembles it
    exactly, a diverged replica raises ConsistencyError, and a layout of the
    wrong size is a ConfigurationError."""
    from paper_2507_03211_b200.errors import ConfigurationError, ConsistencyError
    from paper_2507_03211_b200.scheduler import SliceLayout, execute_sliced_offload, execute_sliced_upload

    buf = np.random.default_rng(0).normal(size=1000)
    lay = SliceLayout.build(0, 1000, 4)
    replicas = execute_sliced_upload(buf, lay)
    assert all(np.array_equal(r.cpu().numpy(), buf) for r in replicas)
    out = np.empty_like(buf)
    execute_sliced_offload(replicas, lay, out)
    assert np.array_equal(out, buf)
    replicas[1][3] += 1e-12
    with pytest.raises(ConsistencyError):
        execute_sliced_offload(replicas, lay, out)
    with pytest.raises(ConfigurationError):
        execute_sliced_upload(buf[:999], lay)


def test_execute_sliced_transfer_through_store_layouts():
    """pkg/tests/test_comm.py:233-241: every block of a store round-trips
    through its fixed thread-aligned layout unchanged."""
    from paper_2507_03211_b200.scheduler import apply_thread_aligned_layout, execute_sliced_offload, \
        execute_sliced_upload

    host = HostStore(DEEP, 7)
    before = host.theta.clone()
    apply_thread_aligned_layout(host, 4)
    for bl in host.layouts:
        lay = host.slice_plan["layouts"][bl.block_id]
        replicas = execute_sliced_upload(host.block_buf(bl.block_id), lay)
        execute_sliced_offload(replicas, lay, host.block_buf(bl.block_id))
    assert torch.equal(host.theta, before)


@pytest.mark.parametrize("mode", ["events", "threads", "serial"])
def test_reference_constructor_form(mode):
    """OffloadedZo(store, hyper, capacity=None, cost=None, mode=...) exactly as
    the reference's tests call it (pkg/tests/test_offload.py:118-241): no batch
    argument (sized by the first step), simulated executors mapped to real
    streams, the cost model accepted and unused; same records as resident."""
    recs, _, final = _resident(DEEP, 3)
    host = HostStore(DEEP, 7)
    rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), cost=object(), mode=mode)
    for j, s in enumerate(iteration_seeds(9, 3), 1):
        r = rt.step(make_batch(DEEP, 2, 40 + j), s)
        assert (r.loss_pos, r.loss_neg, r.g) == recs[j - 1]
    rt.flush()
    assert np.array_equal(host.theta.numpy(), final)
    with pytest.raises(ProtocolError):
        OffloadedZo(HostStore(DEEP, 7), zo.ZoHyper(EPS, LR), mode="bogus")


def test_capacity_bound_run_and_too_small_capacity():
    """pkg/tests/test_offload.py:208-215: a byte capacity that holds the
    persistent blocks + 3 streamed blocks runs (and equals resident); one that
    cannot hold two streamed slots is a ConfigurationError, not a crash."""
    from paper_2507_03211_b200.errors import ConfigurationError
    from paper_2507_03211_b200.model import model_layout

    recs, _, final = _resident(DEEP, 2)
    lay = model_layout(DEEP)
    per = lay[1].elem_count * 8
    persistent = (lay[0].elem_count + lay[-1].elem_count) * 8
    host = HostStore(DEEP, 7)
    rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), capacity=persistent + 3 * per)
    assert len(rt.wids) >= 2 and len(rt.slots) >= 2
    for j, s in enumerate(iteration_seeds(9, 2), 1):
        r = rt.step(make_batch(DEEP, 2, 40 + j), s)
        assert (r.loss_pos, r.loss_neg, r.g) == recs[j - 1]
    rt.flush()
    assert np.array_equal(host.theta.numpy(), final)
    big = OffloadedZo(HostStore(DEEP, 7), zo.ZoHyper(EPS, LR), capacity=persistent + 10 * per)
    assert big.wids == []                      # everything fits: nothing streams
    with pytest.raises(ConfigurationError):
        OffloadedZo(HostStore(DEEP, 7), zo.ZoHyper(EPS, LR), capacity=persistent + per)


def test_sliced_offload_divergence_guard():
    """comm.py:336-340 in the distributed schedule (OffloadedZo(verify=True)):
    diverged block replicas are refused before their slices are written
    back, on every rank; verify is rejected where full replicas do not exist."""
    from paper_2507_03211_b200.errors import ConfigurationError

    res = H.run(H.verify_offload_worker, 2)
    assert all(r[1] for r in res) and all(r[2] for r in res)
    with pytest.raises(ConfigurationError):
        OffloadedZo(HostStore(DEEP, 7), zo.ZoHyper(EPS, LR), batch=2, verify=True)


# ---------------------------------------------------------------------------
# parity with the REAL reference's recorded OffloadedZo runs (tests/golden,
# zosim's OffloadedZo.step / flush, scheduler.py:243-283, 393-410)
# ---------------------------------------------------------------------------
GOLDEN_F32 = ["tiny32", "ragged32", "mid32", "wide32"]     # (tiny64 is an f64 store: the device master is fp32)


def _golden_cfg(golden, name):
    c = next(c for c in golden["_meta"]["cases"] if c["name"] == name)
    return ModelConfig(c["vocab"], c["d"], c["heads"], c["n_blocks"], c["seq"], "f32"), c["batch"], c["steps"]


def _zmax(om, seeds):
    from oracle import zo_oracle as O

    return max(float(np.abs(np.concatenate(O.z_stream(s, om.sizes))).max()) for s in seeds)


@pytest.mark.parametrize("mode", ["streams", "serial"])
@pytest.mark.parametrize("name", GOLDEN_F32)
def test_offload_oracle_f32_matches_reference_offload_run(name, mode, golden):
    """OffloadedZo with the reference's z injected and the fp32 parity
    forward reproduces zosim's recorded OffloadedZo trajectory: losses to
    1e-6, g to 1e-4 relative; the host master after K steps (one update
    behind, test_offload.py:130-150) is within lr*|dg|*max|z| per step of the
    reference's unflushed buffers, and after flush of its final weights."""
    from oracle import zo_oracle as O
    from paper_2507_03211_b200.rng import RngStateManager

    cfg, bsz, steps = _golden_cfg(golden, name)
    host = HostStore(cfg, 7)
    rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=bsz, mode=mode, mgr=RngStateManager("oracle"),
                     precision="f32")
    ref = golden[f"{name}/offload"]
    seeds = [int(np.uint64(s)) for s in golden[f"{name}/seeds"].tolist()]
    dg = []
    for j, s in enumerate(seeds, 1):
        from paper_2507_03211_b200.model import Batch
        got = rt.step(Batch(golden[f"{name}/ids/{j}"], golden[f"{name}/tgt/{j}"]), s)
        lp, ln, g = ref[j - 1]
        assert abs(got.loss_pos - lp) <= 1e-6 and abs(got.loss_neg - ln) <= 1e-6, (j, got, ref[j - 1])
        assert abs(got.g - g) <= 1e-4 * max(1.0, abs(g)), (got.g, g)
        dg.append(abs(got.g - g))
    om = O.Model(cfg.vocab_size, cfg.d_model, cfg.n_heads, cfg.n_blocks, cfg.seq_len, init_seed=7)
    bound = steps * LR * max(dg) * _zmax(om, seeds) + 1e-6
    rt.sync_host()
    for bl in host.layouts:
        want = golden[f"{name}/lazy_unflushed/{bl.block_id}"]
        assert float(np.abs(host.block_buf(bl.block_id).numpy().astype(np.float64) - want).max()) <= bound
    rt.flush()
    for bl in host.layouts:
        want = golden[f"{name}/final/{bl.block_id}"]
        assert float(np.abs(host.block_buf(bl.block_id).numpy().astype(np.float64) - want).max()) <= bound


@pytest.mark.parametrize("name", GOLDEN_F32)
def test_offload_teacher_forced_reproduces_reference_buffers_and_checksum(name, golden):
    """With the reference's own g fed back as ``g_prev`` (the attribute the
    reference's next step and flush apply, scheduler.py:346-349, 393-410),
    the offload runtime's host master is the reference's bit for bit: the
    unflushed buffers after K steps equal golden ``lazy_unflushed`` and the
    flushed store's SHA-256 equals golden ``offload_sha``."""
    from paper_2507_03211_b200.model import Batch
    from paper_2507_03211_b200.rng import RngStateManager

    cfg, bsz, steps = _golden_cfg(golden, name)
    host = HostStore(cfg, 7)
    rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=bsz, mgr=RngStateManager("oracle"), precision="f32")
    ref = golden[f"{name}/offload"]
    for j, s in enumerate(golden[f"{name}/seeds"].tolist(), 1):
        got = rt.step(Batch(golden[f"{name}/ids/{j}"], golden[f"{name}/tgt/{j}"]), int(np.uint64(s)))
        assert abs(got.loss_pos - ref[j - 1][0]) <= 1e-6 and abs(got.loss_neg - ref[j - 1][1]) <= 1e-6
        rt.g_prev = float(ref[j - 1][2])
    rt.sync_host()
    for bl in host.layouts:
        assert np.array_equal(host.block_buf(bl.block_id).numpy(), golden[f"{name}/lazy_unflushed/{bl.block_id}"])
    rt.flush()
    assert host.checksum() == str(golden[f"{name}/offload_sha"])
    assert host.checksum() == str(golden[f"{name}/streaming_sha"])


def test_offload_oracle_bf16_production_kernels_within_stated_bound(golden):
    """The production (bf16 tcgen05) offload path with the reference's z:
    losses within the bf16 bound of the recorded OffloadedZo run."""
    from paper_2507_03211_b200.model import Batch
    from paper_2507_03211_b200.rng import RngStateManager

    cfg, bsz, steps = _golden_cfg(golden, "mid32")
    rt = OffloadedZo(HostStore(cfg, 7), zo.ZoHyper(EPS, LR), batch=bsz, mgr=RngStateManager("oracle"))
    ref = golden["mid32/offload"]
    for j, s in enumerate(golden["mid32/seeds"].tolist(), 1):
        got = rt.step(Batch(golden[f"mid32/ids/{j}"], golden[f"mid32/tgt/{j}"]), int(np.uint64(s)))
        assert abs(got.loss_pos - ref[j - 1][0]) <= 2e-3 and abs(got.loss_neg - ref[j - 1][1]) <= 2e-3
    rt.flush()


def test_no_slots_when_every_block_is_resident():
    """plan / constructor: with every transformer block resident nothing
    streams, so no slot is allocated, and results still equal the
    resident path; a budget below two slots is a MemoryCapacityError."""
    from paper_2507_03211_b200.errors import MemoryCapacityError
    from paper_2507_03211_b200.scheduler import plan_residency

    recs, _, final = _resident(DEEP, 2)
    host = HostStore(DEEP, 7)
    rt = OffloadedZo(host, zo.ZoHyper(EPS, LR), batch=2, resident_blocks=DEEP.n_blocks)
    assert rt.slots == []
    for j, s in enumerate(iteration_seeds(9, 2), 1):
        r = rt.step(make_batch(DEEP, 2, 40 + j), s)
        assert (r.loss_pos, r.loss_neg, r.g) == recs[j - 1]
    rt.flush()
    assert np.array_equal(host.theta.numpy(), final)
    P = 12 * 32 * 32 + 13 * 32                    # one DEEP transformer block
    with pytest.raises(MemoryCapacityError):
        plan_residency(DEEP, int(1.5 * P * 8))


@pytest.mark.parametrize("redistribute,world,sharded", [("fp32", 2, False), ("bf16", 2, False), ("bf16", 4, True),
                                                        ("fp32", 4, True)])
def test_copy_engine_data_plane_equals_collective(redistribute, world, sharded):
    """The copy-engine data plane (peers' slot / staging buffers mapped once
    through CUDA IPC, slices pulled with cudaMemcpyAsync between two host
    barriers) moves the same bytes as the collective plane: records and the
    flushed master bit for bit, fp32 all-gather and bf16 exchange, host or
    HBM-sharded master (gloo ranks sharing one GPU)."""
    a = H.run(H.sliced_dir_worker, world, redistribute, 3, sharded, "none", "2d")
    b = H.run(H.sliced_dir_ce_worker, world, redistribute, 3, sharded, "2d")
    for x, y in zip(a, b):
        assert x[1] == y[1]
        assert np.array_equal(x[2], y[2])
        assert x[3]["param"] == y[3]["param"]          # same accounted bytes
        assert x[3]["ce_exchanges"] == 0 and y[3]["ce_exchanges"] > 0
