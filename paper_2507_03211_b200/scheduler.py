"""Block-streaming ZO runtime with CPU parameter offload (mirror of
src/zosim/scheduler.py:201-423, the ZO2 schedule of Alg. 3).

The fp32 master lives in pinned host memory (HostStore).  The embedding and
the LM head stay device-resident (scheduler.py:231-239); transformer blocks
stream through ``n_slots`` device slots.  Three real CUDA streams replace the
reference's simulated U / C / O queues (scheduler.py:131-198):

  U(i)  upload stream    H2D copy of block i's fp32 master into a free slot
                         (with N ranks: each rank copies its 1/N slice over its
                         own PCIe link, then an all-gather over NVLink fills the
                         rest -- comm.py:314-328)
  C(i)  compute stream   fused update_{j-1} + perturb_j pass on the slot, then
                         both directional forwards of block i
  O(i)  offload stream   D2H of the updated master (with N ranks: own slice
                         only -- comm.py:331-342)

Event edges reproduce the reference's op graph (scheduler.py:285-322): C(i)
waits U(i) and follows C(i-1) on its stream; O(i) waits C(i); U(i+n_slots)
waits O(i) (slot reuse), so in steady state O(i-1) / C(i) / U(i+1) overlap.
The update of iteration j is applied to each block on the device right before
it is perturbed in iteration j+1 (the host master lags one update,
test_offload.py:130-150); ``flush`` applies the last one.

With one direction per rank (PertP / 2D) and ``redistribute="bf16"`` the
exchange is the direction-aware one of SURVEY 8e: U(i) is the own fp32 slice
only; C(i) updates that slice and writes both directions' perturbed values
for it (bf16 weights in key order, fp32 vectors), every rank receives only
its own direction's bf16 slices from the peers (half the NVLink bytes of the
fp32 all-gather), and a strided copy lays them out as the GEMM operands.
The perturbed values still come from the fp32 master, so the result is
bit-identical to the fp32 redistribution.

``compress="split16"`` (transfer compression) halves the
PCIe bytes of every streamed block: the fp32 master is kept as two exact
16-bit planes, bits(theta) = hi << 16 | lo.  The hi plane (the bf16
truncation) lives in pinned host memory and is what U(i) / O(i) move; the lo
plane stays in HBM (2 B/param of the streamed blocks, or of this rank's
slices); ``zo_planes_join`` / ``zo_planes_split`` rebuild / split the fp32
block on the device, so every kernel sees the same fp32 values and the run
is bit-identical to the uncompressed one.  The host fp32 master of streamed
blocks is rebuilt by ``sync_host`` / ``flush``.
"""

from __future__ import annotations

import hashlib
import time
from typing import NamedTuple

import numpy as np
import torch

from . import _lib as L
from . import ops
from .engine import MINUS, PLUS, SegTable, ShadowPlan, Workspace, block_extent
from .errors import ConfigurationError, ConsistencyError, MemoryCapacityError, ProtocolError
from .model import EMBEDDING, HEAD, TRANSFORMER, Batch, ModelConfig, init_block_host, model_layout
from .rng import RngStateManager
from .zo import ZoHyper, ZoStep, _u64_as_i64

UPLOAD, COMPUTE, OFFLOAD = "upload", "compute", "offload"


class HostStore:
    """The model's fp32 master in pinned host memory, in key order
    (the reference's ParamStore, model.py:160-200).

    ``shared``: path of a shared-memory file (e.g. under /dev/shm) holding the
    master, so the one-process-per-GPU ranks of a node all see ONE host master
    -- each rank uploads / writes back only its own slices (comm.py:314-342).
    The creator (``init`` != "attach") fills it; other ranks attach with
    init="attach" after a barrier.  The mapping is page-locked with
    cudaHostRegister so H2D/D2H run at full PCIe rate."""

    def __init__(self, config: ModelConfig, init_seed: int = 7, init: str = "host", device=None,
                 shared: str | None = None, numa: bool = False):
        """numa: bind this process to the CPUs of its GPU's NUMA node before
        the master is allocated, so the pinned pages are node-local
        (sharded.bind_to_gpu_numa)."""
        config.validate()
        self.config, self.init_seed = config, init_seed
        self.layouts = model_layout(config)
        self.total_params = sum(b.elem_count for b in self.layouts)
        self.shared = shared
        self.numa = None
        if numa:
            from .sharded import bind_to_gpu_numa

            self.numa = bind_to_gpu_numa(torch.device(device or f"cuda:{torch.cuda.current_device()}"))
        if shared is None:
            self.theta = torch.empty(self.total_params, dtype=torch.float32, pin_memory=True)
        else:
            import os

            if init != "attach":
                with open(shared, "wb") as f:
                    f.truncate(self.total_params * 4)
            self.theta = torch.from_file(shared, shared=True, size=self.total_params, dtype=torch.float32)
            rc = torch.cuda.cudart().cudaHostRegister(self.theta.data_ptr(), self.total_params * 4, 0)
            self._registered = int(rc) == 0
            _ = os
        if init == "attach":
            return
        if init == "host":
            for bl in self.layouts:
                self.block_buf(bl.block_id).copy_(torch.from_numpy(init_block_host(config, bl, init_seed)))
        elif init == "philox":
            from .engine import DeviceStore  # noqa: F401  (library / device checks)

            dev = torch.device(device or f"cuda:{torch.cuda.current_device()}")
            seed = (0x1A2B3C4D << 32) ^ int(init_seed)
            chunk = 1 << 26
            for bl in self.layouts:
                for name in bl.names:
                    k, n = bl.key(name), bl.size(name)
                    dst = self.theta[k:k + n]
                    if name.endswith("_g"):
                        dst.fill_(1.0)
                    elif name.startswith("b") or name.endswith("_b"):
                        dst.zero_()
                    else:
                        for o in range(0, n, chunk):
                            m = min(chunk, n - o)
                            z = torch.empty(m, dtype=torch.float32, device=dev)
                            L.call("zo_philox_normals", seed, k + o, m, z.data_ptr(), L.stream_ptr())
                            dst[o:o + m].copy_(z.mul_(0.02))        # straight into the pinned master
        elif init != "none":
            raise ConfigurationError(f"unknown init {init!r}")

    def block_buf(self, bid: int) -> torch.Tensor:
        bl = self.layouts[bid]
        return self.theta[bl.key0:bl.key0 + bl.elem_count]

    def close(self):
        if self.shared is not None and getattr(self, "_registered", False):
            torch.cuda.cudart().cudaHostUnregister(self.theta.data_ptr())
            self._registered = False

    def checksum(self) -> str:
        h = hashlib.sha256()
        for bl in self.layouts:
            h.update(self.block_buf(bl.block_id).numpy().tobytes())
        return h.hexdigest()


class BlockSlot:
    """Device buffers for one block: fp32 master copy + per-direction shadows,
    exposing the same wview / vview / theta_ptr interface as DeviceStore so
    the forward launch plans can read a streamed block."""

    def __init__(self, plan: ShadowPlan, layouts, template_bid: int, dirs, device, pad_to: int = 0,
                 shadows: bool = True):
        self.plan, self.layouts = plan, layouts
        bl = layouts[template_bid]
        n = max(bl.elem_count, pad_to)
        self.theta = torch.zeros(n, dtype=torch.float32, device=device)
        self.wsh, self.vsh = [None, None], [None, None]
        if shadows and plan.views[template_bid]:     # (a real-OPT embedding has the tied head's shadow)
            wlo, whi, vlo, vhi = block_extent(plan, template_bid)
            for s in dirs:
                self.wsh[s] = torch.zeros(whi - wlo, dtype=torch.bfloat16, device=device)
                self.vsh[s] = torch.zeros(vhi - vlo, dtype=torch.float32, device=device)
        self.bid = template_bid

    def bind(self, bid: int):
        self.bid = bid
        return self

    @property
    def key0(self) -> int:
        return self.layouts[self.bid].key0

    def theta_ptr(self, key: int) -> int:
        return self.theta.data_ptr() + 4 * (key - self.key0)

    def wview(self, s: int, bid: int, name: str):
        b, off, rows, cols, ld = self.plan.views[bid][name]
        wlo, _, vlo, _ = block_extent(self.plan, bid)
        if b == "v":                      # f32 parity mode: weights live in the fp32 shadow
            return self.vsh[s][off - vlo:off - vlo + rows * ld].view(rows, ld), rows, cols
        return self.wsh[s][off - wlo:off - wlo + rows * ld].view(rows, ld), rows, cols

    def vview(self, s: int, bid: int, name: str) -> torch.Tensor:
        b, off, rows, cols, ld = self.plan.views[bid][name]
        vlo = block_extent(self.plan, bid)[2]
        return self.vsh[s][off - vlo:off - vlo + cols]


def rebased_table(plan: ShadowPlan, bid: int, device) -> SegTable:
    """The block's perturb segments with shadow offsets relative to its slot."""
    return SegTable(rebased_segments(plan, bid), device)


def rebased_segments(plan: ShadowPlan, bid: int) -> list:
    if plan.views[bid]:
        wlo, _, vlo, _ = block_extent(plan, bid)
    else:
        wlo = vlo = 0
    segs = []
    for (src, rows, cols, dst, ld, kind) in plan.segments[bid]:
        if kind == L.ZO_SHADOW_BF16:
            dst -= wlo
        elif kind == L.ZO_SHADOW_F32:
            dst -= vlo
        segs.append((src, rows, cols, dst, ld, kind))
    return segs


# -----------------------------------------------------------------------------
# slicing (comm.py:106-119, 314-358)
# -----------------------------------------------------------------------------

class Slice(NamedTuple):
    """One contiguous slice of a block (comm.py's Slice: owner, offset, length)."""
    owner: int
    offset: int
    length: int


class SliceLayout:
    """Ceil-width slices, owner i = rank i, last one may be short
    (comm.py:106-119)."""

    def __init__(self, block_id: int, total: int, n: int):
        if n < 1:
            raise ConfigurationError(f"slice count must be >= 1, got {n}")
        self.block_id, self.total, self.n = block_id, total, n
        self.width = -(-total // n)
        self.slices = []
        off = 0
        for owner in range(n):
            length = max(min(self.width, total - off), 0)
            self.slices.append(Slice(owner, off, length))
            off += length

    def __eq__(self, other):
        return isinstance(other, SliceLayout) and (self.block_id, self.total, self.n, self.slices) == (
            other.block_id, other.total, other.n, other.slices)

    __hash__ = None

    @classmethod
    def build(cls, block_id: int, total: int, n: int) -> "SliceLayout":
        return cls(block_id, total, n)


def sliced_upload_time(total: int, n: int, host_bw: float, peer_bw: float) -> float:
    """The reference's analytic redistribution cost (comm.py:250-256), the
    model the measured per-block upload is compared against:
    T_comm = ceil(M/n)/BW_host + (M - ceil(M/n))/BW_peer."""
    width = -(-total // n)
    return width / host_bw + (total - width) / peer_bw


def apply_thread_aligned_layout(store, n: int) -> dict:
    """Fix per-block slice boundaries once (comm.py:345-358); changing n later
    is a ProtocolError."""
    plan = getattr(store, "slice_plan", None)
    if plan is not None:
        if plan["n"] != n:
            raise ProtocolError(f"slice layout already fixed for n={plan['n']}; changing to n={n} requires "
                                "re-initialization")
        return plan
    store.slice_plan = {"n": n, "layouts": {bl.block_id: SliceLayout(bl.block_id, bl.elem_count, n)
                                            for bl in store.layouts}}
    return store.slice_plan


def sliced_upload(host_block: torch.Tensor, slot_theta: torch.Tensor, layout: SliceLayout, fabric, rank: int,
                  stream=None, gather: bool = True):
    """Phase 1: this rank's slice host -> device over its PCIe link; phase 2:
    the peers' slices arrive by an all-gather of the slot (NVLink), never
    from the host (comm.py:314-328).  slot_theta is padded to n * width."""
    owner, off, ln = layout.slices[rank]
    w = layout.width
    with torch.cuda.stream(stream) if stream is not None else _null():
        if ln:
            slot_theta[rank * w:rank * w + ln].copy_(host_block[off:off + ln], non_blocking=True)
        if layout.n > 1 and gather:
            fabric.all_gather_tensor(slot_theta[:layout.n * w], slot_theta[rank * w:(rank + 1) * w], tag="param")


def execute_sliced_upload(host_buf, layout: SliceLayout, devices=None) -> list:
    """comm.py:314-328 for one process driving ``layout.n`` device replicas
    (``devices``: one CUDA device per owner; default: all on the current
    GPU).  Phase 1: each replica pulls its own slice from the host; phase 2:
    the rest comes from the owning replica (device to device -- NVLink peer
    copies between GPUs), never from the host.  ``host_buf``: numpy array or
    tensor (shared, not copied).  Returns the replicas (device tensors)."""
    host = torch.as_tensor(host_buf)
    if host.numel() != layout.total:
        raise ConfigurationError("layout does not match buffer size")
    devs = list(devices) if devices is not None else [torch.device("cuda", torch.cuda.current_device())] * layout.n
    if len(devs) != layout.n:
        raise ConfigurationError(f"need {layout.n} devices, got {len(devs)}")
    reps = [torch.empty(layout.total, dtype=host.dtype, device=d) for d in devs]
    for s in layout.slices:
        if s.length:
            reps[s.owner][s.offset:s.offset + s.length].copy_(host[s.offset:s.offset + s.length])
    for s in layout.slices:
        for dst in range(layout.n):
            if dst != s.owner and s.length:
                reps[dst][s.offset:s.offset + s.length].copy_(reps[s.owner][s.offset:s.offset + s.length])
    for d in set(devs):
        torch.cuda.synchronize(d)
    return reps


def execute_sliced_offload(replicas: list, layout: SliceLayout, host_buf) -> None:
    """comm.py:331-342: each replica writes only its owned slice back, after
    checking that the replicas are bit-identical (ConsistencyError otherwise:
    a diverged replica would reassemble a corrupt block)."""
    from .ops import hash_u64

    ref = replicas[0]
    for r in replicas[1:]:
        same = torch.equal(r, ref) if r.device == ref.device else \
            int(hash_u64(r).item()) == int(hash_u64(ref).item())
        if not same:
            raise ConsistencyError("device replicas diverged; offload would reassemble a corrupt block")
    host = torch.as_tensor(host_buf)
    for s in layout.slices:
        if s.length:
            host[s.offset:s.offset + s.length].copy_(replicas[s.owner][s.offset:s.offset + s.length])


def sliced_offload(slot_theta: torch.Tensor, host_block: torch.Tensor, layout: SliceLayout, rank: int,
                   stream=None):
    """Each rank writes back only its owned slice (comm.py:331-342)."""
    owner, off, ln = layout.slices[rank]
    with torch.cuda.stream(stream) if stream is not None else _null():
        if ln:
            host_block[off:off + ln].copy_(slot_theta[off:off + ln], non_blocking=True)


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def check_slices_identical(fabric, rank: int, slot_theta: torch.Tensor, n: int):
    """Divergence guard before offload (comm.py:336-340)."""
    from .ops import hash_u64

    h = int(hash_u64(slot_theta[:n]).item()) & ((1 << 64) - 1)
    got = list(zip(fabric.all_gather(rank, float(h & 0xFFFFFFFF), tag="checksum"),
                   fabric.all_gather(rank, float(h >> 32), tag="checksum")))
    if len(set(got)) != 1:
        raise ConsistencyError("device replicas diverged; offload would reassemble a corrupt block")


# -----------------------------------------------------------------------------
# the runtime
# -----------------------------------------------------------------------------

class OffloadedZo:
    """ZO2 streaming runtime over one GPU (or one rank of a sliced mesh).

    ``mode``: "streams" (U/C/O overlapped on three CUDA streams) or "serial"
    (everything on one stream; the equivalence oracle, scheduler.py:324-341).
    With ``fabric`` (world N): sliced H2D + all-gather / own-slice D2H, and
    the loss exchange of the strategy in ``strategy`` ("mezo" for both
    directions per rank (ZO-DDP when N > 1), "2d" for one direction per rank).
    """

    def __init__(self, host: HostStore, hyper: ZoHyper, batch: int | None = None, device=None, n_slots: int = 3,
                 mode: str = "streams", fabric=None, strategy: str = "mezo", trace: bool = False,
                 resident_blocks: int = 0, redistribute: str = "fp32", compress: str = "none",
                 capacity: int | None = None, cost=None, verify: bool = False, mgr: RngStateManager | None = None,
                 precision: str = "bf16"):
        """resident_blocks: keep the first k transformer blocks on the device
        for the whole run (uploaded once, written back at flush / sync_host)
        and stream only the rest -- use whatever HBM the model leaves free,
        so only the blocks that do not fit cross PCIe every step.  The
        results are bit-identical for every k (same kernels, same order).

        redistribute: "fp32" (all-gather the fp32 slices; every rank updates
        and perturbs the whole block) or "bf16" (one direction per rank only:
        the direction-aware bf16 exchange described in the module docstring).

        compress: "none" or "split16" (hi / lo 16-bit planes: half the PCIe
        bytes per streamed block, lo kept in device memory; module docstring).

        The reference's constructor form ``OffloadedZo(store, hyper,
        capacity=None, cost=None, mode="events")`` (scheduler.py:209-216) is
        accepted as is: ``batch`` may be omitted (activations are sized by the
        first step's batch); ``capacity`` is the device-memory budget in bytes
        (the reference's MemoryPool capacity) and picks ``resident_blocks`` /
        ``n_slots`` through ``plan_residency`` after the persistent embedding
        and head; ``cost`` is accepted and unused (real streams replace the
        simulated cost model); the simulated executors "events" / "threads"
        map to the real concurrent "streams".

        verify (sliced schedule over a fabric, fp32 redistribution): before a
        rank writes its slice of a streamed block back, the ranks compare a
        64-bit hash of their whole block copy and refuse to offload diverged
        replicas (ConsistencyError; comm.py:336-340).  A host-synchronising
        collective per block, so off by default (a debug guard, like the
        strategies' ``verify``).

        mgr: RngStateManager("oracle") injects the reference's numpy z (the
        whole model's stream per iteration, zo.py:90-125) instead of the
        in-register Philox z; precision="f32" runs the fp32 parity forward
        (SURVEY 8c mode (i)).  Together they reproduce the reference's
        OffloadedZo trajectory (tests/test_gpu_offload.py)."""
        mode = {"events": "streams", "threads": "streams"}.get(mode, mode)
        if mode not in ("streams", "serial"):
            raise ProtocolError(f"unknown scheduler mode {mode!r}")
        self.cost = cost
        if n_slots < 2:
            raise ConfigurationError("need at least 2 block slots")
        self.host, self.hyper, self.mode, self.trace = host, hyper.validate(), mode, trace
        self.mgr = mgr or RngStateManager()
        if precision not in ("bf16", "f32"):
            raise ConfigurationError(f"precision must be 'bf16' or 'f32', got {precision!r}")
        self.precision = precision
        cfg = self.config = host.config
        if precision == "f32" and cfg.arch != "zosim":
            raise ConfigurationError("the f32 parity mode covers the zosim architecture")
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        L.lib()
        self.layouts = host.layouts
        self.plan = ShadowPlan(cfg, self.layouts, f32_weights=precision == "f32")
        self.fabric = fabric
        self.world = fabric.k if fabric is not None else 1
        self.rank = fabric.rank if fabric is not None else 0
        from .strategies import MeshLayout
        self.mesh = MeshLayout("ddp" if strategy == "mezo" else strategy, self.world, self.rank) \
            if fabric is not None else None
        self.dirs = self.mesh.dirs if self.mesh is not None else (PLUS, MINUS)
        if redistribute not in ("fp32", "bf16"):
            raise ConfigurationError(f"redistribute must be 'fp32' or 'bf16', got {redistribute!r}")
        if redistribute == "bf16" and (fabric is None or len(self.dirs) != 1):
            raise ConfigurationError("bf16 redistribution needs a mesh with one direction per rank "
                                     "(strategy 'pertp' or '2d')")
        if redistribute == "bf16" and precision == "f32":
            raise ConfigurationError("the f32 parity mode redistributes fp32 blocks (redistribute='fp32')")
        self.redistribute = redistribute
        if verify and (fabric is None or redistribute == "bf16"):
            raise ConfigurationError("verify compares full block replicas: it needs a fabric and the fp32 "
                                     "redistribution (with bf16 only the own slice is materialised)")
        self.verify = verify
        if compress not in ("none", "split16"):
            raise ConfigurationError(f"compress must be 'none' or 'split16', got {compress!r}")
        if compress == "split16" and getattr(host, "is_sharded", False) and not getattr(host, "on_host", False):
            raise ConfigurationError("transfer compression applies to a host master (the HBM-sharded master "
                                     "has no PCIe leg)")
        self.compress = compress
        if fabric is not None:
            apply_thread_aligned_layout(host, self.world)
        emb, head = self.layouts[0].block_id, self.layouts[-1].block_id
        wids = [bl.block_id for bl in self.layouts if bl.kind == TRANSFORMER]
        if capacity is not None:
            nd = len(self.dirs)
            persistent = sum(self.layouts[b].elem_count for b in (emb, head)) * (4 + 2 * nd)
            per = self.layouts[wids[0]].elem_count * (4 + 2 * nd) if wids else 0
            if wids and capacity - persistent < 2 * per:
                raise MemoryCapacityError(f"device capacity {capacity} B cannot hold the persistent blocks "
                                         f"({persistent} B) and two streamed block slots ({2 * per} B)")
            if wids:
                resident_blocks, n_slots = plan_residency(cfg, capacity - persistent, n_dirs=nd, compress=compress)
        if not 0 <= resident_blocks <= len(wids):
            raise ConfigurationError(f"resident_blocks must be in [0, {len(wids)}], got {resident_blocks}")
        self.resident = wids[:resident_blocks]          # computed in place, never streamed
        self.wids = wids[resident_blocks:]              # streamed through the slots
        pad = lambda bid: (-(-self.layouts[bid].elem_count // self.world)) * self.world  # noqa: E731
        self.persistent = {emb: BlockSlot(self.plan, self.layouts, emb, self.dirs, self.device, pad(emb)),
                           head: BlockSlot(self.plan, self.layouts, head, self.dirs, self.device, pad(head))}
        for bid in self.resident:
            self.persistent[bid] = BlockSlot(self.plan, self.layouts, bid, self.dirs, self.device, pad(bid))
        tpl = self.wids[0] if self.wids else head
        # no streamed block -> no slots (everything is persistent)
        self.slots = [BlockSlot(self.plan, self.layouts, tpl, self.dirs, self.device, pad(tpl))
                      for _ in range(n_slots if self.wids else 0)]
        self._bf16 = {}
        self._phase_ev = []                      # trace: (phase, start event, end event, bytes)
        self.phase_stats = {}                    # trace: phase -> {"ms", "bytes", "n"} summed over steps
        if redistribute == "bf16" and self.wids:
            me = self.dirs[0]
            for slot in self.slots:                   # both directions' vectors, for the peers
                slot.vsh[1 - me] = torch.zeros_like(slot.vsh[me])
            # key-ordered bf16 staging of both directions, shared by the slots
            # (C(i) runs on one stream)
            self._stage = {d: torch.zeros(pad(tpl), dtype=torch.bfloat16, device=self.device) for d in (PLUS, MINUS)}
            self._vgather = torch.zeros(self.world * 2 * self.slots[0].vsh[me].numel(), dtype=torch.float32,
                                        device=self.device)
            self._dir_of = [PLUS if q % 2 == 0 else MINUS for q in range(self.world)]
        self._hi, self._lo = {}, {}
        if compress == "split16" and self.wids:
            self._init_planes()
        self.tables = {bl.block_id: rebased_table(self.plan, bl.block_id, self.device) for bl in self.layouts}
        for bid, slot in self.persistent.items():      # embedding + head stay on the device
            self._upload(bid, slot, None)
        torch.cuda.synchronize()
        self.scal = torch.zeros(4, dtype=torch.int64, device=self.device)
        self.record = torch.zeros(3, dtype=torch.float64, device=self.device)
        self.local = torch.zeros(2, dtype=torch.float64, device=self.device)
        self.gathered = torch.zeros(2 * self.world, dtype=torch.float64, device=self.device)
        self.ws = {s: Workspace(cfg, batch, cfg.seq_len, self.device, f32=precision == "f32")
                   for s in self.dirs} if batch else None
        self._zc = self._zp = None             # oracle mode: this / the previous iteration's z (device f64)
        self.streams = {COMPUTE: torch.cuda.current_stream(self.device)}
        if mode == "streams":
            self.streams[UPLOAD] = torch.cuda.Stream(self.device)
            self.streams[OFFLOAD] = torch.cuda.Stream(self.device)
        else:
            self.streams[UPLOAD] = self.streams[OFFLOAD] = self.streams[COMPUTE]
        self.iteration, self._g_prev, self.last_seed, self._pending = 0, 0.0, None, False
        self.timelines = []
        self.uploaded_params = self.offloaded_params = 0

    @property
    def g_prev(self) -> float:
        return self._g_prev

    @g_prev.setter
    def g_prev(self, g: float) -> None:
        """The reference applies ``self.g_prev`` as the deferred update
        (scheduler.py:346-349 -> dual_forward); replacing it replaces the
        device's lr * g_prev the next fused pass / flush applies."""
        self._g_prev = float(g)
        self.scal[2:3].fill_(int(np.float64(self.hyper.lr * float(g)).view(np.int64)))

    # -- byte movement --------------------------------------------------------------
    def _own(self, bid):
        """(offset, length) of the part of block bid this rank moves over PCIe."""
        if self.fabric is None:
            return 0, self.layouts[bid].elem_count
        _, off, ln = self.host.slice_plan["layouts"][bid].slices[self.rank]
        return off, ln

    def _init_planes(self):
        """Split this rank's part of every streamed block once: lo into HBM,
        hi into pinned host memory."""
        own = {bid: self._own(bid) for bid in self.wids}
        total = sum(ln for _, ln in own.values())
        wmax = max(ln for _, ln in own.values())
        self._hi_pool = torch.empty(total, dtype=torch.int16, pin_memory=True)
        self._lo_pool = torch.empty(total, dtype=torch.int16, device=self.device)
        for slot in self.slots:
            slot.hi_stage = torch.empty(wmax, dtype=torch.int16, device=self.device)
        tmp = torch.empty(wmax, dtype=torch.float32, device=self.device)
        pos = 0
        for bid in self.wids:
            off, ln = own[bid]
            self._hi[bid] = self._hi_pool[pos:pos + ln]
            self._lo[bid] = self._lo_pool[pos:pos + ln]
            pos += ln
            tmp[:ln].copy_(self._host_part(bid))
            ops.planes_split(tmp[:ln], self.slots[0].hi_stage[:ln], self._lo[bid])
            self._hi[bid].copy_(self.slots[0].hi_stage[:ln])
        torch.cuda.synchronize(self.device)

    def pcie_bytes_per_step(self):
        """(H2D, D2H) bytes this rank moves per step for the streamed blocks."""
        if getattr(self.host, "is_sharded", False) and not getattr(self.host, "on_host", False):
            return 0, 0                                  # HBM-sharded master: no PCIe leg
        per = 2 if self.compress == "split16" else 4
        n = sum(self._own(bid)[1] for bid in self.wids)
        return per * n, per * n

    def _host_part(self, bid) -> torch.Tensor:
        """The part of block ``bid``'s master this rank moves over PCIe: the
        whole block (one GPU), its slice of the shared host master, or its
        own per-rank slice (ShardStore)."""
        if getattr(self.host, "is_sharded", False):
            return self.host.slice_of(bid)
        off, ln = self._own(bid)
        return self.host.block_buf(bid)[off:off + ln]

    class _Phase:
        """CUDA-event bracket of one byte movement / compute phase on a stream
        (trace mode only); resolved per step into ``phase_stats``."""

        def __init__(self, rt, name, stream, nbytes):
            self.rt, self.name, self.stream, self.nbytes = rt, name, stream, nbytes

        def __enter__(self):
            if self.rt.trace:
                self.e0 = torch.cuda.Event(enable_timing=True)
                self.e0.record(self.stream)
            return self

        def __exit__(self, *a):
            if self.rt.trace:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(self.stream)
                self.rt._phase_ev.append((self.name, self.e0, e1, self.nbytes))
            return False

    def _phase(self, name, stream, nbytes=0):
        return OffloadedZo._Phase(self, name, stream or torch.cuda.current_stream(self.device), nbytes)

    def _gather_slot(self, bid, slot, stream):
        """Phase 2 of the sliced upload: the peers' fp32 slices over NVLink."""
        if self.fabric is None or self.world == 1:
            return
        w = self.host.slice_plan["layouts"][bid].width
        with torch.cuda.stream(stream) if stream is not None else _null(), \
                self._phase("nvlink_allgather", stream, 4 * (self.world - 1) * w):
            self.fabric.all_gather_tensor(slot.theta[:self.world * w],
                                          slot.theta[self.rank * w:(self.rank + 1) * w], tag="param")

    def _upload(self, bid, slot, stream, gather=None):
        slot.bind(bid)
        if gather is None:      # the bf16 exchange replaces the fp32 all-gather of streamed blocks
            gather = not (self.redistribute == "bf16" and bid in self.wids)
        off, ln = self._own(bid)
        sharded_hbm = getattr(self.host, "is_sharded", False) and not getattr(self.host, "on_host", False)
        with torch.cuda.stream(stream) if stream is not None else _null():
            if bid in self._lo:                          # hi plane over PCIe, joined with the resident lo
                with self._phase("h2d", stream, 2 * ln):
                    slot.hi_stage[:ln].copy_(self._hi[bid], non_blocking=True)
                ops.planes_join(slot.hi_stage[:ln], self._lo[bid], slot.theta[off:off + ln])
            elif ln:
                with self._phase("d2d" if sharded_hbm else "h2d", stream, 4 * ln):
                    slot.theta[off:off + ln].copy_(self._host_part(bid), non_blocking=True)
        if gather:
            self._gather_slot(bid, slot, stream)

    def _offload(self, bid, slot, stream):
        if self.verify and bid in self.wids:
            with torch.cuda.stream(stream) if stream is not None else _null():
                check_slices_identical(self.fabric, self.rank, slot.theta, self.layouts[bid].elem_count)
        off, ln = self._own(bid)
        sharded_hbm = getattr(self.host, "is_sharded", False) and not getattr(self.host, "on_host", False)
        with torch.cuda.stream(stream) if stream is not None else _null():
            if bid in self._lo:                          # split: lo stays, hi goes to the host
                ops.planes_split(slot.theta[off:off + ln], slot.hi_stage[:ln], self._lo[bid])
                with self._phase("d2h", stream, 2 * ln):
                    self._hi[bid].copy_(slot.hi_stage[:ln], non_blocking=True)
            elif ln:                                     # own slice only (comm.py:331-342)
                with self._phase("d2d" if sharded_hbm else "d2h", stream, 4 * ln):
                    self._host_part(bid).copy_(slot.theta[off:off + ln], non_blocking=True)

    # -- compute --------------------------------------------------------------------
    def _perturb(self, bid, slot, flags, stream):
        t, eps = self.tables[bid], self.hyper.epsilon
        sa = PLUS if PLUS in self.dirs else None
        sb = MINUS if MINUS in self.dirs else None
        wa = slot.wsh[PLUS].data_ptr() if sa is not None and slot.wsh[PLUS] is not None else 0
        va = slot.vsh[PLUS].data_ptr() if sa is not None and slot.vsh[PLUS] is not None else 0
        wb = slot.wsh[MINUS].data_ptr() if sb is not None and slot.wsh[MINUS] is not None else 0
        vb = slot.vsh[MINUS].data_ptr() if sb is not None and slot.vsh[MINUS] is not None else 0
        zmode, zc, zp = self._zargs()
        L.check(L.lib().zo_perturb_update(slot.theta.data_ptr(), slot.key0, t.segs.data_ptr(), t.prefix.data_ptr(),
                                          t.n_segs, t.n_tiles, wa, va, wb, vb, +eps, -eps, flags,
                                          self.scal.data_ptr(), zmode, zc, zp, 0, int(stream.cuda_stream)))

    def _update_flag(self):
        """Philox: always request the update (the device pending flag gates
        it, so one launch plan serves every step); oracle z: only when a
        previous iteration's z exists to regenerate the update from."""
        return L.ZO_PU_UPDATE if (not self.mgr.oracle or self._zp is not None) else 0

    def _zargs(self):
        """(zmode, z_cur ptr, z_prev ptr) for the perturb / embedding kernels;
        oracle z tensors hold the whole model's stream (z_key0 = 0)."""
        if not self.mgr.oracle:
            return L.ZO_Z_PHILOX, 0, 0
        return (L.ZO_Z_ORACLE, 0 if self._zc is None else self._zc.data_ptr(),
                0 if self._zp is None else self._zp.data_ptr())

    def _bf16_plan(self, bid):
        """Per streamed block, built once: this rank's slice of the perturb
        segments (bf16 weights -> key-ordered staging, fp32 vectors -> their
        shadow slots), the strided re-layout of the staging into the GEMM
        operands, and the owning rank of every vector shadow element."""
        if bid in self._bf16:
            return self._bf16[bid]
        lay = self.host.slice_plan["layouts"][bid]
        key0, total, w = self.layouts[bid].key0, lay.total, lay.width
        rng = [(key0 + q * w, key0 + min((q + 1) * w, total)) for q in range(self.world)]
        lo, hi = rng[self.rank]
        me = self.dirs[0]
        owner = torch.zeros(self.slots[0].vsh[me].numel(), dtype=torch.int64)
        clipped, relayout = [], []
        for (src, rows, cols, dst, ld, kind) in rebased_segments(self.plan, bid):
            end = src + rows * cols
            if kind == L.ZO_SHADOW_BF16:
                relayout.append((src - key0, rows, cols, dst, ld))
            elif kind == L.ZO_SHADOW_F32:
                if rows > 1 and ld != cols:
                    raise ConfigurationError("bf16 redistribution needs contiguous vector shadows")
                for q, (a, b) in enumerate(rng):
                    a, b = max(src, a), min(end, b)
                    if a < b:
                        owner[dst + a - src:dst + b - src] = q
            a, b = max(src, lo), min(end, hi)
            if a >= b:
                continue
            if kind == L.ZO_SHADOW_BF16:
                clipped.append((a, 1, b - a, a - key0, b - a, kind))
            elif kind == L.ZO_SHADOW_F32:
                clipped.append((a, 1, b - a, dst + a - src, b - a, kind))
            else:
                clipped.append((a, 1, b - a, 0, b - a, kind))
        plan = (SegTable(clipped, self.device), relayout, owner.to(self.device), w)
        self._bf16[bid] = plan
        return plan

    def _perturb_slice(self, bid, slot, flags, stream):
        """Update this rank's slice of the block's master and (with the shadow
        flags) write both directions' perturbed values for it."""
        t = self._bf16_plan(bid)[0]
        eps = self.hyper.epsilon
        L.check(L.lib().zo_perturb_update(slot.theta.data_ptr(), slot.key0, t.segs.data_ptr(), t.prefix.data_ptr(),
                                          t.n_segs, t.n_tiles, self._stage[PLUS].data_ptr(),
                                          slot.vsh[PLUS].data_ptr(), self._stage[MINUS].data_ptr(),
                                          slot.vsh[MINUS].data_ptr(), +eps, -eps, flags, self.scal.data_ptr(),
                                          *self._zargs(), 0, int(stream.cuda_stream)))

    def _redistribute_bf16(self, bid, slot, stream):
        """C(i) prologue of the bf16 exchange: own slice -> both directions,
        peers' slices of this rank's direction in, laid out as GEMM operands."""
        _, relayout, owner, w = self._bf16_plan(bid)
        me = self.dirs[0]
        self._perturb_slice(bid, slot, self._update_flag() | L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B, stream)
        nv = slot.vsh[me].numel()
        with torch.cuda.stream(stream), self._phase("nvlink_exchange", stream, 2 * (self.world - 1) * w
                                                     + 8 * (self.world - 1) * nv):
            self.fabric.exchange_slices(self._stage, me, self._dir_of, w, tag="param")
            vg = self._vgather[:self.world * 2 * nv]
            self.fabric.all_gather_tensor(vg, torch.cat([slot.vsh[PLUS], slot.vsh[MINUS]]), tag="param_vec")
        with torch.cuda.stream(stream):
            slot.vsh[me].copy_(vg.view(self.world, 2, nv)[:, me].gather(0, owner[None])[0])
            stage, wsh = self._stage[me], slot.wsh[me]
            for (s0, rows, cols, d0, ld) in relayout:
                torch.as_strided(wsh, (rows, cols), (ld, 1), d0).copy_(stage[s0:s0 + rows * cols].view(rows, cols))

    def _shadow_flags(self):
        f = 0
        if PLUS in self.dirs:
            f |= L.ZO_PU_SHADOW_A
        if MINUS in self.dirs:
            f |= L.ZO_PU_SHADOW_B
        return f

    def _compute(self, bid, slot, stream):
        """C(i): fused update+perturb of the block, then each direction's forward."""
        if self.redistribute == "bf16" and bid in self.wids:
            self._redistribute_bf16(bid, slot, stream)
        else:
            self._perturb(bid, slot, self._update_flag() | self._shadow_flags(), stream)
        eps = self.hyper.epsilon
        for s in self.dirs:
            loss_out = self.local.data_ptr() + 8 * s
            slots = dict(self.persistent)       # the tied OPT head reads the embedding slot
            slots[bid] = slot
            zmode = L.ZO_Z_ORACLE if self.mgr.oracle else L.ZO_Z_PHILOX
            calls = _store_view(self).forward_calls(s, self.ws[s], +eps if s == PLUS else -eps,
                                                    zmode=zmode, z_cur=self._zc, stream=stream, blocks=[bid],
                                                    slots=slots, scal=self.scal, loss_out=loss_out)
            for fn, args in calls:
                L.check(fn(*args))

    def _finalize(self, stream):
        eps, lr = self.hyper.epsilon, self.hyper.lr
        st = int(stream.cuda_stream)
        if self.fabric is None:
            L.check(L.lib().zo_grad_finalize(self.local.data_ptr(), self.local.data_ptr() + 8, float(eps),
                                             float(lr), self.scal.data_ptr(), self.record.data_ptr(), st))
        else:
            with torch.cuda.stream(stream):
                self.fabric.all_gather_tensor(self.gathered, self.local, tag="loss")
            sp, op, sm, om = self.mesh.layout
            L.check(L.lib().zo_grad_finalize_groups(self.gathered.data_ptr(), self.mesh.n_groups, sp, op, sm, om,
                                                    self.mesh.group, float(eps), float(lr), self.scal.data_ptr(),
                                                    self.record.data_ptr(), st))

    # -- one iteration (scheduler.py:243-283) -----------------------------------------
    def step(self, batch: Batch, seed: int) -> ZoStep:
        self.iteration += 1
        batch.validate(self.config)
        B, T = batch.token_ids.shape
        if self.ws is None:                      # reference constructor form: sized by the first batch
            self.ws = {s: Workspace(self.config, B, T, self.device, f32=self.precision == "f32")
                       for s in self.dirs}
        for ws in self.ws.values():
            if ws.batch != B or ws.seq != T:
                raise ConfigurationError("batch shape differs from the runtime's workspace")
            _load(ws, batch)
        self.scal[0:1].fill_(_u64_as_i64(seed))
        self.scal[3:4].fill_(1 if self._pending else 0)
        if self.mgr.oracle:                      # the reference's z of this iteration, whole model, key order
            self.mgr.reset(seed)
            self._zp = self._zc if self._pending else None
            self._zc = torch.from_numpy(self.mgr.generator(seed).standard_normal(self.host.total_params)).to(
                self.device)
        cs, us, os_ = self.streams[COMPUTE], self.streams[UPLOAD], self.streams[OFFLOAD]
        ev = {}
        rec = []
        self._phase_ev = []

        def mark(kind, bid, stream):
            e = torch.cuda.Event(enable_timing=self.trace)
            e.record(stream)
            ev[(kind, bid)] = e
            return e

        t0 = torch.cuda.Event(enable_timing=self.trace)
        t0.record(cs)
        start = mark("start", -1, cs)
        us.wait_event(start)
        os_.wait_event(start)
        emb, head = self.layouts[0].block_id, self.layouts[-1].block_id
        n = len(self.slots)

        def upload(k):                                         # U(wids[k]) into slot k % n
            eu = torch.cuda.Event(enable_timing=self.trace)
            eu.record(us)
            self._upload(self.wids[k], self.slots[k % n], us)
            mark(UPLOAD, self.wids[k], us)
            rec.append((UPLOAD, self.wids[k], eu))

        for k in range(min(n, len(self.wids))):                # fill every slot up front: the uploads
            upload(k)                                          # run under the embedding / resident blocks
        e_c = torch.cuda.Event(enable_timing=self.trace)
        e_c.record(cs)
        self._compute(emb, self.persistent[emb], cs)
        mark(COMPUTE, emb, cs)
        rec.append((COMPUTE, emb, e_c))
        for bid in self.resident:                              # resident blocks: no U / O
            er = torch.cuda.Event(enable_timing=self.trace)
            er.record(cs)
            self._compute(bid, self.persistent[bid], cs)
            mark(COMPUTE, bid, cs)
            rec.append((COMPUTE, bid, er))
        for idx, i in enumerate(self.wids):
            slot = self.slots[idx % n]
            cs.wait_event(ev[(UPLOAD, i)])                        # C(i) after U(i) (and C(i-1): same stream)
            ec = torch.cuda.Event(enable_timing=self.trace)
            ec.record(cs)
            self._compute(i, slot, cs)
            mark(COMPUTE, i, cs)
            rec.append((COMPUTE, i, ec))
            os_.wait_event(ev[(COMPUTE, i)])                       # O(i) after C(i)
            eo = torch.cuda.Event(enable_timing=self.trace)
            eo.record(os_)
            self._offload(i, slot, os_)
            mark(OFFLOAD, i, os_)
            rec.append((OFFLOAD, i, eo))
            if idx + n < len(self.wids):                           # U(i+n) into this slot once O(i) freed it
                us.wait_event(ev[(OFFLOAD, i)])
                upload(idx + n)
        eh = torch.cuda.Event(enable_timing=self.trace)
        eh.record(cs)
        self._compute(head, self.persistent[head], cs)
        self._finalize(cs)
        mark(COMPUTE, head, cs)
        rec.append((COMPUTE, head, eh))
        cs.wait_event(mark("tail", -1, os_))
        r = self.record.cpu().numpy()
        errs = [int(ws.err.item()) for ws in self.ws.values()]
        if any(errs):
            self._pending = False          # the blocks consumed the pending update; the device armed none
            _store_view(self).check_errors(*self.ws.values(), flags=errs)
        if self.trace:
            self.timelines.append([{"op": k, "block_id": b, "stream": k, "start": t0.elapsed_time(e),
                                    "end": t0.elapsed_time(ev[(k, b)])} for k, b, e in rec])
            for name, e0, e1, nb in self._phase_ev:
                st_ = self.phase_stats.setdefault(name, {"ms": 0.0, "bytes": 0, "n": 0})
                st_["ms"] += e0.elapsed_time(e1)
                st_["bytes"] += nb
                st_["n"] += 1
            for k, b, e in rec:
                if k == COMPUTE and b in self.wids:
                    st_ = self.phase_stats.setdefault("compute", {"ms": 0.0, "bytes": 0, "n": 0})
                    st_["ms"] += e.elapsed_time(ev[(k, b)])
                    st_["n"] += 1
            self._phase_ev = []
        self.uploaded_params += sum(self.layouts[i].elem_count for i in self.wids)
        self.offloaded_params += sum(self.layouts[i].elem_count for i in self.wids)
        st = ZoStep(self.iteration, seed, float(r[0]), float(r[1]), float(r[2]))
        self._g_prev, self.last_seed, self._pending = st.g, seed, True
        self.host.unflushed = True
        return st

    # -- end of run (scheduler.py:393-415) ------------------------------------------------
    def flush(self) -> None:
        """Apply the last iteration's deferred update to every block and sync
        the device-resident blocks back to the host."""
        if not self._pending:
            raise ProtocolError("flush with no pending update (double flush?)")
        cs = self.streams[COMPUTE]
        self.scal[3:4].fill_(1)
        self._zp = self._zc                      # oracle mode: the last iteration's z
        for i in self.wids:
            slot = self.slots[0]
            self._upload(i, slot, cs)
            if self.redistribute == "bf16":
                self._perturb_slice(i, slot, L.ZO_PU_UPDATE, cs)     # own slice only
            else:
                self._perturb(i, slot, L.ZO_PU_UPDATE, cs)
            self._offload(i, slot, cs)
            cs.synchronize()
        for bid, slot in self.persistent.items():
            self._perturb(bid, slot, L.ZO_PU_UPDATE, cs)
        self.scal[3:4].fill_(0)
        self.sync_host()
        self._pending = False
        self._zc = self._zp = None
        self.host.unflushed = False

    def sync_host(self) -> None:
        """Copy the persistent device blocks back to the host master (and,
        with split16 compression, rebuild the streamed blocks' fp32 master
        from the hi / lo planes)."""
        cs = self.streams[COMPUTE]
        if self._lo:
            stage = self.slots[0].hi_stage
            tmp = torch.empty(stage.numel(), dtype=torch.float32, device=self.device)
            for bid in self.wids:
                off, ln = self._own(bid)
                with torch.cuda.stream(cs):
                    stage[:ln].copy_(self._hi[bid], non_blocking=True)
                    ops.planes_join(stage[:ln], self._lo[bid], tmp[:ln])
                    self._host_part(bid).copy_(tmp[:ln], non_blocking=True)
                cs.synchronize()
        for bid, slot in self.persistent.items():
            if getattr(self.host, "is_sharded", False):
                self.host.offload_from(bid, slot.theta, cs)
                continue
            hb = self.host.block_buf(bid)
            with torch.cuda.stream(cs):
                hb.copy_(slot.theta[:hb.numel()], non_blocking=True)
        cs.synchronize()

    @property
    def last_timeline(self):
        return self.timelines[-1] if self.timelines else []

    def makespan(self) -> float:
        tl = self.last_timeline
        return max(e["end"] for e in tl) if tl else float("nan")


def plan_residency(config: ModelConfig, budget_bytes: int, n_dirs: int = 2, max_slots: int = 8,
                   compress: str = "none"):
    """(resident_blocks, n_slots) for OffloadedZo under a device-memory budget
    for the transformer blocks: a block costs 4 B/param of fp32 master + 2 B
    per direction of bf16 shadow, resident or in a slot, and with
    compress="split16" every streamed block also keeps its 2 B/param lo plane
    on the device.  As many blocks as fit stay resident (each one removes a
    block's H2D + D2H per step); the slots only need to prefetch what PCIe
    can move while the resident blocks compute (~1 upload per 8 resident
    blocks at the measured 49 GB/s and ~3 ms of compute per OPT-13B block), so
    they get just that depth (>= 3, or whatever fits).  The embedding / head /
    activations are outside the budget."""
    from .model import model_layout

    if compress not in ("none", "split16"):
        raise ConfigurationError(f"compress must be 'none' or 'split16', got {compress!r}")
    blocks = [bl for bl in model_layout(config) if bl.kind == TRANSFORMER]
    nb = len(blocks)
    P = blocks[0].elem_count
    per = P * (4 + 2 * n_dirs)
    lo = P * (2 if compress == "split16" else 0)          # per streamed block
    if nb * per <= budget_bytes:
        return nb, 0

    def kmax(slots):          # resident blocks that fit beside `slots` slots
        return int((budget_bytes - slots * per - nb * lo) // (per - lo))

    fit = int((budget_bytes - nb * lo) // per)            # slots that fit with nothing resident
    if fit < 2:
        raise MemoryCapacityError(f"device budget {budget_bytes} B cannot hold two streamed block slots "
                                  f"({2 * per} B) beside the lo planes ({nb * lo} B)")
    if kmax(0) <= 3:
        return 0, min(3, fit)
    for slots in range(3, max_slots + 1):
        k = kmax(slots)
        if k < 0:
            return 0, min(3, fit)
        if slots >= min(max_slots, max(3, k // 8 + 1)):
            return k, slots
    return max(kmax(max_slots), 0), max_slots


def _load(ws: Workspace, batch: Batch):
    ids = np.asarray(batch.token_ids).reshape(-1).astype(np.int32)
    tg = np.asarray(batch.targets).reshape(-1).astype(np.int32)
    ws.ids.copy_(torch.from_numpy(ids))
    ws.tgt.copy_(torch.from_numpy(tg))


class _StoreView:
    """Adapter giving OffloadedZo the DeviceStore.forward_calls builder
    without allocating a resident master."""

    def __init__(self, rt: OffloadedZo):
        from .engine import DeviceStore

        self.config, self.layouts, self.plan = rt.config, rt.layouts, rt.plan
        self.scal = rt.scal
        self.precision = rt.precision
        self._fc = DeviceStore.forward_calls.__get__(self)
        self.check_errors = DeviceStore.check_errors.__get__(self)
        self._fc32 = DeviceStore.forward_calls_f32.__get__(self)

    def forward_calls(self, *a, **k):
        return self._fc(*a, **k)

    def forward_calls_f32(self, *a, **k):
        return self._fc32(*a, **k)


def _store_view(rt: OffloadedZo) -> _StoreView:
    if not hasattr(rt, "_sv"):
        rt._sv = _StoreView(rt)
    return rt._sv


def activation_nbytes(config: ModelConfig, batch_size: int) -> int:
    """Device bytes of one directional activation tensor (scheduler.py:435-438), fp32 residual."""
    return batch_size * config.seq_len * config.d_model * 4


def time_step(rt: OffloadedZo, batch: Batch, seed: int) -> float:
    torch.cuda.synchronize()
    t = time.perf_counter()
    rt.step(batch, seed)
    return time.perf_counter() - t
