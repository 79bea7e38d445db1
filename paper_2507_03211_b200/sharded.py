"""Sharded fp32 master: in HBM (ZeRO-3 style)
or in per-rank, NUMA-local pinned host memory (the sliced offload of configs
#4 / #5).

Instead of the pinned host master of the ZO2 offload runtime, the fp32 master
is split over the N ranks' HBM with the reference's slice layout
(comm.py:106-119, fixed at init like apply_thread_aligned_layout,
comm.py:345-358): rank r keeps slice r of every block, ``ceil(P_blk / N)``
elements.  The block-streaming schedule of scheduler.OffloadedZo runs
unchanged; only its two byte movements change:

  upload(b)    own slice HBM -> slot (device copy) + all-gather of the other
               slices over NVLink: no PCIe at all
  offload(b)   own slice of the updated block slot -> shard (device copy)

so every rank computes the identical fused update+perturb on the whole block
(z is keyed by the global element index) and the shards stay exactly the
slices of the resident master -- sharded == resident bit for bit, like the
sliced offload path.  Per-GPU HBM at the OPT-175B shape on 8 ranks: 87.6 GB
of shards + the resident embedding / head + 3 block slots.

``where="host"`` keeps the same slices in pinned host memory instead: each
rank owns ONLY its 1/N of every block (87.6 GB per rank at 175B / 8, not the
701 GB master on every rank), allocated after the process is bound to the
CPUs of its GPU's NUMA node (``bind_to_gpu_numa``), so the pages are local to
the socket whose PCIe root serves that GPU.  upload(b) is then the own slice
over this rank's PCIe link (comm.py:314-328 phase 1) and offload(b) the own
slice back (comm.py:331-342); the full master exists only when gathered for
flush checks / checkpoints (``gather_master``).
"""

from __future__ import annotations

import hashlib

import numpy as np
import torch

from . import _lib as L
from .errors import ConfigurationError
from .model import ModelConfig, init_block_host, model_layout
from .scheduler import SliceLayout


class ShardStore:
    """This rank's slices of the fp32 master, resident in HBM.

    ``fabric`` is a fabric.TorchFabric (None: one rank owning everything).
    ``init``: "host" (zosim's numpy draw of each block, the slice kept) or
    "philox" (random-init at scale, each rank drawing only its slice)."""

    is_sharded = True

    def __init__(self, config: ModelConfig, fabric=None, init_seed: int = 7, init: str = "host", device=None,
                 where: str = "hbm", numa: bool = True):
        config.validate()
        if where not in ("hbm", "host"):
            raise ConfigurationError(f"where must be 'hbm' or 'host', got {where!r}")
        self.on_host = where == "host"
        self.config, self.init_seed, self.fabric = config, init_seed, fabric
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        L.lib()
        self.layouts = model_layout(config)
        self.total_params = sum(b.elem_count for b in self.layouts)
        self.n = fabric.k if fabric is not None else 1
        self.rank = fabric.rank if fabric is not None else 0
        self.slice_plan = {"n": self.n, "layouts": {bl.block_id: SliceLayout(bl.block_id, bl.elem_count, self.n)
                                                    for bl in self.layouts}}
        self.offsets, off = {}, 0
        for bl in self.layouts:
            self.offsets[bl.block_id] = off
            off += self.slice_plan["layouts"][bl.block_id].width
        self.numa = bind_to_gpu_numa(self.device) if (self.on_host and numa) else None
        if self.on_host:          # first touch by this (NUMA-bound) process -> node-local pages
            self.shard = torch.zeros(max(off, 1), dtype=torch.float32, pin_memory=True)
        else:
            self.shard = torch.zeros(max(off, 1), dtype=torch.float32, device=self.device)
        if init == "host":
            for bl in self.layouts:
                _, lo, ln = self.own(bl.block_id)
                if ln:
                    buf = init_block_host(config, bl, init_seed)
                    self.slice_of(bl.block_id).copy_(torch.from_numpy(buf[lo:lo + ln]))
        elif init == "philox":
            self._init_philox(init_seed)
        elif init != "none":
            raise ConfigurationError(f"unknown init {init!r}")
        self.unflushed = False

    # -- layout ---------------------------------------------------------------------
    def own(self, bid: int):
        """(owner, offset, length) of this rank's slice of block ``bid``."""
        return self.slice_plan["layouts"][bid].slices[self.rank]

    def slice_of(self, bid: int) -> torch.Tensor:
        _, _, ln = self.own(bid)
        o = self.offsets[bid]
        return self.shard[o:o + ln]

    @property
    def shard_bytes(self) -> int:
        return self.shard.numel() * 4

    def host_part(self, bid: int) -> torch.Tensor:
        """The part of block ``bid`` this rank moves over PCIe (its slice)."""
        return self.slice_of(bid)

    def _init_philox(self, init_seed: int):
        """DeviceStore._init_philox restricted to this rank's slices: the same
        values the resident store draws (z keyed by the global element)."""
        seed = (0x1A2B3C4D << 32) ^ int(init_seed)
        for bl in self.layouts:
            _, lo, ln = self.own(bl.block_id)
            dst = self.slice_of(bl.block_id)
            for name in bl.names:
                a, b = bl.offsets[name], bl.offsets[name] + bl.size(name)
                i0, i1 = max(a, lo), min(b, lo + ln)
                if i0 >= i1:
                    continue
                seg = dst[i0 - lo:i1 - lo]
                if name.endswith("_g"):
                    seg.fill_(1.0)
                elif name.startswith("b") or name.endswith("_b"):
                    seg.zero_()
                else:
                    for c0 in range(i0, i1, 1 << 26):
                        c1 = min(i1, c0 + (1 << 26))
                        tmp = seg[c0 - i0:c1 - i0] if not self.on_host else \
                            torch.empty(c1 - c0, dtype=torch.float32, device=self.device)
                        L.call("zo_philox_normals", seed, bl.key0 + c0, c1 - c0, tmp.data_ptr(), L.stream_ptr())
                        tmp.mul_(0.02)
                        if self.on_host:
                            seg[c0 - i0:c1 - i0].copy_(tmp)

    # -- the two byte movements of the streaming schedule ----------------------------
    def upload_into(self, bid: int, slot_theta: torch.Tensor, stream=None, gather: bool = True) -> None:
        """Own slice -> its place in the (n * width padded) slot, then the
        peers' slices by an all-gather over NVLink (comm.py:314-328 with the
        host leg replaced by a device copy)."""
        lay = self.slice_plan["layouts"][bid]
        _, off, ln = self.own(bid)
        w = lay.width
        ctx = torch.cuda.stream(stream) if stream is not None else _Null()
        with ctx:
            if ln:
                slot_theta[self.rank * w:self.rank * w + ln].copy_(self.slice_of(bid), non_blocking=True)
            if self.n > 1 and gather:
                self.fabric.all_gather_tensor(slot_theta[:self.n * w],
                                              slot_theta[self.rank * w:(self.rank + 1) * w], tag="param")

    def offload_from(self, bid: int, slot_theta: torch.Tensor, stream=None) -> None:
        """Own slice of the updated block back into the shard (comm.py:331-342)."""
        _, off, ln = self.own(bid)
        ctx = torch.cuda.stream(stream) if stream is not None else _Null()
        with ctx:
            if ln:
                self.slice_of(bid).copy_(slot_theta[off:off + ln], non_blocking=True)

    # -- whole-master views (collective when sharded: every rank must call) ----------
    def gather_block(self, bid: int) -> torch.Tensor:
        lay = self.slice_plan["layouts"][bid]
        buf = torch.zeros(self.n * lay.width, dtype=torch.float32, device=self.device)
        self.upload_into(bid, buf)
        torch.cuda.current_stream().synchronize()
        return buf[:lay.total]

    def gather_master(self) -> np.ndarray:
        return np.concatenate([self.gather_block(bl.block_id).cpu().numpy() for bl in self.layouts])

    @property
    def theta(self) -> torch.Tensor:
        """The full master (a gathered copy; collective) -- checkpointing and tests."""
        return torch.from_numpy(self.gather_master())

    def checksum(self) -> str:
        h = hashlib.sha256()
        for bl in self.layouts:
            h.update(self.gather_block(bl.block_id).cpu().numpy().tobytes())
        return h.hexdigest()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def bind_to_gpu_numa(device) -> dict:
    """Pin this process to the CPUs NVML reports as local to ``device``'s
    PCIe root (its NUMA node), so pinned buffers allocated afterwards are
    first-touched on that node and the H2D / D2H of the sliced schedule never
    cross the socket interconnect.  No-op (reported) where NVML or the
    affinity call is unavailable."""
    import os

    info = {"bound": False, "cpus": None, "node": None}
    try:
        import pynvml

        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(device).uuid)
        h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        ncpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1 and 64 * i + b < ncpu}
        if cpus and len(cpus) < ncpu:
            os.sched_setaffinity(0, cpus)
            info.update(bound=True, cpus=len(cpus))
        elif cpus:
            info.update(cpus=len(cpus))          # one node (or no topology): nothing to restrict
        try:
            bus = pynvml.nvmlDeviceGetPciInfo(h).busId
            bus = (bus.decode() if isinstance(bus, bytes) else bus).lower()[-12:]     # dddd:bb:dd.f
            with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
                info["node"] = int(f.read().strip())
        except (OSError, ValueError, AttributeError):
            pass
    except Exception as e:  # noqa: BLE001  (NVML missing / no permission: keep the default placement)
        info["error"] = type(e).__name__
    return info
