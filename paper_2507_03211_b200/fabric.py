"""Collective fabric over torch.distributed (mirror of src/zosim/fabric.py).

The reference runs K ranks as threads exchanging Python values through
barriers (fabric.py:34-51); here each rank is a process (one per GPU) and
the collectives are NCCL over NVLink (or gloo for CPU tests).  The API keeps
the reference's determinism contract:

  all_gather       values ordered by rank                     fabric.py:90-94
  broadcast        root's value on every rank                  fabric.py:96-103
  all_reduce_mean  FIXED ascending-rank sum / k (bit-stable)   fabric.py:105-113
  bytes_by_tag / collective_log accounting                     fabric.py:65-80

NCCL's own all_reduce does not promise the reference's summation order, so
every reduction is an all_gather followed by an ordered local sum -- the
payloads are 8-byte scalars, so this costs the same.
"""

from __future__ import annotations

import datetime

import numpy as np
import torch
import torch.distributed as dist

from .errors import ConfigurationError, FabricFault


def _payload_bytes(value) -> int:
    if isinstance(value, torch.Tensor):
        return value.numel() * value.element_size()
    if isinstance(value, np.ndarray):
        return value.nbytes
    if isinstance(value, (list, tuple)):
        return sum(_payload_bytes(v) for v in value)
    if isinstance(value, (bytes, bytearray, str)):
        return len(value)
    if value is None:
        return 0
    return 8


class TorchFabric:
    """K processes with ordered, deterministic collectives.

    data_plane: "collective" moves the offload's block slices with NCCL
    (all_gather_into_tensor / batched send-recv: SM-driven kernels);
    "copy_engine" maps the peers' buffers once through CUDA IPC and has every
    rank PULL the slices it needs with cudaMemcpyAsync -- the DMA copy engines,
    so the transfer takes no SMs from the GEMMs it overlaps (option
    b) -- between two host barriers per exchange.  Same bytes, same results."""

    CE_MIN_BYTES = 64 << 10        # smaller payloads (the loss exchange) stay collective

    def __init__(self, group=None, data_plane: str = "collective"):
        if not dist.is_initialized():
            raise FabricFault("torch.distributed is not initialised")
        if data_plane not in ("collective", "copy_engine"):
            raise ConfigurationError(f"data_plane must be 'collective' or 'copy_engine', got {data_plane!r}")
        self.data_plane = data_plane
        self._peer_storages: dict = {}
        self.ce_exchanges = 0          # exchanges that went through the copy engines
        self.group = group
        self.rank = dist.get_rank(group)
        self.k = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.bytes_by_tag: dict = {}
        self.collective_log: list = []
        self._subgroups: dict = {}

    def _account(self, kind, tag, participants, nbytes):
        self.bytes_by_tag[tag] = self.bytes_by_tag.get(tag, 0) + nbytes
        self.collective_log.append({"kind": kind, "tag": tag, "participants": participants})

    def subgroup(self, ranks):
        """Process group for an ascending tuple of ranks.  new_group is a
        collective over the whole world, so the mesh's group FAMILIES are
        created together, in a fixed order, on every rank: PertP pairs
        (2i, 2i+1) and the two direction branches (even / odd ranks)."""
        ranks = tuple(sorted(ranks))
        if ranks not in self._subgroups:
            k = self.k
            pairs = [(2 * i, 2 * i + 1) for i in range(k // 2)]
            branches = [tuple(range(0, k, 2)), tuple(range(1, k, 2))]
            if ranks in pairs:
                family = pairs
            elif ranks in branches:
                family = branches
            else:
                family = [ranks]
            for g in family:
                if g not in self._subgroups:
                    self._subgroups[g] = dist.new_group(list(g), backend=self.backend)
        return self._subgroups[ranks]

    def _dev(self):
        if self.backend == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    # -- scalar / small-object collectives ------------------------------------
    def all_gather(self, rank, value, tag, group=None) -> list:
        """Every participant's float/int value, ordered by rank."""
        ranks = tuple(range(self.k)) if group is None else tuple(sorted(group))
        pg = None if group is None else self.subgroup(ranks)
        self._account("all_gather", tag, len(ranks), _payload_bytes(value))
        t = torch.tensor([float(value)], dtype=torch.float64, device=self._dev())
        out = [torch.empty_like(t) for _ in ranks]
        try:
            dist.all_gather(out, t, group=pg)
        except Exception as e:  # noqa: BLE001
            raise FabricFault(f"collective failed: {e}") from e
        return [float(o.item()) for o in out]

    def broadcast(self, rank, value, tag, root=0, group=None):
        self._account("broadcast", tag, self.k, _payload_bytes(value) if rank == root else 0)
        t = torch.tensor([int(value) if rank == root else 0], dtype=torch.int64, device=self._dev())
        try:
            dist.broadcast(t, src=root, group=self.group)
        except Exception as e:  # noqa: BLE001
            raise FabricFault(f"collective failed: {e}") from e
        return int(t.item())

    def all_reduce_mean(self, rank, value, tag, group=None) -> float:
        vals = self.all_gather(rank, value, tag, group)
        self.collective_log[-1]["kind"] = "all_reduce"
        total = 0.0
        for v in vals:            # fixed ascending-rank order (fabric.py:105-113)
            total += v
        return total / len(vals)

    # -- copy-engine data plane -------------------------------------------------
    def _use_ce(self, t: torch.Tensor) -> bool:
        return (self.data_plane == "copy_engine" and self.k > 1 and t.is_cuda
                and t.numel() * t.element_size() >= self.CE_MIN_BYTES
                and not torch.cuda.is_current_stream_capturing())

    def _peers_of(self, t: torch.Tensor) -> list:
        """Every rank's storage corresponding to ``t``'s, as flat tensors of
        t's dtype (rank order).  Collective on first use: the storages' CUDA
        IPC handles are all-gathered; corresponding buffers are allocated in
        the same order on every rank, so their views share storage offsets."""
        st = t.untyped_storage()
        key = st.data_ptr()
        peers = self._peer_storages.get(key)
        if peers is None:
            from torch.multiprocessing.reductions import reduce_tensor

            flat = torch.empty(0, dtype=t.dtype, device=t.device).set_(st)
            fn, args = reduce_tensor(flat)
            objs = [None] * self.k
            dist.all_gather_object(objs, args, group=self.group)
            peers = [flat if q == self.rank else fn(*objs[q]) for q in range(self.k)]
            self._peer_storages[key] = peers
        return peers

    def _ce_pull(self, dst: torch.Tensor, pulls) -> None:
        """pulls: (element range in dst, rank, source tensor) -- every rank has
        written its part before the first barrier, and nobody reuses its buffer
        before every rank has finished reading (second barrier)."""
        self.ce_exchanges += 1
        cur = torch.cuda.current_stream()
        cur.synchronize()
        dist.barrier(group=self.group)
        for (a, b), src in pulls:
            dst[a:b].copy_(src, non_blocking=True)        # cudaMemcpyAsync: a DMA copy engine
        cur.synchronize()
        dist.barrier(group=self.group)

    # -- device tensor gather (the step's loss exchange) ------------------------
    def all_gather_tensor(self, out: torch.Tensor, inp: torch.Tensor, tag: str) -> None:
        """out[k*n:(k+1)*n] = inp of rank k.  NCCL: in place on the GPU (no host
        round trip, graph-capturable); gloo: staged through host memory;
        copy-engine plane: pulled from the peers' buffers."""
        self._account("all_gather", tag, self.k, _payload_bytes(inp))
        if self._use_ce(out):
            n, r = inp.numel(), self.rank
            mine = out[r * n:(r + 1) * n]
            if inp.data_ptr() != mine.data_ptr():
                mine.copy_(inp)
            peers, off = self._peers_of(out), out.storage_offset()
            self._ce_pull(out, [((q * n, (q + 1) * n), peers[q][off + q * n:off + (q + 1) * n])
                                for q in range(self.k) if q != r])
            return
        if self.backend == "nccl":
            dist.all_gather_into_tensor(out, inp, group=self.group)
            return
        h = inp.detach().cpu()
        parts = [torch.empty_like(h) for _ in range(self.k)]
        dist.all_gather(parts, h, group=self.group)
        out.copy_(torch.cat(parts).to(out.device))

    def exchange_slices(self, bufs: dict, my_dir: int, dir_of: list, width: int, tag: str) -> None:
        """Direction-aware redistribution: every rank k holds
        slice [k*w, (k+1)*w) of each direction's buffer in ``bufs``; rank q
        receives slice k of ``bufs[dir_of[q]]`` from every k into its own
        ``bufs[my_dir]``, so it pulls only (K-1)*w elements of its direction
        -- half the bytes of the fp32 all-gather when the buffers are bf16.
        NCCL: point-to-point sends / receives straight between the buffers;
        gloo: staged through host memory (tests)."""
        r, w, mine = self.rank, width, bufs[my_dir]
        self._account("exchange", tag, self.k, w * mine.element_size())   # own slice, as all_gather_tensor counts
        if self.k == 1:
            return
        if self._use_ce(mine):
            peer_bufs = {d: self._peers_of(bufs[d]) for d in sorted(bufs)}    # symmetric registration
            src, off = peer_bufs[my_dir], mine.storage_offset()
            self._ce_pull(mine, [((q * w, (q + 1) * w), src[q][off + q * w:off + (q + 1) * w])
                                 for q in range(self.k) if q != r])
            return
        if self.backend == "nccl":
            peer = (lambda q: q) if self.group is None else (lambda q: dist.get_global_rank(self.group, q))
            ops = []
            for q in range(self.k):
                if q == r:
                    continue
                ops.append(dist.P2POp(dist.isend, bufs[dir_of[q]][r * w:(r + 1) * w], peer(q), self.group))
                ops.append(dist.P2POp(dist.irecv, mine[q * w:(q + 1) * w], peer(q), self.group))
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            return
        dirs = sorted(bufs)      # gloo has no 16-bit integer type: carry the bits widened to int32
        h = torch.stack([bufs[d][r * w:(r + 1) * w].view(torch.int16) for d in dirs]).cpu().to(torch.int32)
        parts = [torch.empty_like(h) for _ in range(self.k)]
        dist.all_gather(parts, h, group=self.group)
        mi = dirs.index(my_dir)
        for q in range(self.k):
            if q != r:
                mine[q * w:(q + 1) * w].view(torch.int16).copy_(parts[q][mi].to(torch.int16).to(mine.device))

    def barrier(self):
        dist.barrier(group=self.group)

    def stats(self) -> dict:
        return {"bytes_by_tag": dict(self.bytes_by_tag), "collectives": len(self.collective_log)}


def init_from_env(backend: str = "nccl", timeout_s: float = 60.0) -> TorchFabric:
    """torchrun-style initialisation; a rank that never joins surfaces as
    FabricFault after `timeout_s` (the reference's 60 s barrier timeout)."""
    if not dist.is_initialized():
        dist.init_process_group(backend, timeout=datetime.timedelta(seconds=timeout_s))
    return TorchFabric()
