"""Distribution strategies on B200s (mirror of src/zosim/strategies.py).

One process per GPU; every rank holds a full fp32 replica and derives the
same direction z from the shared seed (Philox keyed by global element), so
replicas stay bit-identical with ZERO parameter traffic:

  PertP  (pertp_step, strategies.py:92-125)   2 ranks; rank 0 evaluates the
         +eps forward, rank 1 the -eps forward of the same batch
  ZO-DDP (ddp_step, strategies.py:128-151)    K ranks, both directions on a
         disjoint batch shard each; g = ordered mean of the K shard g's
  2D     (twod_step, strategies.py:154-222)   n_groups x 2 mesh; rank 2i is
         group i's +eps worker, rank 2i+1 its -eps worker

Per step the only collective is ONE rank-ordered all_gather of 16 bytes per
rank (each rank's [L+, L-] slots, device-resident f64, NCCL over NVLink),
after which every rank evaluates the same ordered reduction on the GPU
(zo_grad_finalize_groups) -- bit-identical g on every rank, and equal to the
reference's ascending-rank arithmetic (fabric.py:105-113).  A PertP/2D rank
writes only its own direction's shadows (10 B/param perturb pass instead of
12), and the update is folded into the next step's pass (MeshZo) or applied
eagerly at the end of the step (the *_step functions, like the reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .engine import MINUS, PLUS, DeviceStore
from .errors import ConfigurationError, ConsistencyError, DimensionError, NumericError, ProtocolError
from .model import Batch
from .rng import RngStateManager
from .zo import (NativeGraph, ZoHyper, ZoStep, _block_events, _finish_record, _priority_streams, _record,
                 _record_and_wait, _u64_as_i64, _wait)

PLUS_DIR, MINUS_DIR = +1, -1


@dataclass(frozen=True)
class RankAssignment:
    """strategies.py:35-47."""

    rank: int
    group: int
    direction: int
    n_groups: int

    @property
    def pair_ranks(self):
        return (2 * self.group, 2 * self.group + 1)


def mesh_assignments(n_groups: int):
    """rank 2i = +eps, 2i+1 = -eps of group i (strategies.py:50-56)."""
    return [RankAssignment(r, r // 2, PLUS_DIR if r % 2 == 0 else MINUS_DIR, n_groups) for r in range(2 * n_groups)]


class MeshLayout:
    """Where group i's L+ and L- sit in the rank-ordered gather of every
    rank's 2 loss slots, and which directions this rank evaluates."""

    def __init__(self, strategy: str, world: int, rank: int):
        if strategy not in ("pertp", "ddp", "2d"):
            raise ConfigurationError(f"unknown strategy {strategy!r}")
        if strategy == "pertp" and world != 2:
            raise ConfigurationError(f"direction parallelism needs exactly 2 workers, got {world}")
        if strategy == "2d" and world % 2:
            raise ConfigurationError(f"2d mesh needs an even number of ranks, got {world}")
        self.strategy, self.world, self.rank = strategy, world, rank
        if strategy == "ddp":
            self.n_groups, self.group = world, rank
            self.dirs = (PLUS, MINUS)
            self.layout = (2, 0, 2, 1)            # L+_i = g[2i], L-_i = g[2i+1]
        else:
            self.n_groups, self.group = world // 2, rank // 2
            self.dirs = (PLUS,) if rank % 2 == 0 else (MINUS,)
            self.layout = (4, 0, 4, 3)            # L+_i = rank 2i slot 0, L-_i = rank 2i+1 slot 1

    def grad_host(self, gathered, eps: float) -> float:
        """The reduction the GPU kernel performs, in Python floats (for CPU
        tests of the gather layout)."""
        sp, op, sm, om = self.layout
        total = 0.0
        for i in range(self.n_groups):
            total += (gathered[i * sp + op] - gathered[i * sm + om]) / (2.0 * eps)
        return total / self.n_groups


def broadcast_seed(fabric, rank: int, seed=None, root: int = 0) -> int:
    """strategies.py:59-61."""
    return int(fabric.broadcast(rank, seed, tag="seed", root=root))


class MeshZo:
    """One rank's lazy-update ZO step under pertp / ddp / 2d (the multi-GPU
    counterpart of StreamingZo).  ``step`` is the public API; ``step_calls``
    is the launch plan the benchmark replays."""

    def __init__(self, store: DeviceStore, hyper: ZoHyper, fabric, strategy: str, batch: int, seq: int,
                 mgr: RngStateManager | None = None, graph: bool = True, overlap: str = "fill"):
        """graph: from the second step on, replay the step's launches -- the
        fused pass, the forward(s), the NCCL loss all-gather and the ordered
        g reduction -- from one captured CUDA graph (NCCL fabrics only: a
        gloo collective stages through the host and cannot be captured).
        overlap: "fill" (Philox runs) perturbs blocks 2.. as short-CTA
        launches on a low-priority stream under the high-priority forward,
        as StreamingZo's fill plan; "none": the whole pass, then the forward.
        Same arithmetic either way."""
        if overlap not in ("fill", "none"):
            raise ConfigurationError(f"unknown step plan {overlap!r} (plans: 'fill', 'none')")
        self.store, self.hyper, self.fabric = store, hyper.validate(), fabric
        self.mesh = MeshLayout(strategy, fabric.k, fabric.rank)
        for s in self.mesh.dirs:
            if store.wsh[s] is None:
                raise ConfigurationError("store lacks the shadow buffers of this rank's direction")
        self.mgr = mgr or RngStateManager()      # "oracle": the reference's z injected (parity runs)
        self.ws = {s: store.workspace(s, batch, seq) for s in self.mesh.dirs}
        dev = store.device
        self.local = torch.zeros(2, dtype=torch.float64, device=dev)
        self.gathered = torch.zeros(2 * fabric.k, dtype=torch.float64, device=dev)
        self.iteration, self._pending, self._g_prev, self.last_seed = 0, False, 0.0, None
        self._zc = self._zp = None
        self.overlap = overlap if not self.mgr.oracle else "none"
        self.graph = bool(graph) and not self.mgr.oracle and getattr(fabric, "backend", None) == "nccl"
        self._graphs = {}          # io flag -> captured step
        self._io = None

    @property
    def g_prev(self) -> float:
        return self._g_prev

    @g_prev.setter
    def g_prev(self, g: float) -> None:
        """Replacing g_prev replaces the deferred update the next step's
        fused pass (or flush) applies, as in the reference (zo.py:267-278)."""
        self._g_prev = float(g)
        self.store.scal[2:3].fill_(int(np.float64(self.hyper.lr * float(g)).view(np.int64)))

    def step_calls(self, update: bool = True, zc=None, zp=None):
        s, eps, m = self.store, self.hyper.epsilon, self.mesh
        zmode = L.ZO_Z_ORACLE if self.mgr.oracle else L.ZO_Z_PHILOX
        flags = (L.ZO_PU_UPDATE if update else 0)
        sa = sb = None
        sc_a = sc_b = 0.0
        if PLUS in m.dirs:
            flags |= L.ZO_PU_SHADOW_A
            sa, sc_a = PLUS, +eps
        if MINUS in m.dirs:
            flags |= L.ZO_PU_SHADOW_B
            sb, sc_b = MINUS, -eps
        if self.overlap == "fill" and zmode == L.ZO_Z_PHILOX:
            calls = self._fill_calls(flags, sa, sb, sc_a, sc_b)
        else:
            calls = s.perturb_call(s.model_table, flags, sc_a, sc_b, sa=sa, sb=sb, zmode=zmode, z_cur=zc,
                                   z_prev=zp)
            for d in m.dirs:
                loss_out = self.local.data_ptr() + 8 * d
                calls += s.forward_calls(d, self.ws[d], +eps if d == PLUS else -eps, zmode=zmode, z_cur=zc,
                                         loss_out=loss_out)
        calls.append((_gather, (self.fabric, self.gathered, self.local)))
        sp, op, sm, om = m.layout
        calls.append((L.lib().zo_grad_finalize_groups,
                      (self.gathered.data_ptr(), m.n_groups, sp, op, sm, om, m.group, float(eps),
                       float(self.hyper.lr), s.scal.data_ptr(), s.record.data_ptr(), L.stream_ptr())))
        return calls

    def _fill_calls(self, flags, sa, sb, sc_a, sc_b):
        """The fused pass of the embedding + block 1 on the high-priority
        stream, blocks 2.. as ZO_PU_FILL launches on the low-priority stream
        (one event per block), this rank's forward(s) on the high-priority
        stream waiting for each block's event; both streams join the caller's
        stream before the loss exchange (StreamingZo.fill_step_calls)."""
        s, eps = self.store, self.hyper.epsilon
        nl = len(s.layouts)
        main = torch.cuda.current_stream()
        hi, lo = _priority_streams(s)
        ev = _block_events(s, nl + 3)
        calls = [(_record_and_wait, (ev[nl], main, hi)), (_wait, (lo, ev[nl]))]
        calls += s.perturb_call(s.head_table(), flags, sc_a, sc_b, sa=sa, sb=sb, stream=hi)
        for b in range(2, nl):
            calls += s.perturb_call(s.block_tables[b], flags | L.ZO_PU_FILL, sc_a, sc_b, sa=sa, sb=sb, stream=lo)
            calls.append((_record, (ev[b], lo)))
        for i, d in enumerate(self.mesh.dirs):
            sc, loss_out = (+eps if d == PLUS else -eps), self.local.data_ptr() + 8 * d
            calls += s.forward_calls(d, self.ws[d], sc, stream=hi, blocks=[0, 1], loss_out=loss_out)
            for b in range(2, nl):
                if i == 0:
                    calls.append((_wait, (hi, ev[b])))
                calls += s.forward_calls(d, self.ws[d], sc, stream=hi, blocks=[b], loss_out=loss_out)
        calls.append((_record_and_wait, (ev[nl + 1], hi, main)))
        calls.append((_record_and_wait, (ev[nl + 2], lo, main)))
        return calls

    def replay(self, io: bool = False):
        """Capture the Philox step once (the first step ran eagerly, so the
        NCCL communicator, kernel attributes and TMA descriptors exist), then
        replay it; seeds / pending flag / g live on the device, so one graph
        serves every step.  io=True (the public step): the graph also copies
        the shard / seed / pending flag in from pinned staging and the record /
        error flags out (zo_copy_async nodes)."""
        g = self._graphs.get(io)
        if g is None:
            def build():
                calls = self.step_calls()
                if io:
                    cin, cout = self._io_calls()
                    calls = cin + calls + cout
                return calls

            g = None
            if self.overlap == "fill":
                try:
                    g = NativeGraph(self.store.run, build)      # replays with launch priorities
                except Exception:                               # noqa: BLE001
                    # a communicator that refuses a raw stream capture: torch's
                    # capture (node priorities dropped, same launches)
                    torch.cuda.synchronize()
                    g = None
            if g is None:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    self.store.run(build())
            self._graphs[io] = g
        g.replay()

    def _io_bufs(self):
        ws0 = next(iter(self.ws.values()))
        io = self._io
        if io is None or io["M"] != ws0.M:
            io = self._io = {"M": ws0.M,
                             "ids": torch.empty(2, ws0.M, dtype=torch.int32, pin_memory=True),
                             "scal": torch.zeros(2, dtype=torch.int64, pin_memory=True),
                             "rec": torch.zeros(3, dtype=torch.float64, pin_memory=True),
                             "err": torch.zeros(4, dtype=torch.int32, pin_memory=True)}
        return io

    def _io_calls(self):
        s, lib, st = self.store, L.lib(), L.stream_ptr()
        io = self._io_bufs()
        nb = 4 * io["M"]
        cin, seen = [], set()
        for ws in self.ws.values():                # the directions' workspaces may share ids / targets
            if ws.ids.data_ptr() in seen:
                continue
            seen.add(ws.ids.data_ptr())
            cin += [(lib.zo_copy_async, (ws.ids.data_ptr(), io["ids"].data_ptr(), nb, st)),
                    (lib.zo_copy_async, (ws.tgt.data_ptr(), io["ids"].data_ptr() + nb, nb, st))]
        cin += [(lib.zo_copy_async, (s.scal.data_ptr(), io["scal"].data_ptr(), 8, st)),
                (lib.zo_copy_async, (s.scal.data_ptr() + 24, io["scal"].data_ptr() + 8, 8, st))]
        cout = [(lib.zo_copy_async, (io["rec"].data_ptr(), s.record.data_ptr(), 24, st))]
        for i, ws in enumerate(self.ws.values()):
            cout.append((lib.zo_copy_async, (io["err"].data_ptr() + 4 * i, ws.err.data_ptr(), 4, st)))
        return cin, cout

    def _step_graph_io(self, shard: Batch, seed: int) -> ZoStep:
        s = self.store
        shard.validate(s.config)
        ids, tg = np.asarray(shard.token_ids), np.asarray(shard.targets)
        ws0 = next(iter(self.ws.values()))
        if ids.shape != (ws0.batch, ws0.seq) or tg.shape != ids.shape:
            raise DimensionError(f"batch shape {ids.shape} does not match workspace ({ws0.batch}, {ws0.seq})")
        if ids.size and (ids.min() < 0 or ids.max() >= s.config.vocab_size):
            raise DimensionError("token id out of embedding range")
        io = self._io_bufs()
        h = io["ids"].numpy()
        h[0] = ids.reshape(-1)
        h[1] = tg.reshape(-1)
        io["scal"].numpy()[:] = (_u64_as_i64(seed), 1 if self._pending else 0)
        self.replay(io=True)
        torch.cuda.current_stream().synchronize()
        wss = list(self.ws.values())
        s.check_errors(*wss, flags=[int(v) for v in io["err"].numpy()[:len(wss)]])
        r = io["rec"].numpy()
        return ZoStep(self.iteration, seed, float(r[0]), float(r[1]), float(r[2]))

    def stage(self, shard: Batch):
        shard.validate(self.store.config)
        for ws in self.ws.values():
            self.store.load_batch(ws, shard.token_ids, shard.targets)

    def step(self, shard: Batch, seed: int) -> ZoStep:
        """Lazy step: applies the previous iteration's update (folded), then
        this iteration's directional forward(s), loss exchange and g."""
        self.iteration += 1
        s = self.store
        try:
            if self.graph and self.iteration > 1:
                st = self._step_graph_io(shard, seed)
            else:
                self.stage(shard)
                s.scal[0:1].fill_(_u64_as_i64(seed))
                s.scal[3:4].fill_(1 if self._pending else 0)
                if self.mgr.oracle:
                    self._zp = self._zc if self._pending else None
                    self.mgr.reset(seed)
                    self._zc = torch.from_numpy(self.mgr.generator(seed).standard_normal(s.total_params)).to(s.device)
                s.run(self.step_calls(update=not self.mgr.oracle or self._zp is not None, zc=self._zc, zp=self._zp))
                st = _finish_record(s, list(self.ws.values()), self.iteration, seed)
        except NumericError:
            self._pending, s.unflushed = False, False     # nothing armed (see StreamingZo.step)
            raise
        self._pending, self._g_prev, self.last_seed = True, st.g, seed
        s.unflushed = True
        return st

    def flush(self) -> None:
        if not self._pending:
            raise ProtocolError("flush with no pending update (double flush?)")
        s = self.store
        s.scal[3:4].fill_(1)
        zmode = L.ZO_Z_ORACLE if self.mgr.oracle else L.ZO_Z_PHILOX
        s.run(s.perturb_call(s.model_table, L.ZO_PU_UPDATE, 0.0, 0.0, sa=None, sb=None, zmode=zmode,
                             z_prev=self._zc))
        s.scal[3:4].fill_(0)
        torch.cuda.current_stream().synchronize()
        self._pending = False
        self._zc = self._zp = None
        s.unflushed = False


def _gather(fabric, gathered, local):
    fabric.all_gather_tensor(gathered, local, tag="loss")
    return 0


def check_replicas(fabric, rank: int, store: DeviceStore) -> None:
    """Replica-divergence guard (strategies.py:86-89): a 64-bit device hash of
    the fp32 master, gathered and compared (instead of SHA-256 strings)."""
    from .ops import hash_u64

    h = int(hash_u64(store.theta).item()) & ((1 << 64) - 1)
    lo, hi = float(h & 0xFFFFFFFF), float(h >> 32)
    los = fabric.all_gather(rank, lo, tag="checksum")
    his = fabric.all_gather(rank, hi, tag="checksum")
    if len(set(zip(los, his))) != 1:
        raise ConsistencyError(f"parameter replicas diverged across ranks: {list(zip(his, los))}")


def _eager_step(fabric, rank, store, shard, hyper, seed, strategy, mgr, iteration, verify, ordering="pertp_inner"):
    hyper.validate()
    mgr = mgr or RngStateManager()
    seed = broadcast_seed(fabric, rank, seed if rank == 0 else None)
    mesh = MeshLayout(strategy, fabric.k, rank)
    eps = hyper.epsilon
    B, T = shard.token_ids.shape
    zc = None
    zmode = L.ZO_Z_PHILOX
    if mgr.oracle:
        mgr.reset(seed)
        zc = torch.from_numpy(mgr.generator(seed).standard_normal(store.total_params)).to(store.device)
        zmode = L.ZO_Z_ORACLE
    store.scal[0:1].fill_(_u64_as_i64(seed))
    store.scal[3:4].fill_(0)
    local = torch.zeros(2, dtype=torch.float64, device=store.device)
    calls = []
    flags, sa, sb, sca, scb = 0, None, None, 0.0, 0.0
    if PLUS in mesh.dirs:
        flags, sa, sca = flags | L.ZO_PU_SHADOW_A, PLUS, +eps
    if MINUS in mesh.dirs:
        flags, sb, scb = flags | L.ZO_PU_SHADOW_B, MINUS, -eps
    calls += store.perturb_call(store.model_table, flags, sca, scb, sa=sa, sb=sb, zmode=zmode, z_cur=zc)
    wss = []
    for d in mesh.dirs:
        ws = store.workspace(d, B, T)
        store.load_batch(ws, shard.token_ids, shard.targets)
        wss.append(ws)
        calls += store.forward_calls(d, ws, +eps if d == PLUS else -eps, zmode=zmode, z_cur=zc,
                                     loss_out=local.data_ptr() + 8 * d)
    store.run(calls)
    store.check_errors(*wss)
    lh = local.cpu().numpy()
    # the loss exchange, with the reference's collective structure
    if strategy == "ddp":
        g_local = (float(lh[0]) - float(lh[1])) / (2.0 * eps)
        g = fabric.all_reduce_mean(rank, g_local, tag="grad")
        rec = (float(lh[0]), float(lh[1]), g)
    elif ordering == "pertp_inner" or strategy == "pertp":
        mine = float(lh[0] if PLUS in mesh.dirs else lh[1])
        pair = None if strategy == "pertp" else (2 * mesh.group, 2 * mesh.group + 1)
        pl = fabric.all_gather(rank, mine, tag="loss", group=pair)
        g_group = (pl[0] - pl[1]) / (2.0 * eps)
        if strategy == "pertp":
            g = g_group
        else:
            all_g = fabric.all_gather(rank, g_group, tag="grad")
            total = 0.0
            for i in range(mesh.n_groups):
                total += all_g[2 * i]
            g = total / mesh.n_groups
        rec = (pl[0], pl[1], g)
    elif ordering == "ddp_inner":
        mine = float(lh[0] if PLUS in mesh.dirs else lh[1])
        branch = tuple(range(0, fabric.k, 2)) if PLUS in mesh.dirs else tuple(range(1, fabric.k, 2))
        bl = fabric.all_gather(rank, mine, tag="loss", group=branch)
        pair = (2 * mesh.group, 2 * mesh.group + 1)
        both = [fabric.all_gather(rank, v, tag="loss", group=pair) for v in bl]
        plus = [b[0] for b in both]
        minus = [b[1] for b in both]
        total = 0.0
        for i in range(mesh.n_groups):
            total += (plus[i] - minus[i]) / (2.0 * eps)
        g = total / mesh.n_groups
        rec = (plus[mesh.group], minus[mesh.group], g)
    else:
        raise ConfigurationError(f"unknown mesh ordering {ordering!r}")
    # eager update theta -= (lr g) z on every rank (strategies.py:81-83)
    store.set_pending(hyper.lr * g, seed, True)
    store.run(store.perturb_call(store.model_table, L.ZO_PU_UPDATE, 0.0, 0.0, sa=None, sb=None, zmode=zmode,
                                 z_prev=zc))
    store.scal[3:4].fill_(0)
    torch.cuda.current_stream().synchronize()
    if verify:
        check_replicas(fabric, rank, store)
    return ZoStep(iteration, seed, rec[0], rec[1], rec[2])


def pertp_step(fabric, rank, store, batch, hyper, seed, mgr=None, iteration=1, verify=True) -> ZoStep:
    """Direction parallelism on exactly two ranks (strategies.py:92-125)."""
    if fabric.k != 2:
        raise ConfigurationError(f"direction parallelism needs exactly 2 workers, got {fabric.k}")
    return _eager_step(fabric, rank, store, batch, hyper, seed, "pertp", mgr, iteration, verify)


def ddp_step(fabric, rank, store, shard, hyper, seed, mgr=None, iteration=1, verify=True) -> ZoStep:
    """ZO-DDP (strategies.py:128-151): g = ordered mean of per-shard g."""
    return _eager_step(fabric, rank, store, shard, hyper, seed, "ddp", mgr, iteration, verify)


def twod_step(fabric, rank, assign, store, shard, hyper, seed, ordering="pertp_inner", mgr=None, iteration=1,
              verify=True) -> ZoStep:
    """n_groups x 2 mesh (strategies.py:154-222)."""
    if ordering not in ("pertp_inner", "ddp_inner"):
        raise ConfigurationError(f"unknown mesh ordering {ordering!r}")
    if fabric.k != 2 * assign.n_groups:
        raise ConfigurationError(f"mesh needs {2 * assign.n_groups} ranks (= {assign.n_groups} groups x 2), "
                                 f"fabric has {fabric.k}")
    return _eager_step(fabric, rank, store, shard, hyper, seed, "2d", mgr, iteration, verify, ordering)
