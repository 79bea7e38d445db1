"""Zeroth-order optimizer API on the GPU (mirror of src/zosim/zo.py).

Same names, arguments and error behaviour as the reference:

  ZoHyper, ZoStep, zo_grad                       zo.py:42-84
  perturb_block / perturb_params                 zo.py:90-113
  update_block / update_params                   zo.py:116-130
  mezo_step  (Alg. 1, eager)                     zo.py:136-168
  dual_forward (Alg. 2, one block)               zo.py:181-224
  flush_pending_update, StreamingZo (lazy)       zo.py:227-293

What differs is where the work happens: parameters are the fp32 master
``store.theta`` on the GPU; a perturbation writes the bf16/fp32 shadows the
forward kernels read (never the master, so restore is free and exact); the
whole-model step is ONE fused perturb/update launch + two forwards + a device
projected-gradient kernel, with the update of step j folded into the
perturbation pass of step j+1 (StreamingZo) or applied eagerly (mezo_step).

``mgr`` selects the direction source: RngStateManager("philox") (default,
in-register counter-based z) or RngStateManager("oracle") (the reference's
numpy PCG64 z injected; perturb/update arithmetic then matches the reference
bit for bit).
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .engine import MINUS, PLUS, DeviceStore
from .errors import DimensionError, NumericError, ProtocolError
from .model import EMBEDDING, HEAD, Batch
from .rng import PhiloxKey, RngStateManager


@dataclass(frozen=True)
class ZoHyper:
    epsilon: float
    lr: float
    steps: int = 1

    def validate(self) -> "ZoHyper":
        if not self.epsilon > 0:
            raise NumericError(f"epsilon must be > 0, got {self.epsilon}")
        if not self.lr > 0:
            raise NumericError(f"lr must be > 0, got {self.lr}")
        if self.steps < 1:
            raise NumericError(f"steps must be >= 1, got {self.steps}")
        return self


@dataclass
class ZoStep:
    iteration: int
    seed: int
    loss_pos: float
    loss_neg: float
    g: float

    def to_json(self) -> str:
        return json.dumps({"iter": self.iteration, "seed": self.seed, "loss_pos": self.loss_pos,
                           "loss_neg": self.loss_neg, "g": self.g})


def zo_grad(loss_pos: float, loss_neg: float, epsilon: float) -> float:
    if epsilon == 0:
        raise NumericError("epsilon must be nonzero")
    return (loss_pos - loss_neg) / (2.0 * epsilon)


# ---------------------------------------------------------------------------
# scalar staging helpers
# ---------------------------------------------------------------------------

def _u64_as_i64(x: int) -> int:
    return int(np.uint64(int(x) & ((1 << 64) - 1)).view(np.int64))


def _scal_tensor(device, seed_cur=0, seed_prev=0, lr_g=0.0, pending=0) -> torch.Tensor:
    h = np.zeros(4, dtype=np.int64)
    h[0], h[1] = _u64_as_i64(seed_cur), _u64_as_i64(seed_prev)
    h[2] = np.float64(lr_g).view(np.int64)
    h[3] = pending
    return torch.from_numpy(h).to(device)


def _write_scal(store: DeviceStore, seed_cur: int, pending: bool) -> None:
    """Host writes the iteration seed; keeps seed_prev / lr_g_prev left by
    the device gradient kernel and sets the pending flag explicitly
    (zo.py:267-271: a flag, not g != 0)."""
    store.scal[0:1].fill_(_u64_as_i64(seed_cur))
    store.scal[3:4].fill_(1 if pending else 0)


def _oracle_z(mgr: RngStateManager, seed: int, n: int, device) -> torch.Tensor:
    mgr.reset(seed)
    return torch.from_numpy(mgr.generator(seed).standard_normal(n)).to(device)


def _stage_batch(store: DeviceStore, batch: Batch):
    batch.validate(store.config)
    B, T = batch.token_ids.shape
    wsp, wsn = store.workspace(PLUS, B, T), store.workspace(MINUS, B, T)
    store.load_batch(wsp, batch.token_ids, batch.targets)     # ids/targets are shared by both
    return wsp, wsn


def _finish(store: DeviceStore, wsp, wsn, iteration: int, seed: int) -> ZoStep:
    return _finish_record(store, [wsp, wsn], iteration, seed)


def _finish_record(store: DeviceStore, wss, iteration: int, seed: int) -> ZoStep:
    lp, ln, g = store.read_step(list(wss))     # one D2H + one sync
    return ZoStep(iteration, seed, lp, ln, g)


# ---------------------------------------------------------------------------
# whole-model steps (the hot path)
# ---------------------------------------------------------------------------

def mezo_step(store: DeviceStore, batch: Batch, hyper: ZoHyper, seed: int, mgr: RngStateManager | None = None,
              iteration: int = 1) -> ZoStep:
    """Alg. 1 (zo.py:136-168): L+ at theta+eps z, L- at theta-eps z, g, then
    theta -= (lr g) z before returning."""
    hyper.validate()
    mgr = mgr or RngStateManager()
    eps = hyper.epsilon
    wsp, wsn = _stage_batch(store, batch)
    zc = _oracle_z(mgr, seed, store.total_params, store.device) if mgr.oracle else None
    zmode = L.ZO_Z_ORACLE if mgr.oracle else L.ZO_Z_PHILOX
    _write_scal(store, seed, pending=False)
    t = store.model_table
    calls = store.perturb_call(t, L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B, +eps, -eps, zmode=zmode, z_cur=zc)
    calls += store.forward_calls(PLUS, wsp, +eps, zmode=zmode, z_cur=zc)
    calls += store.forward_calls(MINUS, wsn, -eps, zmode=zmode, z_cur=zc)
    calls += store.grad_call(wsp, wsn, eps, hyper.lr)
    calls += store.perturb_call(t, L.ZO_PU_UPDATE, 0.0, 0.0, sa=None, sb=None, zmode=zmode, z_prev=zc)
    store.run(calls)
    store.scal[3:4].fill_(0)                  # the update has been applied
    return _finish(store, wsp, wsn, iteration, seed)


class StreamingZo:
    """Lazy-update executor (zo.py:245-293): the update of iteration j is
    folded into iteration j+1's perturbation pass; ``flush`` applies the last
    one.  Numerically identical to repeated ``mezo_step`` after flush."""

    def __init__(self, store: DeviceStore, hyper: ZoHyper, mgr: RngStateManager | None = None,
                 overlap: bool | str = "fill", graph: bool = True):
        self.store = store
        self.hyper = hyper.validate()
        self.mgr = mgr or RngStateManager()
        # "stacked" (default): the fused pass, then both directional forwards
        # as one launch per layer over stacked activations; False / "none":
        # the fused pass, then the two forwards on two streams (also the plan
        # for shapes the stacked GEMMs cannot split and for oracle-z runs).
        # Both plans give identical results.
        # "fill": the stacked forward on a high-priority stream while the
        # perturb pass of blocks 2.. runs block by block as short-lived CTAs on
        # a low-priority stream, each block's forward waiting only for its own
        # block's pass -- the pass fills the SMs the forward's kernels leave
        # idle (partial waves, launch gaps) instead of running before it.
        if overlap not in (False, None, "none", "stacked", "fill"):
            raise ProtocolError(f"unknown step plan {overlap!r} (plans: 'stacked', 'fill', 'none')")
        self.overlap = overlap if (overlap in ("stacked", "fill") and not self.mgr.oracle) else None
        self.dual_stream = True
        # Philox steps replay one captured CUDA graph per batch shape (the
        # step's scalars are device-resident, so the launches never change)
        self.graph = graph and not self.mgr.oracle
        self._graphs = {}
        self._ios = {}             # batch rows -> pinned staging of the I/O-carrying graph
        self.iteration = 0
        self._g_prev = 0.0
        self.last_seed = None
        self._pending = False
        self._z_prev = None

    @property
    def g_prev(self) -> float:
        return self._g_prev

    @g_prev.setter
    def g_prev(self, g: float) -> None:
        """The reference's next step / flush applies ``self.g_prev``
        (zo.py:267-293); replacing it replaces the device's lr * g_prev too."""
        self._g_prev = float(g)
        self.store.scal[2:3].fill_(int(np.float64(self.hyper.lr * float(g)).view(np.int64)))

    def step_calls(self, wsp, wsn, zc=None, zp=None, update=True):
        """One lazy step: fused (update_{j-1} + perturb_j) pass, both
        directional forwards, device projected gradient.  With update=True the
        kernel applies the pending update iff the device flag says so, which is
        what lets a captured graph replay steps unchanged."""
        s, eps = self.store, self.hyper.epsilon
        zmode = L.ZO_Z_ORACLE if self.mgr.oracle else L.ZO_Z_PHILOX
        flags = (L.ZO_PU_UPDATE if update else 0) | L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B
        calls = s.perturb_call(s.model_table, flags, +eps, -eps, zmode=zmode, z_cur=zc, z_prev=zp)
        if self.dual_stream:
            # the two directional forwards are independent: run -eps on a side
            # stream so each fills the other's partial GEMM waves
            main, side = torch.cuda.current_stream(), _side_stream(s)
            ev = _block_events(s, len(s.layouts))
            calls.append((_record_and_wait, (ev[0], main, side)))
            calls += s.forward_calls(PLUS, wsp, +eps, zmode=zmode, z_cur=zc)
            calls += s.forward_calls(MINUS, wsn, -eps, zmode=zmode, z_cur=zc, stream=side)
            calls.append((_record_and_wait, (ev[1], side, main)))
        else:
            calls += s.forward_calls(PLUS, wsp, +eps, zmode=zmode, z_cur=zc)
            calls += s.forward_calls(MINUS, wsn, -eps, zmode=zmode, z_cur=zc)
        calls += s.grad_call(wsp, wsn, eps, self.hyper.lr)
        return calls

    def stacked_step_calls(self, wsp, wsn):
        """Same step with both directional forwards as ONE launch per layer
        over stacked [+eps; -eps] activations (DeviceStore.forward_calls_stacked):
        every GEMM fills twice the tiles, so the partial last wave and each
        launch's prologue / tail are paid once per layer, not once per
        direction.  Bit-identical to step_calls (same per-tile arithmetic)."""
        if self.mgr.oracle:
            raise ProtocolError("the stacked plan runs the Philox direction only")
        s, eps = self.store, self.hyper.epsilon
        ws = s.stacked_workspace(wsp.batch, wsp.seq)
        flags = L.ZO_PU_UPDATE | L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B
        calls = s.perturb_call(s.model_table, flags, +eps, -eps)
        calls += s.forward_calls_stacked(ws, eps)
        calls += s.grad_call_stacked(ws, eps, self.hyper.lr)
        return calls

    def fill_step_calls(self, wsp, wsn):
        """The stacked step with the perturb pass split by block: embedding +
        block 1 at full speed on the forward's (high-priority) stream, blocks
        2.. and the head as ZO_PU_FILL launches on a low-priority stream, one
        event per block; block b's forward waits for block b's event only.
        Same per-element arithmetic as stacked_step_calls (bit-identical)."""
        if self.mgr.oracle:
            raise ProtocolError("the fill plan runs the Philox direction only")
        s, eps = self.store, self.hyper.epsilon
        ws = s.stacked_workspace(wsp.batch, wsp.seq)
        nl = len(s.layouts)
        main = torch.cuda.current_stream()
        hi, lo = _priority_streams(s)
        ev = _block_events(s, nl + 3)          # [b] block b's pass done; [nl] start; [nl+1], [nl+2] joins
        flags = L.ZO_PU_UPDATE | L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B
        calls = [(_record_and_wait, (ev[nl], main, hi)), (_wait, (lo, ev[nl]))]
        calls += s.perturb_call(s.head_table(), flags, +eps, -eps, stream=hi)
        for b in range(2, nl):
            calls += s.perturb_call(s.block_tables[b], flags | L.ZO_PU_FILL, +eps, -eps, stream=lo)
            calls.append((_record, (ev[b], lo)))
        calls += s.forward_calls_stacked(ws, eps, stream=hi, blocks=[0, 1])
        for b in range(2, nl):
            calls.append((_wait, (hi, ev[b])))
            calls += s.forward_calls_stacked(ws, eps, stream=hi, blocks=[b])
        calls += s.grad_call_stacked(ws, eps, self.hyper.lr, stream=hi)
        calls.append((_record_and_wait, (ev[nl + 1], hi, main)))
        calls.append((_record_and_wait, (ev[nl + 2], lo, main)))
        return calls

    def _stacked_ok(self, wsp):
        return self.overlap in ("stacked", "fill") and self.store.stackable(wsp.batch, wsp.seq)

    def _plan(self, wsp, wsn, zc=None, zp=None, update=True):
        if self._stacked_ok(wsp):
            if self.overlap == "fill":
                return self.fill_step_calls(wsp, wsn)
            return self.stacked_step_calls(wsp, wsn)
        return self.step_calls(wsp, wsn, zc, zp, update=update)

    def _replay(self, wsp, wsn, io: bool = False):
        """Capture the step's launches once per (batch shape, plan) -- the
        first step ran eagerly, so one-time kernel attributes and TMA
        descriptors already exist -- then replay the graph on the current
        stream.  io=False: the caller uploaded the batch and seed; io=True
        (the public step): the graph itself copies the batch / seed / pending
        flag in from pinned staging and the record / error flags back out."""
        key = (wsp.batch, wsp.seq, self.overlap, self.dual_stream, io)
        g = self._graphs.get(key)
        if g is None:
            def build():
                calls = self._plan(wsp, wsn)
                if io:
                    cin, cout = self._io_calls(wsp)
                    calls = cin + calls + cout
                return calls

            if self.overlap == "fill" and self._stacked_ok(wsp):
                g = NativeGraph(self.store.run, build)          # replays with launch priorities
            else:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    self.store.run(build())                     # stream handles bound inside the capture
            self._graphs[key] = g
        g.replay()

    def _io_bufs(self, wsp):
        """Pinned staging of the graph-carried step I/O for M = B*T rows:
        ids / targets in, (seed, pending) in, the ZoStep record and the
        workspaces' error flags out."""
        # one staging set per batch shape, alive as long as the graphs that captured its pointers
        io = self._ios.get(wsp.M)
        if io is None:
            io = self._ios[wsp.M] = {"M": wsp.M,
                                     "ids": torch.empty(2, wsp.M, dtype=torch.int32, pin_memory=True),
                                     "scal": torch.zeros(2, dtype=torch.int64, pin_memory=True),
                                     "rec": torch.zeros(3, dtype=torch.float64, pin_memory=True),
                                     "err": torch.zeros(4, dtype=torch.int32, pin_memory=True)}
        return io

    def _io_wss(self, wsp, wsn):
        wss = [wsp, wsn]
        if self._stacked_ok(wsp):
            wss.append(self.store.stacked_workspace(wsp.batch, wsp.seq))
        return wss

    def _io_calls(self, wsp):
        """(in, out) copy launches of the I/O-carrying graph, on the capture stream."""
        s, lib, st = self.store, L.lib(), L.stream_ptr()
        io = self._io_bufs(wsp)
        B, T = wsp.batch, wsp.seq
        wsn = s.workspace(MINUS, B, T)
        nb = 4 * wsp.M
        cin = [(lib.zo_copy_async, (wsp.ids.data_ptr(), io["ids"].data_ptr(), nb, st)),
               (lib.zo_copy_async, (wsp.tgt.data_ptr(), io["ids"].data_ptr() + nb, nb, st)),
               (lib.zo_copy_async, (s.scal.data_ptr(), io["scal"].data_ptr(), 8, st)),           # seed_cur
               (lib.zo_copy_async, (s.scal.data_ptr() + 24, io["scal"].data_ptr() + 8, 8, st))]  # pending
        cout = [(lib.zo_copy_async, (io["rec"].data_ptr(), s.record.data_ptr(), 24, st))]
        for i, ws in enumerate(self._io_wss(wsp, wsn)):
            cout.append((lib.zo_copy_async, (io["err"].data_ptr() + 4 * i, ws.err.data_ptr(), 4, st)))
        return cin, cout

    def _step_graph_io(self, batch: Batch, seed: int, pending: bool) -> ZoStep:
        """A replayed step whose graph carries its own I/O: the host fills
        pinned memory, launches once, synchronises once and reads pinned memory."""
        s = self.store
        batch.validate(s.config)
        ids, tg = np.asarray(batch.token_ids), np.asarray(batch.targets)
        B, T = ids.shape
        wsp, wsn = s.workspace(PLUS, B, T), s.workspace(MINUS, B, T)
        if tg.shape != ids.shape:
            raise DimensionError(f"targets shape {tg.shape} does not match ids {ids.shape}")
        if ids.size and (ids.min() < 0 or ids.max() >= s.config.vocab_size):
            raise DimensionError("token id out of embedding range")
        io = self._io_bufs(wsp)
        h = io["ids"].numpy()
        h[0] = ids.reshape(-1)
        h[1] = tg.reshape(-1)
        io["scal"].numpy()[:] = (_u64_as_i64(seed), 1 if pending else 0)
        self._replay(wsp, wsn, io=True)
        torch.cuda.current_stream().synchronize()
        wss = self._io_wss(wsp, wsn)
        errs = [int(v) for v in io["err"].numpy()[:len(wss)]]
        s.check_errors(*wss, flags=errs)
        r = io["rec"].numpy()
        return ZoStep(self.iteration, seed, float(r[0]), float(r[1]), float(r[2]))

    def step(self, batch: Batch, seed: int) -> ZoStep:
        self.iteration += 1
        self.mgr.reset(seed)
        self.mgr.push_state(self.mgr.capture(seed))
        apply_pending = self.iteration > 1 and self._pending
        if apply_pending:
            self.mgr.pop_state()
        try:
            if self.graph and self.iteration > 1:
                st = self._step_graph_io(batch, seed, apply_pending)
                zc = None
            else:
                wsp, wsn = _stage_batch(self.store, batch)
                zc = _oracle_z(self.mgr, seed, self.store.total_params, self.store.device) if self.mgr.oracle else None
                _write_scal(self.store, seed, pending=apply_pending)
                self.store.run(self._plan(wsp, wsn, zc, self._z_prev if apply_pending else None,
                                          update=apply_pending or not self.mgr.oracle))
                st = _finish_record(self.store, self._io_wss(wsp, wsn), self.iteration, seed)
        except NumericError:
            # the step's pass consumed the pending update and the device did
            # not arm a new one (zo_grad_finalize gates on a finite g), so
            # nothing is pending: flush / the next step must not re-apply one
            self.mgr.pop_state()
            self._pending, self.store.unflushed = False, False
            raise
        self._g_prev, self.last_seed, self._pending, self._z_prev = st.g, seed, True, zc
        self.store.unflushed = True
        return st

    def flush(self) -> None:
        if not self._pending:
            raise ProtocolError("flush with no pending update (double flush?)")
        self.mgr.pop_state()
        s = self.store
        zmode = L.ZO_Z_ORACLE if self.mgr.oracle else L.ZO_Z_PHILOX
        # the update uses self.g_prev like zo.py:287-293 (equal to the device's
        # lr*g unless the caller replaced it; both are the same f64 product)
        s.set_pending(self.hyper.lr * self.g_prev, self.last_seed, True)
        s.run(s.perturb_call(s.model_table, L.ZO_PU_UPDATE, 0.0, 0.0, sa=None, sb=None, zmode=zmode,
                             z_prev=self._z_prev))
        s.scal[3:4].fill_(0)
        torch.cuda.current_stream().synchronize()
        self._pending = False
        self.store.unflushed = False


def _side_stream(store: DeviceStore):
    return store.side_stream()


def _block_events(store: DeviceStore, n: int):
    return store.block_events(n)


def _record_and_wait(ev, main, side):
    ev.record(main)
    side.wait_event(ev)
    return 0


def _record(ev, stream):
    ev.record(stream)
    return 0


def _wait(stream, ev):
    stream.wait_event(ev)
    return 0


def _priority_streams(store: DeviceStore):
    """(high, low) priority streams of the fill plan (lower number = higher)."""
    return store.priority_streams()


class NativeGraph:
    """A step captured with the library's own graph API (zo_graph_*): unlike
    torch.cuda.CUDAGraph it instantiates with per-node priorities, so the
    fill plan's low-priority pass keeps yielding SMs on replay.  Capture runs
    on a private stream forked from the caller's; replay on the current one."""

    def __init__(self, run, build):
        import ctypes
        self._lib = L.lib()
        cur = torch.cuda.current_stream()
        cap = torch.cuda.Stream(device=cur.device)
        cap.wait_stream(cur)
        self.exec = ctypes.c_void_p()
        with torch.cuda.stream(cap):
            L.check(self._lib.zo_graph_begin(L.stream_ptr(cap)))
            try:
                run(build())          # the plan binds the capture stream as its "current" stream
            finally:
                rc = self._lib.zo_graph_end(L.stream_ptr(cap), ctypes.byref(self.exec))
            L.check(rc)
        cur.wait_stream(cap)

    def replay(self):
        L.check(self._lib.zo_graph_launch(self.exec, L.stream_ptr(torch.cuda.current_stream())))

    def __del__(self):
        try:
            if self.exec:
                self._lib.zo_graph_destroy(self.exec)
        except Exception:
            pass


def flush_pending_update(store: DeviceStore, g_last: float, seed: int, mgr: RngStateManager, lr: float) -> None:
    """zo.py:227-242: apply the deferred update of the most recent iteration
    to every block."""
    try:
        mgr.pop_state()
    except ProtocolError as e:
        raise ProtocolError("flush with no pending update (double flush?)") from e
    update_params(store, g_last, lr, mgr.generator(seed) if not mgr.oracle else _restart(mgr, seed))


def _restart(mgr, seed):
    mgr.reset(seed)
    return mgr.generator(seed)


# ---------------------------------------------------------------------------
# per-block API (API parity with the reference; the step above is the fast path)
# ---------------------------------------------------------------------------

class DeviceBlock:
    """One block of a DeviceStore, shaped like zosim.ParamBlock
    (model.py:104-157): ``buf`` is the fp32 master view on the GPU."""

    def __init__(self, store: DeviceStore, block_id: int):
        self.store, self.block_id = store, block_id
        bl = store.layouts[block_id]
        self.kind, self.names, self.offsets, self.elem_count = bl.kind, bl.names, bl.offsets, bl.elem_count
        self.shapes = bl.shapes
        self.key0 = bl.key0
        self.n_heads = store.config.n_heads
        self.pert_scale = 0.0
        self._zsrc = (L.ZO_Z_PHILOX, None, 0)     # (mode, z tensor | seed, z_key0) of the open cycle

    @property
    def buf(self) -> torch.Tensor:
        return self.store.block_buf(self.block_id)

    def tensor(self, name: str) -> torch.Tensor:
        o = self.offsets[name]
        n = int(np.prod(self.shapes[name]))
        return self.buf[o:o + n].view(self.shapes[name])

    @property
    def nbytes(self) -> int:
        return self.elem_count * 4

    @property
    def dtype(self):
        return torch.float32

    def spec(self):
        return [(n, self.shapes[n]) for n in self.names]

    def copy(self) -> torch.Tensor:
        """ParamBlock.copy (model.py:152-157): the block's master values;
        refused mid-perturbation."""
        if self.pert_scale != 0.0:
            raise ProtocolError(f"block {self.block_id} copied mid-perturbation")
        return self.buf.clone()


def store_blocks(store: DeviceStore):
    if not hasattr(store, "_blocks"):
        store._blocks = [DeviceBlock(store, i) for i in range(len(store.layouts))]
    return store._blocks


def _draw(block: DeviceBlock, gen):
    """(zmode, z tensor, seed) for one block; a numpy Generator is advanced
    by exactly elem_count draws, like zo.py:96/124."""
    if isinstance(gen, PhiloxKey):
        return L.ZO_Z_PHILOX, None, gen.seed
    if isinstance(gen, np.random.Generator):
        return L.ZO_Z_ORACLE, torch.from_numpy(gen.standard_normal(block.elem_count)).to(block.store.device), 0
    raise DimensionError(f"unsupported direction source {type(gen).__name__}")


def perturb_block(block: DeviceBlock, scale: float, gen) -> None:
    """zo.py:90-107: the block's forward view becomes base + cumulative_scale * z
    (computed from the untouched master, so closing the cycle is exact)."""
    s = block.store
    zmode, z, seed = _draw(block, gen)
    new_scale = block.pert_scale + scale
    scal = _scal_tensor(s.device, seed_cur=seed)
    t = s.block_tables[block.block_id]
    fn = L.lib().zo_perturb_update
    rc = fn(s.theta.data_ptr(), 0, t.segs.data_ptr(), t.prefix.data_ptr(), t.n_segs, t.n_tiles,
            s.wsh[PLUS].data_ptr(), s.vsh[PLUS].data_ptr(), 0, 0, float(new_scale), 0.0, L.ZO_PU_SHADOW_A,
            scal.data_ptr(), zmode, 0 if z is None else z.data_ptr(), 0, block.key0, L.stream_ptr())
    L.check(rc)
    block.pert_scale = new_scale
    block._zsrc = (zmode, z if z is not None else seed, block.key0)
    block._keepalive = scal


def _refresh_view(block: DeviceBlock) -> None:
    s = block.store
    scal = _scal_tensor(s.device)
    t = s.block_tables[block.block_id]
    L.check(L.lib().zo_perturb_update(s.theta.data_ptr(), 0, t.segs.data_ptr(), t.prefix.data_ptr(), t.n_segs,
                                      t.n_tiles, s.wsh[PLUS].data_ptr(), s.vsh[PLUS].data_ptr(), 0, 0, 0.0, 0.0,
                                      L.ZO_PU_SHADOW_A, scal.data_ptr(), L.ZO_Z_PHILOX, 0, 0, 0, L.stream_ptr()))
    block._keepalive = scal


def perturb_params(store: DeviceStore, scale: float, gen) -> None:
    for b in store_blocks(store):
        perturb_block(b, scale, gen)


def update_block(block: DeviceBlock, g: float, lr: float, gen) -> None:
    """zo.py:116-125: theta <- theta - (lr*g) z, refused mid-perturbation."""
    if block.pert_scale != 0.0:
        raise ProtocolError(f"block {block.block_id} updated while a perturbation cycle is open "
                            f"(cumulative scale {block.pert_scale})")
    s = block.store
    zmode, z, seed = _draw(block, gen)
    scal = _scal_tensor(s.device, seed_prev=seed, lr_g=lr * g, pending=1)
    t = s.block_tables[block.block_id]
    rc = L.lib().zo_perturb_update(s.theta.data_ptr(), 0, t.segs.data_ptr(), t.prefix.data_ptr(), t.n_segs,
                                   t.n_tiles, 0, 0, 0, 0, 0.0, 0.0, L.ZO_PU_UPDATE, scal.data_ptr(), zmode, 0,
                                   0 if z is None else z.data_ptr(), block.key0, L.stream_ptr())
    L.check(rc)
    torch.cuda.current_stream().synchronize()


def update_params(store: DeviceStore, g: float, lr: float, gen) -> None:
    for b in store_blocks(store):
        update_block(b, g, lr, gen)


def forward_block(block: DeviceBlock, x) -> torch.Tensor:
    """model.py:298-346 on the block's current (possibly perturbed) view.
    Embedding takes token ids [B, T]; others take fp32 activations [B, T, d]
    on the device; the head returns fp32 logits [B, T, V]."""
    s, cfg = block.store, block.store.config
    if block.kind == EMBEDDING:
        ids = np.asarray(x.cpu() if torch.is_tensor(x) else x)
        if ids.ndim != 2 or not np.issubdtype(ids.dtype, np.integer):
            raise DimensionError("embedding block expects integer token ids of shape (batch, seq)")
        B, T = ids.shape
        if T > cfg.seq_len:
            raise DimensionError(f"sequence length {T} exceeds positions {cfg.seq_len}")
        ws = s.workspace(PLUS, B, T)
        s.load_batch(ws, ids, np.zeros_like(ids))
    else:
        if not torch.is_tensor(x) or x.dim() != 3 or x.shape[2] != cfg.d_model:
            raise DimensionError(f"{block.kind} block expects activations of shape (batch, seq, {cfg.d_model})")
        B, T = x.shape[0], x.shape[1]
        ws = s.workspace(PLUS, B, T)
        ws.x[:, :cfg.d_model].copy_(x.reshape(B * T, cfg.d_model))
    if block.kind != EMBEDDING and block.pert_scale == 0.0:
        _refresh_view(block)          # unperturbed view = bf16/fp32 copy of the master
    if block.kind == HEAD and cfg.arch == "opt":
        emb = store_blocks(s)[0]      # tied head: reads the embedding block's current view
        if emb.pert_scale == 0.0:
            _refresh_view(emb)
    zmode, zsrc, zkey0 = block._zsrc
    logits = None
    if block.kind == HEAD:
        logits = torch.empty(B * T, cfg.vocab_size, dtype=torch.float32, device=s.device)
    calls = s.forward_calls(PLUS, ws, 0.0, blocks=[block.block_id], head_mode="logits", logits=logits)
    if block.kind == EMBEDDING and block.pert_scale != 0.0:
        fn, args = calls[0]
        args = list(args)
        args[9] = float(block.pert_scale)
        if zmode == L.ZO_Z_PHILOX:
            scal = _scal_tensor(s.device, seed_cur=zsrc)
            args[10], args[11] = scal.data_ptr(), L.ZO_Z_PHILOX
            block._keepalive2 = scal
        else:
            args[11], args[12], args[13] = L.ZO_Z_ORACLE, zsrc.data_ptr(), zkey0
        calls = [(fn, tuple(args))]
    s.run(calls)
    if block.kind == HEAD:
        if cfg.arch != "opt":
            logits += s.vview(PLUS, block.block_id, "b_out")
        return logits.view(B, T, cfg.vocab_size)
    s.check_errors(ws)
    return ws.x[:, :cfg.d_model].clone().view(B, T, cfg.d_model)


def forward(store: DeviceStore, token_ids) -> torch.Tensor:
    """Full-model logits at the current (unperturbed or perturbed) views."""
    x = token_ids
    for b in store_blocks(store):
        x = forward_block(b, x)
    return x


def loss(logits: torch.Tensor, batch: Batch) -> float:
    """Mean CE over all positions in f64 (model.py:357-372)."""
    if logits.dim() != 3:
        raise DimensionError(f"logits must be (batch, seq, vocab), got shape {tuple(logits.shape)}")
    tg = torch.as_tensor(np.asarray(batch.targets), device=logits.device).long()
    if tuple(logits.shape[:2]) != tuple(tg.shape):
        raise DimensionError("logits shape does not match targets")
    l64 = logits.double()
    if not torch.isfinite(l64).all():
        raise NumericError("non-finite logits")
    lse = torch.logsumexp(l64, dim=-1)
    picked = l64.gather(-1, tg[..., None])[..., 0]
    return float((lse - picked).mean())


def dual_forward(block: DeviceBlock, hyper: ZoHyper, seed: int, mgr: RngStateManager, rs, lrs, g_prev: float,
                 input_pos, input_neg, apply_pending: bool):
    """Alg. 2 for one block (zo.py:181-224): optional deferred update, then
    the +eps and -eps forwards and the closing restore."""
    eps = hyper.epsilon
    if apply_pending:
        if lrs is None:
            raise ProtocolError(f"block {block.block_id}: pending update but no previous-iteration RNG state")
        mgr.restore(seed, lrs)
        update_block(block, g_prev, hyper.lr, mgr.generator(seed))
        lrs = mgr.capture(seed)
    mgr.restore(seed, rs)
    perturb_block(block, +eps, mgr.generator(seed))
    out_pos = forward_block(block, input_pos)
    mgr.restore(seed, rs)
    perturb_block(block, -2.0 * eps, mgr.generator(seed))
    out_neg = forward_block(block, input_neg)
    mgr.restore(seed, rs)
    perturb_block(block, +eps, mgr.generator(seed))
    rs = mgr.capture(seed)
    return out_pos, out_neg, rs, lrs
