"""Device-resident ZO engine: parameter master, shadow layout, workspaces and
the launch plans of the perturb / dual-forward / projected-gradient step.

HBM layout (one GPU, resident model):
  theta       fp32 [P]  master in the reference's (block, tensor, element)
              order; element index == global key of the direction z
  wsh[s]      bf16      perturbed GEMM operands for direction s (s=0: +eps,
              s=1: -eps); each weight keeps the reference's (d_in, d_out)
              row-major layout, wq|wk|wv are interleaved into one
              [d, 3d] operand so QKV is a single GEMM
  vsh[s]      fp32      perturbed LN gains/biases and GEMM biases
  (embedding) no shadow: the gather kernel perturbs the rows it reads
  scal        ZoStepScalars (device) - seeds, lr*g_prev, pending flag
Per-direction workspace: x fp32 [M,d] residual stream, h/ctx bf16 [M,d],
qkv bf16 [M,3d], ff bf16 [M,4d], CE partials [M, V/256, 2].

Every launch is a ctypes call into libzo_b200.so with precomputed integer
arguments ("launch plans"), so a step costs ~one Python call per kernel and
can be captured into a CUDA graph.
"""

from __future__ import annotations

import ctypes as C


import numpy as np
import torch

from . import _lib as L
from .errors import ConfigurationError, DimensionError, NumericError
from .model import EMBEDDING, HEAD, TRANSFORMER, ModelConfig, init_block_host, model_layout

PLUS, MINUS = 0, 1


def _r8(x: int) -> int:
    return (x + 7) // 8 * 8


def _a64(x: int) -> int:
    return (x + 63) // 64 * 64


class ShadowPlan:
    """Where each tensor's perturbed copy lives, and the perturb kernel's
    segment tables (per block and for the whole model)."""

    def __init__(self, config: ModelConfig, layouts, f32_weights: bool = False):
        d, v = config.d_model, config.vocab_size
        self.config = config
        self.f32_weights = f32_weights       # f32 parity mode: weight shadows are fp32 too (in vsh)
        self.w_elems = 0
        self.v_elems = 0
        self.views = {}       # bid -> name -> (buffer 'w'|'v', offset, rows, cols, ld)
        self.segments = {}    # bid -> [ZoSegment fields]

        def walloc(rows, cols):
            ld = _r8(cols)
            if f32_weights:
                off = _a64(self.v_elems)
                self.v_elems = off + rows * ld
                return off, ld
            off = _a64(self.w_elems)
            self.w_elems = off + rows * ld
            return off, ld

        wbuf = "v" if f32_weights else "w"
        wkind = L.ZO_SHADOW_F32 if f32_weights else L.ZO_SHADOW_BF16

        def valloc(n):
            off = (self.v_elems + 3) // 4 * 4
            self.v_elems = off + n
            return off

        tied = config.arch == "opt"     # real OPT: the LM head reads the token embedding
        for bl in layouts:
            vw, segs = {}, []
            if bl.kind == EMBEDDING:
                if tied:
                    # bf16 shadow of tok_emb [V, d] = the head's K-major B operand;
                    # the gather still perturbs the fp32 rows it reads
                    o, ld = walloc(v, d)
                    vw["tok_emb"] = (wbuf, o, v, d, ld)
                for name in bl.names:
                    if tied and name == "tok_emb":
                        segs.append((bl.key(name), v, d, o, ld, wkind) if ld != d else
                                    (bl.key(name), 1, v * d, o, v * d, wkind))
                    else:
                        segs.append((bl.key(name), 1, bl.size(name), 0, bl.size(name), L.ZO_SHADOW_NONE))
            elif bl.kind == TRANSFORMER:
                qo, qld = walloc(d, 3 * d)
                vw["qkv"] = (wbuf, qo, d, 3 * d, qld)
                for name, (r, c) in (("wo", (d, d)), ("w1", (d, 4 * d)), ("w2", (4 * d, d))):
                    o, ld = walloc(r, c)
                    vw[name] = (wbuf, o, r, c, ld)
                for name, n in (("ln1_g", d), ("ln1_b", d), ("bqkv", 3 * d), ("bo", d), ("ln2_g", d),
                                ("ln2_b", d), ("b1", 4 * d), ("b2", d)):
                    vw[name] = ("v", valloc(n), 1, n, n)
                for name in bl.names:
                    k, n = bl.key(name), bl.size(name)
                    if name in ("wq", "wk", "wv"):
                        j = "qkv".index(name[1])
                        segs.append((k, d, d, qo + j * d, qld, wkind))
                    elif name in ("bq", "bk", "bv"):
                        j = "qkv".index(name[1])
                        segs.append((k, 1, d, vw["bqkv"][1] + j * d, d, L.ZO_SHADOW_F32))
                    elif name in ("wo", "w1", "w2"):
                        _, o, r, c, ld = vw[name]
                        if ld == c:
                            segs.append((k, 1, r * c, o, r * c, wkind))
                        else:
                            segs.append((k, r, c, o, ld, wkind))
                    else:
                        segs.append((k, 1, n, vw[name][1], n, L.ZO_SHADOW_F32))
            elif tied:  # real-OPT head: final LayerNorm only
                for name in bl.names:
                    vw[name] = ("v", valloc(d), 1, d, d)
                    segs.append((bl.key(name), 1, d, vw[name][1], d, L.ZO_SHADOW_F32))
            else:  # head
                wo_, wld = walloc(d, v)
                vw["w_out"] = (wbuf, wo_, d, v, wld)
                for name, n in (("lnf_g", d), ("lnf_b", d), ("b_out", v)):
                    vw[name] = ("v", valloc(n), 1, n, n)
                for name in bl.names:
                    k, n = bl.key(name), bl.size(name)
                    if name == "w_out":
                        if wld == v:
                            segs.append((k, 1, d * v, wo_, d * v, wkind))
                        else:
                            segs.append((k, d, v, wo_, wld, wkind))
                    else:
                        segs.append((k, 1, n, vw[name][1], n, L.ZO_SHADOW_F32))
            self.views[bl.block_id] = vw
            self.segments[bl.block_id] = segs
        self.w_elems = _a64(self.w_elems) + 64
        self.v_elems = self.v_elems + 4


def block_extent(plan: ShadowPlan, bid: int):
    """(w_lo, w_hi, v_lo, v_hi): the contiguous shadow ranges of one block."""
    ws = [(o, o + r * ld) for (b, o, r, c, ld) in plan.views[bid].values() if b == "w"] or [(0, 0)]
    vs = [(o, o + r * ld) for (b, o, r, c, ld) in plan.views[bid].values() if b == "v"] or [(0, 0)]
    return (min(a for a, _ in ws), max(b for _, b in ws), min(a for a, _ in vs), max(b for _, b in vs))


class SegTable:
    """Device copy of a segment list + its tile prefix."""

    def __init__(self, segs, device, block_ids=None):
        tile = int(L.lib().zo_perturb_tile_elems())
        arr = (L.ZoSegment * max(1, len(segs)))()
        prefix = np.zeros(len(segs) + 1, dtype=np.int64)
        block_ids = block_ids or [0] * len(segs)
        for i, ((src, rows, cols, dst, ld, kind), bid) in enumerate(zip(segs, block_ids)):
            arr[i] = L.ZoSegment(src, rows, cols, dst, ld, kind, bid)
            n = rows * ((cols + tile - 1) // tile)
            prefix[i + 1] = prefix[i] + n
        raw = np.frombuffer(bytes(arr), dtype=np.uint8).copy()
        self.segs = torch.from_numpy(raw).to(device)
        self.prefix = torch.from_numpy(prefix).to(device)
        self.n_segs = len(segs)
        self.n_tiles = int(prefix[-1])
        self.elems = int(sum(r * c for _, r, c, _, _, _ in segs))


class Workspace:
    """Activations of one directional forward at batch shape (B, T)."""

    def __init__(self, config: ModelConfig, batch: int, seq: int, device, f32: bool = False):
        d, v = config.d_model, config.vocab_size
        self.batch, self.seq, self.M = batch, seq, batch * seq
        M = self.M
        ld = _r8(d)
        adt = torch.float32 if f32 else torch.bfloat16        # f32 parity mode: fp32 activations
        self.x = torch.zeros(M, ld, dtype=torch.float32, device=device)
        self.h = torch.zeros(M, ld, dtype=adt, device=device)
        self.ctx = torch.zeros(M, ld, dtype=adt, device=device)
        self.qkv = torch.zeros(M, _r8(3 * d), dtype=adt, device=device)
        self.ff = torch.zeros(M, _r8(4 * d), dtype=adt, device=device)
        self.logits = torch.zeros(M, _r8(v), dtype=torch.float32, device=device) if f32 else None
        self.n_ce = int(L.lib().zo_gemm_ce_tiles(v))
        self.ce_part = torch.zeros(M, self.n_ce, 2, dtype=torch.float32, device=device)
        self.ce_tgt = torch.zeros(M, dtype=torch.float32, device=device)
        self.row_scratch = torch.zeros(M, dtype=torch.float64, device=device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=device)
        self.ids = torch.zeros(M, dtype=torch.int32, device=device)
        self.tgt = torch.zeros(M, dtype=torch.int32, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)

    @staticmethod
    def gemm(lib, *args):
        """(fn, args) of one GEMM launch; args are zo_gemm_bf16's, stream last."""
        return (lib.zo_gemm_bf16, args)


def _ptr(t):
    return 0 if t is None else t.data_ptr()


class DeviceStore:
    """The model's parameters on one GPU plus everything the ZO step needs.

    ``theta`` is the fp32 master (the reference's ParamStore buffers,
    src/zosim/model.py:160-200, concatenated in block order).
    """

    def __init__(self, config: ModelConfig, init_seed: int = 7, device=None, init: str = "host",
                 directions=(PLUS, MINUS), precision: str = "bf16"):
        """precision "bf16": the production path (bf16 GEMM operands, fp32
        accumulate, tcgen05 kernels); "f32": the parity mode of SURVEY 8c (i),
        fp32 operands and activations through the CUDA-core fp32 kernels."""
        config.validate()
        if precision not in ("bf16", "f32"):
            raise ConfigurationError(f"precision must be 'bf16' or 'f32', got {precision!r}")
        if precision == "f32" and config.arch != "zosim":
            raise ConfigurationError("the f32 parity mode covers the zosim architecture")
        self.precision = precision
        self.config = config
        self.init_seed = init_seed
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        L.lib()
        self.layouts = model_layout(config)
        self.total_params = sum(b.elem_count for b in self.layouts)
        self.theta = torch.empty(self.total_params, dtype=torch.float32, device=self.device)
        if init == "host":
            for bl in self.layouts:
                buf = init_block_host(config, bl, init_seed)
                self.theta[bl.key0:bl.key0 + bl.elem_count].copy_(torch.from_numpy(buf))
        elif init == "philox":
            self._init_philox(init_seed)
        elif init != "none":
            raise ConfigurationError(f"unknown init {init!r}")
        self.plan = ShadowPlan(config, self.layouts, f32_weights=precision == "f32")
        self.directions = tuple(directions)
        self.wsh = [None, None]
        self.vsh = [None, None]
        for s in self.directions:
            self.wsh[s] = torch.zeros(max(self.plan.w_elems, 64), dtype=torch.bfloat16, device=self.device)
            self.vsh[s] = torch.zeros(self.plan.v_elems, dtype=torch.float32, device=self.device)
        self.block_tables = {bid: SegTable(segs, self.device, [bid] * len(segs))
                             for bid, segs in self.plan.segments.items()}
        self.model_table = self.range_table(0, len(self.layouts))
        self.scal = torch.zeros(4, dtype=torch.int64, device=self.device)   # ZoStepScalars
        self.record = torch.zeros(3, dtype=torch.float64, device=self.device)
        self._ws = {}
        # launch resources of the step plans, created on first use (outside graph captures)
        self._side = self._prio = self._events = self._head_table = None

    # -- initialisation at scale -----------------------------------------------
    def _init_philox(self, init_seed: int):
        """Random init on the GPU for models too large for a host numpy draw
        (configs #3-#5 are 'random-init'): weights 0.02 * z(init_seed, key),
        LN gains 1, biases 0 -- same distribution as model.py:203-229."""
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
                        z = torch.empty(m, dtype=torch.float32, device=self.device)
                        L.call("zo_philox_normals", seed, k + o, m, z.data_ptr(), L.stream_ptr())
                        dst[o:o + m].copy_(z.mul_(0.02))

    # -- ParamStore-compatible helpers (model.py:169-200) ----------------------
    @property
    def blocks(self):
        from .zo import store_blocks

        return store_blocks(self)

    @property
    def n_blocks(self) -> int:
        return len(self.layouts)

    @property
    def total_bytes(self) -> int:
        return self.total_params * 4

    def checksum(self) -> str:
        """SHA-256 over the fp32 block buffers in order -- equal to the
        reference's ParamStore.checksum when the values are bit-identical."""
        import hashlib

        h = hashlib.sha256()
        th = self.theta.cpu().numpy()
        for bl in self.layouts:
            h.update(th[bl.key0:bl.key0 + bl.elem_count].tobytes())
        return h.hexdigest()

    def equal(self, other) -> bool:
        return bool(torch.equal(self.theta, other.theta))

    def block(self, block_id: int):
        """ParamStore.block (model.py:181-182)."""
        return self.blocks[block_id]

    def transformer_blocks(self):
        """ParamStore.transformer_blocks (model.py:184-185)."""
        return [b for b in self.blocks if b.kind == TRANSFORMER]

    def copy(self) -> "DeviceStore":
        """ParamStore.copy (model.py:187-188): a new store with this master;
        refused mid-perturbation (model.py:152-157) and with a deferred update
        outstanding (the copy would silently lack it)."""
        from .errors import ProtocolError

        for b in getattr(self, "_blocks", []):
            if b.pert_scale != 0.0:
                raise ProtocolError(f"block {b.block_id} copied mid-perturbation")
        if getattr(self, "unflushed", False):
            raise ProtocolError("copy of a master with a deferred update: call flush() first")
        out = DeviceStore(self.config, init_seed=self.init_seed, device=self.device, init="none",
                          directions=self.directions, precision=self.precision)
        out.theta.copy_(self.theta)
        return out

    # -- views -----------------------------------------------------------------
    def block_buf(self, bid: int) -> torch.Tensor:
        bl = self.layouts[bid]
        return self.theta[bl.key0:bl.key0 + bl.elem_count]

    def theta_ptr(self, key: int) -> int:
        return _ptr(self.theta) + 4 * key

    def wview(self, s: int, bid: int, name: str):
        buf, off, rows, cols, ld = self.plan.views[bid][name]
        src = self.wsh[s] if buf == "w" else self.vsh[s]       # "v": f32 parity-mode weights
        return src[off:off + rows * ld].view(rows, ld), rows, cols

    def vview(self, s: int, bid: int, name: str) -> torch.Tensor:
        buf, off, rows, cols, ld = self.plan.views[bid][name]
        assert buf == "v"
        return self.vsh[s][off:off + cols]

    def workspace(self, s: int, batch: int, seq: int) -> Workspace:
        """Per-direction activations; both directions of a batch shape share
        the device token-id / target buffers (one H2D per step, not two)."""
        key = (s, batch, seq)
        if key not in self._ws:
            ws = Workspace(self.config, batch, seq, self.device, f32=self.precision == "f32")
            other = self._ws.get((1 - s, batch, seq))
            if other is not None:
                ws.ids, ws.tgt = other.ids, other.tgt
            self._ws[key] = ws
        return self._ws[key]

    def stacked_workspace(self, batch: int, seq: int) -> Workspace:
        """Activations of BOTH directions stacked as [+eps rows; -eps rows]
        (2 * batch * seq rows) for the one-launch-per-layer plan
        (forward_calls_stacked); token ids / targets are the per-direction
        workspaces' shared buffers."""
        key = ("stacked", batch, seq)
        if key not in self._ws:
            ws = Workspace(self.config, 2 * batch, seq, self.device)
            base = self.workspace(PLUS, batch, seq)
            ws.ids, ws.tgt = base.ids, base.tgt
            ws.half = batch * seq
            ws.loss2 = torch.zeros(2, dtype=torch.float64, device=self.device)
            self._ws[key] = ws
        return self._ws[key]

    # -- launch resources of the step plans -------------------------------------
    def side_stream(self) -> torch.cuda.Stream:
        """The second stream of the two-stream plan."""
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        return self._side

    def priority_streams(self):
        """(high, low) priority streams of the fill plan (lower number = higher)."""
        if self._prio is None:
            self._prio = (torch.cuda.Stream(device=self.device, priority=-5),
                          torch.cuda.Stream(device=self.device, priority=0))
        return self._prio

    def plan_streams(self) -> list:
        """Every stream a step plan of this store has launched on so far."""
        return [x for x in (self._side, *(self._prio or ())) if x is not None]

    def block_events(self, n: int) -> list:
        """n reusable events (per-block ordering inside a step plan)."""
        if self._events is None or len(self._events) < n:
            self._events = [torch.cuda.Event() for _ in range(n)]
        return self._events

    def head_table(self) -> "SegTable":
        """Segment table of the embedding + first decoder block (the fill plan's
        full-speed part of the perturb pass)."""
        if self._head_table is None:
            self._head_table = self.range_table(0, 2)
        return self._head_table

    def stackable(self, batch: int, seq: int) -> bool:
        """The stacked GEMMs split rows on a CTA-pair tile boundary (bf16 path)."""
        return self.precision == "bf16" and (batch * seq) % 256 == 0

    # -- scalar state ----------------------------------------------------------
    def set_seed(self, seed: int, stream=None):
        self.scal[0:1].fill_(int(seed))

    def set_pending(self, g_lr: float, seed_prev: int, pending: bool):
        host = np.zeros(4, dtype=np.int64)
        host[0] = int(self.scal[0].item())
        host[1] = np.int64(np.uint64(seed_prev & ((1 << 64) - 1)).view(np.int64))
        host[2] = np.float64(g_lr).view(np.int64)
        host[3] = 1 if pending else 0
        self.scal.copy_(torch.from_numpy(host))

    def scalars(self) -> dict:
        h = self.scal.cpu().numpy()
        return {"seed_cur": int(h[0]), "seed_prev": int(h[1]), "lr_g_prev": float(h[2:3].view(np.float64)[0]),
                "pending": int(h[3])}

    def range_table(self, lo: int, hi: int) -> SegTable:
        """Segment table of blocks [lo, hi) in block order, segments tagged
        with their block id."""
        bids = [b for b in sorted(self.plan.segments) if lo <= b < hi]
        return SegTable([x for b in bids for x in self.plan.segments[b]], self.device,
                        [b for b in bids for _ in self.plan.segments[b]])

    def perturb_bytes(self, dirs=(PLUS, MINUS)) -> int:
        """Algorithmic HBM bytes of one fused update + perturb pass over the
        whole model: read + write of the fp32 master (8 B/param) plus each
        written shadow (bf16 weights 2 B, fp32 vectors 4 B, per direction in
        ``dirs``); tensors without a shadow (the embedding's gathered rows)
        move 8 B/param."""
        per = {L.ZO_SHADOW_BF16: 2, L.ZO_SHADOW_F32: 4, L.ZO_SHADOW_NONE: 0}
        return sum(rows * cols * (8 + per[kind] * len(dirs))
                   for segs in self.plan.segments.values() for (_, rows, cols, _, _, kind) in segs)

    # -- launch plans ----------------------------------------------------------
    def perturb_call(self, table: SegTable, flags: int, scale_a: float, scale_b: float, sa=PLUS, sb=MINUS,
                     zmode=L.ZO_Z_PHILOX, z_cur=None, z_prev=None, stream=None):
        fn = L.lib().zo_perturb_update
        args = (_ptr(self.theta), 0, _ptr(table.segs), _ptr(table.prefix), table.n_segs, table.n_tiles,
                _ptr(self.wsh[sa]) if sa is not None else 0, _ptr(self.vsh[sa]) if sa is not None else 0,
                _ptr(self.wsh[sb]) if sb is not None else 0, _ptr(self.vsh[sb]) if sb is not None else 0,
                float(scale_a), float(scale_b), flags, _ptr(self.scal), zmode, _ptr(z_cur), _ptr(z_prev), 0,
                L.stream_ptr(stream))
        return [(fn, args)]

    def forward_calls(self, s: int, ws: Workspace, scale: float, zmode=L.ZO_Z_PHILOX, z_cur=None, stream=None,
                      blocks=None, head_mode="ce", logits=None, loss_out=None, slots=None, scal=None):
        """Launch plan of one directional forward through blocks [0..N+1]
        (embedding -> N decoder blocks -> LN_f + LM head + CE).  ``slots``
        maps block ids to objects with the same wview / vview / theta_ptr
        interface when those blocks live outside this store (offload)."""
        if getattr(self, "precision", "bf16") == "f32":
            return self.forward_calls_f32(s, ws, scale, zmode, z_cur, stream, blocks, head_mode, logits, loss_out,
                                          scal, slots)
        cfg, lib = self.config, L.lib()
        d, H, hd, V = cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.vocab_size
        opt = cfg.arch == "opt"
        pos_off = 2 * d if opt else 0                      # OPT position t reads row t + 2
        ffn_epi = L.ZO_EPI_BIAS_RELU_BF16 if opt else L.ZO_EPI_BIAS_GELU_BF16
        M, B, T = ws.M, ws.batch, ws.seq
        st = L.stream_ptr(stream)
        calls = []
        blocks = range(len(self.layouts)) if blocks is None else blocks
        scal_p = _ptr(scal) if scal is not None else _ptr(self.scal)
        for bid in blocks:
            bl = self.layouts[bid]
            src = (slots or {}).get(bid, self)
            if bl.kind == EMBEDDING:
                calls.append((lib.zo_embed_fwd, (
                    src.theta_ptr(bl.key("tok_emb")), bl.key("tok_emb"),
                    src.theta_ptr(bl.key("pos_emb") + pos_off), bl.key("pos_emb") + pos_off,
                    _ptr(ws.ids), B, T, d, V, float(scale), scal_p, zmode, _ptr(z_cur), 0,
                    _ptr(ws.x), ws.x.stride(0), _ptr(ws.err), st)))
            elif bl.kind == TRANSFORMER:
                v = lambda n: _ptr(src.vview(s, bid, n))  # noqa: E731
                wq, _, _ = src.wview(s, bid, "qkv")
                wo, _, _ = src.wview(s, bid, "wo")
                w1, _, _ = src.wview(s, bid, "w1")
                w2, _, _ = src.wview(s, bid, "w2")
                ldx, ldh = ws.x.stride(0), ws.h.stride(0)
                calls += [
                    (lib.zo_layernorm_fwd, (_ptr(ws.x), ldx, v("ln1_g"), v("ln1_b"), M, d, _ptr(ws.h), ldh, st)),
                    ws.gemm(lib, *(_ptr(ws.h), ldh, _ptr(wq), wq.stride(0), M, 3 * d, d, L.ZO_EPI_BIAS_BF16,
                                        v("bqkv"), _ptr(ws.qkv), ws.qkv.stride(0), 0, 0, 0, 0, st)),
                    (lib.zo_attn_causal_fwd, (_ptr(ws.qkv), ws.qkv.stride(0), B, T, H, hd, _ptr(ws.ctx),
                                              ws.ctx.stride(0), st)),
                    ws.gemm(lib, *(_ptr(ws.ctx), ws.ctx.stride(0), _ptr(wo), wo.stride(0), M, d, d,
                                        L.ZO_EPI_BIAS_RESID_F32, v("bo"), _ptr(ws.x), ldx, 0, 0, 0, 0, st)),
                    (lib.zo_layernorm_fwd, (_ptr(ws.x), ldx, v("ln2_g"), v("ln2_b"), M, d, _ptr(ws.h), ldh, st)),
                    ws.gemm(lib, *(_ptr(ws.h), ldh, _ptr(w1), w1.stride(0), M, 4 * d, d,
                                        ffn_epi, v("b1"), _ptr(ws.ff), ws.ff.stride(0), 0, 0, 0, 0, st)),
                    ws.gemm(lib, *(_ptr(ws.ff), ws.ff.stride(0), _ptr(w2), w2.stride(0), M, d, 4 * d,
                                        L.ZO_EPI_BIAS_RESID_F32, v("b2"), _ptr(ws.x), ldx, 0, 0, 0, 0, st)),
                ]
            else:
                if opt:     # tied head: B = the token embedding's bf16 shadow [V, d], K-major, no bias
                    emb = (slots or {}).get(0, self)
                    wout, _, _ = emb.wview(s, 0, "tok_emb")
                    bout, bflag = 0, L.ZO_GEMM_B_KMAJOR
                else:
                    wout, _, _ = src.wview(s, bid, "w_out")
                    bout, bflag = _ptr(src.vview(s, bid, "b_out")), 0
                calls.append((lib.zo_layernorm_fwd, (_ptr(ws.x), ws.x.stride(0), _ptr(src.vview(s, bid, "lnf_g")),
                                                     _ptr(src.vview(s, bid, "lnf_b")), M, d, _ptr(ws.h),
                                                     ws.h.stride(0), st)))
                if head_mode == "ce":
                    calls.append(ws.gemm(lib, *(_ptr(ws.h), ws.h.stride(0), _ptr(wout), wout.stride(0), M, V, d,
                                                     L.ZO_EPI_CE | bflag, bout, 0, 0, _ptr(ws.tgt), _ptr(ws.ce_part),
                                                     _ptr(ws.ce_tgt), _ptr(ws.err), st)))
                    calls.append((lib.zo_ce_finalize, (_ptr(ws.ce_part), _ptr(ws.ce_tgt), M, ws.n_ce,
                                                       loss_out if loss_out is not None else _ptr(ws.loss),
                                                       _ptr(ws.row_scratch), _ptr(ws.err), st)))
                else:   # materialise logits (API forward(); not on the step)
                    calls.append(ws.gemm(lib, *(_ptr(ws.h), ws.h.stride(0), _ptr(wout), wout.stride(0), M, V, d,
                                                     L.ZO_EPI_F32 | bflag, 0, _ptr(logits), logits.stride(0), 0, 0,
                                                     0, 0, st)))
        return calls

    def forward_calls_f32(self, s, ws, scale, zmode=L.ZO_Z_PHILOX, z_cur=None, stream=None, blocks=None,
                          head_mode="ce", logits=None, loss_out=None, scal=None, slots=None):
        """forward_calls of the f32 parity mode: same block structure, fp32
        operands / activations through zo_gemm_f32, zo_attn_causal_fwd_f32,
        zo_layernorm_fwd_f32; the head materialises fp32 logits and
        zo_ce_rows_f32 + zo_ce_finalize form the f64 loss.  ``slots`` as in
        forward_calls (offloaded blocks)."""
        cfg, lib = self.config, L.lib()
        d, H, hd, V = cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.vocab_size
        M, B, T = ws.M, ws.batch, ws.seq
        st = L.stream_ptr(stream)
        calls = []
        blocks = range(len(self.layouts)) if blocks is None else blocks
        scal_p = _ptr(scal) if scal is not None else _ptr(self.scal)
        ldx, ldh = ws.x.stride(0), ws.h.stride(0)
        for bid in blocks:
            bl = self.layouts[bid]
            src = (slots or {}).get(bid, self)
            if bl.kind == EMBEDDING:
                calls.append((lib.zo_embed_fwd, (
                    src.theta_ptr(bl.key("tok_emb")), bl.key("tok_emb"), src.theta_ptr(bl.key("pos_emb")),
                    bl.key("pos_emb"), _ptr(ws.ids), B, T, d, V, float(scale), scal_p, zmode, _ptr(z_cur), 0,
                    _ptr(ws.x), ldx, _ptr(ws.err), st)))
            elif bl.kind == TRANSFORMER:
                v = lambda n: _ptr(src.vview(s, bid, n))  # noqa: E731
                w = {n: src.wview(s, bid, n)[0] for n in ("qkv", "wo", "w1", "w2")}
                g = lib.zo_gemm_f32
                calls += [
                    (lib.zo_layernorm_fwd_f32, (_ptr(ws.x), ldx, v("ln1_g"), v("ln1_b"), M, d, _ptr(ws.h), ldh, st)),
                    (g, (_ptr(ws.h), ldh, _ptr(w["qkv"]), w["qkv"].stride(0), M, 3 * d, d, L.ZO_EPI_BIAS_BF16,
                         v("bqkv"), _ptr(ws.qkv), ws.qkv.stride(0), st)),
                    (lib.zo_attn_causal_fwd_f32, (_ptr(ws.qkv), ws.qkv.stride(0), B, T, H, hd, _ptr(ws.ctx),
                                                  ws.ctx.stride(0), st)),
                    (g, (_ptr(ws.ctx), ws.ctx.stride(0), _ptr(w["wo"]), w["wo"].stride(0), M, d, d,
                         L.ZO_EPI_BIAS_RESID_F32, v("bo"), _ptr(ws.x), ldx, st)),
                    (lib.zo_layernorm_fwd_f32, (_ptr(ws.x), ldx, v("ln2_g"), v("ln2_b"), M, d, _ptr(ws.h), ldh, st)),
                    (g, (_ptr(ws.h), ldh, _ptr(w["w1"]), w["w1"].stride(0), M, 4 * d, d, L.ZO_EPI_BIAS_GELU_BF16,
                         v("b1"), _ptr(ws.ff), ws.ff.stride(0), st)),
                    (g, (_ptr(ws.ff), ws.ff.stride(0), _ptr(w["w2"]), w["w2"].stride(0), M, d, 4 * d,
                         L.ZO_EPI_BIAS_RESID_F32, v("b2"), _ptr(ws.x), ldx, st)),
                ]
            else:
                wout = src.wview(s, bid, "w_out")[0]
                calls.append((lib.zo_layernorm_fwd_f32, (_ptr(ws.x), ldx, _ptr(src.vview(s, bid, "lnf_g")),
                                                         _ptr(src.vview(s, bid, "lnf_b")), M, d, _ptr(ws.h), ldh,
                                                         st)))
                if head_mode == "ce":
                    calls.append((lib.zo_gemm_f32, (_ptr(ws.h), ldh, _ptr(wout), wout.stride(0), M, V, d,
                                                    L.ZO_EPI_BIAS_BF16, _ptr(src.vview(s, bid, "b_out")),
                                                    _ptr(ws.logits), ws.logits.stride(0), st)))
                    calls.append((lib.zo_ce_rows_f32, (_ptr(ws.logits), ws.logits.stride(0), M, V, _ptr(ws.tgt),
                                                       _ptr(ws.ce_part), _ptr(ws.ce_tgt), ws.n_ce, _ptr(ws.err), st)))
                    calls.append((lib.zo_ce_finalize, (_ptr(ws.ce_part), _ptr(ws.ce_tgt), M, ws.n_ce,
                                                       loss_out if loss_out is not None else _ptr(ws.loss),
                                                       _ptr(ws.row_scratch), _ptr(ws.err), st)))
                else:
                    calls.append((lib.zo_gemm_f32, (_ptr(ws.h), ldh, _ptr(wout), wout.stride(0), M, V, d,
                                                    L.ZO_EPI_F32, 0, _ptr(logits), logits.stride(0), st)))
        return calls

    def forward_calls_stacked(self, ws: Workspace, eps: float, zmode=L.ZO_Z_PHILOX, z_cur=None, stream=None,
                              blocks=None):
        """Both directional forwards as one launch per layer over the stacked
        activations [x+; x-] (rows [0, h) use the +eps shadows, [h, 2h) the
        -eps shadows): zo_layernorm_fwd_split / zo_gemm_bf16_split, attention
        over 2B sequences, two embedding gathers and two CE finalizes.  The
        per-row / per-tile arithmetic equals forward_calls on each direction,
        so losses are bit-identical to the two-stream plan."""
        cfg, lib = self.config, L.lib()
        d, H, hd, V = cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.vocab_size
        M2, h, B2, T = ws.M, ws.half, ws.batch, ws.seq
        opt = cfg.arch == "opt"
        pos_off = 2 * d if opt else 0
        ffn_epi = L.ZO_EPI_BIAS_RELU_BF16 if opt else L.ZO_EPI_BIAS_GELU_BF16
        st = L.stream_ptr(stream)
        ldx, ldh = ws.x.stride(0), ws.h.stride(0)
        calls = []
        for bid in (range(len(self.layouts)) if blocks is None else blocks):
            bl = self.layouts[bid]
            vp = lambda n: _ptr(self.vview(PLUS, bid, n))    # noqa: E731
            vm = lambda n: _ptr(self.vview(MINUS, bid, n))   # noqa: E731

            def wv(n, _bid=bid):
                return self.wview(PLUS, _bid, n)[0], self.wview(MINUS, _bid, n)[0]

            if bl.kind == EMBEDDING:
                for k, sc in ((0, +eps), (1, -eps)):
                    calls.append((lib.zo_embed_fwd, (
                        self.theta_ptr(bl.key("tok_emb")), bl.key("tok_emb"),
                        self.theta_ptr(bl.key("pos_emb") + pos_off), bl.key("pos_emb") + pos_off,
                        _ptr(ws.ids), B2 // 2, T, d, V, float(sc), _ptr(self.scal), zmode, _ptr(z_cur), 0,
                        _ptr(ws.x) + 4 * k * h * ldx, ldx, _ptr(ws.err), st)))
            elif bl.kind == TRANSFORMER:
                (qa, qb), (oa, ob), (f1a, f1b), (f2a, f2b) = wv("qkv"), wv("wo"), wv("w1"), wv("w2")
                g = lib.zo_gemm_bf16_split
                calls += [
                    (lib.zo_layernorm_fwd_split, (_ptr(ws.x), ldx, vp("ln1_g"), vp("ln1_b"), vm("ln1_g"), vm("ln1_b"),
                                                  M2, h, d, _ptr(ws.h), ldh, st)),
                    (g, (_ptr(ws.h), ldh, _ptr(qa), _ptr(qb), qa.stride(0), M2, 3 * d, d, h, L.ZO_EPI_BIAS_BF16,
                         vp("bqkv"), vm("bqkv"), _ptr(ws.qkv), ws.qkv.stride(0), 0, 0, 0, 0, st)),
                    (lib.zo_attn_causal_fwd, (_ptr(ws.qkv), ws.qkv.stride(0), B2, T, H, hd, _ptr(ws.ctx),
                                              ws.ctx.stride(0), st)),
                    (g, (_ptr(ws.ctx), ws.ctx.stride(0), _ptr(oa), _ptr(ob), oa.stride(0), M2, d, d, h,
                         L.ZO_EPI_BIAS_RESID_F32, vp("bo"), vm("bo"), _ptr(ws.x), ldx, 0, 0, 0, 0, st)),
                    (lib.zo_layernorm_fwd_split, (_ptr(ws.x), ldx, vp("ln2_g"), vp("ln2_b"), vm("ln2_g"), vm("ln2_b"),
                                                  M2, h, d, _ptr(ws.h), ldh, st)),
                    (g, (_ptr(ws.h), ldh, _ptr(f1a), _ptr(f1b), f1a.stride(0), M2, 4 * d, d, h, ffn_epi,
                         vp("b1"), vm("b1"), _ptr(ws.ff), ws.ff.stride(0), 0, 0, 0, 0, st)),
                    (g, (_ptr(ws.ff), ws.ff.stride(0), _ptr(f2a), _ptr(f2b), f2a.stride(0), M2, d, 4 * d, h,
                         L.ZO_EPI_BIAS_RESID_F32, vp("b2"), vm("b2"), _ptr(ws.x), ldx, 0, 0, 0, 0, st)),
                ]
            else:
                if opt:
                    wa, wb = self.wview(PLUS, 0, "tok_emb")[0], self.wview(MINUS, 0, "tok_emb")[0]
                    ba = bb = 0
                    flag = L.ZO_GEMM_B_KMAJOR
                else:
                    wa, wb = wv("w_out")
                    ba, bb, flag = vp("b_out"), vm("b_out"), 0
                calls.append((lib.zo_layernorm_fwd_split, (_ptr(ws.x), ldx, vp("lnf_g"), vp("lnf_b"), vm("lnf_g"),
                                                           vm("lnf_b"), M2, h, d, _ptr(ws.h), ldh, st)))
                calls.append((lib.zo_gemm_bf16_split, (_ptr(ws.h), ldh, _ptr(wa), _ptr(wb), wa.stride(0), M2, V, d, h,
                                                       L.ZO_EPI_CE | flag, ba, bb, 0, 0, _ptr(ws.tgt),
                                                       _ptr(ws.ce_part), _ptr(ws.ce_tgt), _ptr(ws.err), st)))
                for k in (0, 1):
                    calls.append((lib.zo_ce_finalize, (_ptr(ws.ce_part) + 4 * k * h * ws.n_ce * 2,
                                                       _ptr(ws.ce_tgt) + 4 * k * h, h, ws.n_ce,
                                                       _ptr(ws.loss2) + 8 * k, _ptr(ws.row_scratch) + 8 * k * h,
                                                       _ptr(ws.err), st)))
        return calls

    def grad_call_stacked(self, ws: Workspace, eps: float, lr: float, stream=None):
        return [(L.lib().zo_grad_finalize, (_ptr(ws.loss2), _ptr(ws.loss2) + 8, float(eps), float(lr),
                                            _ptr(self.scal), _ptr(self.record), L.stream_ptr(stream)))]

    def grad_call(self, ws_pos: Workspace, ws_neg: Workspace, eps: float, lr: float, stream=None):
        return [(L.lib().zo_grad_finalize, (_ptr(ws_pos.loss), _ptr(ws_neg.loss), float(eps), float(lr),
                                            _ptr(self.scal), _ptr(self.record), L.stream_ptr(stream)))]

    @staticmethod
    def run(calls):
        for fn, args in calls:
            rc = fn(*args)
            if rc:
                L.check(rc)

    # -- host <-> device batch staging -----------------------------------------
    def load_batch(self, ws: Workspace, token_ids, targets):
        ids = np.asarray(token_ids)
        tg = np.asarray(targets)
        if ids.shape != (ws.batch, ws.seq) or tg.shape != ids.shape:
            raise DimensionError(f"batch shape {ids.shape} does not match workspace ({ws.batch}, {ws.seq})")
        if ids.size and (ids.min() < 0 or ids.max() >= self.config.vocab_size):
            raise DimensionError("token id out of embedding range")
        M = ids.size
        stage = getattr(self, "_stage", None)
        if stage is None or stage.shape[1] < M:
            stage = self._stage = torch.empty(2, max(M, 1), dtype=torch.int32, pin_memory=True)
        st = stage.numpy()
        st[0, :M] = ids.reshape(-1)
        st[1, :M] = tg.reshape(-1)
        torch.cuda.current_stream().synchronize() if getattr(self, "_stage_busy", False) else None
        ws.ids.copy_(stage[0, :M], non_blocking=True)       # pinned -> device, async
        ws.tgt.copy_(stage[1, :M], non_blocking=True)
        self._stage_busy = True

    def check_errors(self, *wss, flags=None):
        errs = flags if flags is not None else [int(ws.err.item()) for ws in wss]
        for ws, e in zip(wss, errs):        # clear every flagged workspace before raising
            if e:
                ws.err.zero_()
        e = 0
        for x in errs:
            e |= int(x)
        if e & 4:
            raise DimensionError("token id out of embedding range")
        if e:
            raise NumericError("non-finite logits")

    def read_step(self, wss):
        """One D2H for the step record and the error flags (pinned, then a
        single stream sync)."""
        out = getattr(self, "_readback", None)
        if out is None:
            out = self._readback = torch.empty(3, dtype=torch.float64, pin_memory=True)
            self._errback = torch.empty(4, dtype=torch.int32, pin_memory=True)
        out.copy_(self.record, non_blocking=True)
        for i, ws in enumerate(wss[:4]):
            self._errback[i:i + 1].copy_(ws.err, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        self._stage_busy = False
        errs = [int(v) for v in self._errback.numpy()[:len(wss[:4])]]
        self.check_errors(*wss[:4], flags=errs)
        h = out.numpy()
        return float(h[0]), float(h[1]), float(h[2])


def init_model(config: ModelConfig, init_seed: int, device=None, init: str = "host") -> DeviceStore:
    """zosim.init_model (model.py:203-229) returning a GPU-resident store."""
    return DeviceStore(config, init_seed=init_seed, device=device, init=init)
