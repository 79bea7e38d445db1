"""Tensor-level wrappers over the C ABI (torch tensors in, async on a stream).

These are the building blocks the ZO engine (engine.py) composes; they do
shape checks and pass raw device pointers to libzo_b200.so.  Every call
launches native sm_100a kernels -- there is no fallback path.
"""

from __future__ import annotations

import torch

from . import _lib as L
from .errors import DimensionError


def _p(t):
    return 0 if t is None else t.data_ptr()


def _ld(t):
    return t.stride(0) if t.dim() == 2 else t.shape[-1]


def gemm(a: torch.Tensor, b: torch.Tensor, epilogue: int, out=None, bias=None, m=None, n=None, k=None,
         targets=None, ce_part=None, ce_tgt=None, err=None, stream=None):
    """out (+)= epilogue(a[M,K] @ b[K,N]) on tcgen05.  a, b bf16 2-D with unit
    inner stride (b as [N, K] when ``epilogue`` carries ZO_GEMM_B_KMAJOR);
    bias fp32 [N]."""
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise DimensionError("gemm operands must be bf16")
    M = m if m is not None else a.shape[0]
    K = k if k is not None else a.shape[1]
    bkm = bool(epilogue & L.ZO_GEMM_B_KMAJOR)       # b given as [N, K] (K contiguous)
    N = n if n is not None else b.shape[0 if bkm else 1]
    if b.shape[1 if bkm else 0] < K or a.stride(-1) != 1 or b.stride(-1) != 1:
        raise DimensionError("gemm: operand shapes/strides do not match")
    ldo = 0 if out is None else _ld(out)
    L.call("zo_gemm_bf16", _p(a), _ld(a), _p(b), _ld(b), M, N, K, epilogue, _p(bias), _p(out), ldo,
           _p(targets), _p(ce_part), _p(ce_tgt), _p(err), L.stream_ptr(stream))
    return out


def ce_tiles(n: int) -> int:
    return int(L.lib().zo_gemm_ce_tiles(n))


def layernorm(x: torch.Tensor, g: torch.Tensor, b: torch.Tensor, out: torch.Tensor, rows=None, d=None, stream=None):
    rows = rows if rows is not None else x.shape[0]
    d = d if d is not None else g.shape[0]
    L.call("zo_layernorm_fwd", _p(x), _ld(x), _p(g), _p(b), rows, d, _p(out), _ld(out), L.stream_ptr(stream))
    return out


def attention(qkv: torch.Tensor, batch: int, seq: int, heads: int, head_dim: int, out: torch.Tensor, stream=None):
    L.call("zo_attn_causal_fwd", _p(qkv), _ld(qkv), batch, seq, heads, head_dim, _p(out), _ld(out),
           L.stream_ptr(stream))
    return out


def ce_finalize(ce_part, ce_tgt, rows, n_tiles, loss_out, row_scratch, err, stream=None):
    L.call("zo_ce_finalize", _p(ce_part), _p(ce_tgt), rows, n_tiles, _p(loss_out), _p(row_scratch), _p(err),
           L.stream_ptr(stream))


def embed(tok, tok_key0, pos, pos_key0, ids, batch, seq, d, vocab, scale, scal, zmode, z, z_key0, x, err,
          stream=None):
    L.call("zo_embed_fwd", _p(tok), tok_key0, _p(pos), pos_key0, _p(ids), batch, seq, d, vocab, float(scale),
           _p(scal), zmode, _p(z), z_key0, _p(x), _ld(x), _p(err), L.stream_ptr(stream))


def perturb_update(theta, theta_key0, segs, prefix, n_segs, n_tiles, wsh_a, vsh_a, wsh_b, vsh_b, scale_a, scale_b,
                   flags, scal, zmode=L.ZO_Z_PHILOX, z_cur=None, z_prev=None, z_key0=0, stream=None):
    L.call("zo_perturb_update", _p(theta), theta_key0, _p(segs), _p(prefix), n_segs, n_tiles, _p(wsh_a), _p(vsh_a),
           _p(wsh_b), _p(vsh_b), float(scale_a), float(scale_b), flags, _p(scal), zmode, _p(z_cur), _p(z_prev),
           z_key0, L.stream_ptr(stream))


def grad_finalize(loss_pos, loss_neg, eps, lr, scal, record, stream=None):
    L.call("zo_grad_finalize", _p(loss_pos), _p(loss_neg), float(eps), float(lr), _p(scal), _p(record),
           L.stream_ptr(stream))


def grad_finalize_groups(losses, n_groups, layout, mine, eps, lr, scal, record, stream=None):
    """layout = (plus_stride, plus_off, minus_stride, minus_off) into `losses`."""
    sp, op, sm, om = layout
    L.call("zo_grad_finalize_groups", _p(losses), n_groups, sp, op, sm, om, mine, float(eps), float(lr), _p(scal),
           _p(record), L.stream_ptr(stream))


def philox_normals(seed: int, e0: int, n: int, device="cuda", stream=None) -> torch.Tensor:
    out = torch.empty(n, dtype=torch.float32, device=device)
    L.call("zo_philox_normals", seed & ((1 << 64) - 1), e0, n, _p(out), L.stream_ptr(stream))
    return out


def hash_u64(t: torch.Tensor, stream=None) -> torch.Tensor:
    out = torch.empty(1, dtype=torch.int64, device=t.device)
    scratch = torch.empty(256, dtype=torch.int64, device=t.device)
    L.call("zo_hash_u64", _p(t), t.numel() * t.element_size(), _p(out), _p(scratch), L.stream_ptr(stream))
    return out


def planes_join(hi: torch.Tensor, lo: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """out (fp32) = the float whose bits are hi << 16 | lo (int16 planes)."""
    n = out.numel()
    if hi.numel() != n or lo.numel() != n or out.dtype != torch.float32:
        raise ValueError("planes_join: hi / lo / out sizes or dtype mismatch")
    L.call("zo_planes_join", _p(hi), _p(lo), _p(out), n, L.stream_ptr(stream))
    return out


def planes_split(theta: torch.Tensor, hi: torch.Tensor, lo: torch.Tensor, stream=None) -> None:
    """hi / lo (int16) = the upper / lower 16 bits of each fp32 of theta."""
    n = theta.numel()
    if hi.numel() != n or lo.numel() != n or theta.dtype != torch.float32:
        raise ValueError("planes_split: theta / hi / lo sizes or dtype mismatch")
    L.call("zo_planes_split", _p(theta), _p(hi), _p(lo), n, L.stream_ptr(stream))
