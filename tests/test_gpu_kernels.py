"""Kernel-level parity of the sm_100a library against plain torch fp32
references of the same op (bf16 operands where the kernel consumes bf16)."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200 import ops  # noqa: E402

DEV = "cuda"


def _rand(*shape, scale=1.0, dtype=torch.bfloat16, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.randn(*shape, generator=g) * scale).to(DEV, dtype)


GEMM_SHAPES = [(128, 256, 64), (128, 128, 128), (256, 512, 512), (200, 304, 136), (64, 96, 32),
               (16, 16, 16), (1000, 1000, 1000), (2048, 2048, 2048), (512, 6144, 2048), (64, 50272, 768)]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_f32_matches_torch(M, N, K):
    a, b = _rand(M, K, seed=1), _rand(K, N, seed=2)
    out = torch.full((M, N), float("nan"), device=DEV)
    ops.gemm(a, b, L.ZO_EPI_F32, out=out)
    torch.cuda.synchronize()
    ref = a.float() @ b.float()
    torch.testing.assert_close(out, ref, rtol=2e-3, atol=2e-3 * math.sqrt(K / 64))


@pytest.mark.parametrize("M,N,K", [(256, 768, 256), (200, 304, 136), (2048, 8192, 2048)])
def test_gemm_bias_and_gelu_epilogues(M, N, K):
    a, b = _rand(M, K, seed=3, scale=0.5), _rand(K, N, seed=4, scale=0.1)
    bias = _rand(N, dtype=torch.float32, seed=5)
    out = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    ops.gemm(a, b, L.ZO_EPI_BIAS_BF16, out=out, bias=bias)
    ref = a.float() @ b.float() + bias
    torch.testing.assert_close(out.float(), ref, rtol=1e-2, atol=1e-2)
    ops.gemm(a, b, L.ZO_EPI_BIAS_GELU_BF16, out=out, bias=bias)
    refg = torch.nn.functional.gelu(ref, approximate="tanh")
    torch.testing.assert_close(out.float(), refg, rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("M,N,K", [(256, 768, 3072), (200, 304, 136), (2048, 2048, 8192)])
def test_gemm_residual_epilogue(M, N, K):
    a, b = _rand(M, K, seed=6, scale=0.5), _rand(K, N, seed=7, scale=0.05)
    bias = _rand(N, dtype=torch.float32, seed=8)
    x = _rand(M, N, dtype=torch.float32, seed=9)
    ref = x + (a.float() @ b.float() + bias)
    ops.gemm(a, b, L.ZO_EPI_BIAS_RESID_F32, out=x, bias=bias)
    torch.testing.assert_close(x, ref, rtol=1e-4, atol=2e-3)


@pytest.mark.parametrize("M,V,K", [(64, 50272, 768), (130, 1000, 64), (32, 16, 16)])
def test_gemm_ce_epilogue_and_finalize(M, V, K):
    a, b = _rand(M, K, seed=10, scale=0.5), _rand(K, V, seed=11, scale=0.1)
    bias = _rand(V, dtype=torch.float32, seed=12, scale=0.1)
    tg = torch.randint(0, V, (M,), generator=torch.Generator().manual_seed(3)).to(DEV, torch.int32)
    nt = ops.ce_tiles(V)
    part = torch.empty(M, nt, 2, device=DEV)
    tl = torch.empty(M, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    ops.gemm(a, b, L.ZO_EPI_CE, bias=bias, targets=tg, ce_part=part, ce_tgt=tl, err=err)
    loss = torch.empty(1, dtype=torch.float64, device=DEV)
    scratch = torch.empty(M, dtype=torch.float64, device=DEV)
    ops.ce_finalize(part, tl, M, nt, loss, scratch, err)
    logits = (a.float() @ b.float() + bias).double()
    ref = torch.nn.functional.cross_entropy(logits, tg.long())
    assert err.item() == 0
    assert abs(loss.item() - ref.item()) < 1e-4
    torch.testing.assert_close(tl.double(), logits.gather(1, tg.long()[:, None])[:, 0], rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("M,N,K", [(256, 768, 256), (200, 304, 136), (2048, 8192, 2048), (64, 512, 128)])
def test_gemm_relu_epilogue(M, N, K):
    """real-OPT FFN up-projection: relu(h @ W1 + b1) -> bf16."""
    a, b = _rand(M, K, seed=31, scale=0.5), _rand(K, N, seed=32, scale=0.1)
    bias = _rand(N, dtype=torch.float32, seed=33)
    out = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    ops.gemm(a, b, L.ZO_EPI_BIAS_RELU_BF16, out=out, bias=bias)
    ref = torch.relu(a.float() @ b.float() + bias)
    torch.testing.assert_close(out.float(), ref, rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (64, 96, 32), (256, 512, 512), (200, 304, 136),
                                   (1000, 1000, 1000), (2048, 4096, 2048)])
def test_gemm_b_kmajor_f32(M, N, K):
    """B given transposed ([N, K], K contiguous): single-CTA and CTA-pair
    kernels with the K-major UMMA B descriptor."""
    a, bt = _rand(M, K, seed=34), _rand(N, K, seed=35)
    out = torch.full((M, N), float("nan"), device=DEV)
    ops.gemm(a, bt, L.ZO_EPI_F32 | L.ZO_GEMM_B_KMAJOR, out=out)
    torch.cuda.synchronize()
    torch.testing.assert_close(out, a.float() @ bt.float().t(), rtol=2e-3, atol=2e-3 * math.sqrt(K / 64))


@pytest.mark.parametrize("M,V,K", [(64, 50272, 768), (512, 1000, 64), (32, 16, 16)])
def test_gemm_tied_head_ce(M, V, K):
    """Tied LM head: logits = h @ E^T with E the [V, d] embedding (K-major B)
    and no bias, through the CE epilogue (real OPT)."""
    a, emb = _rand(M, K, seed=36, scale=0.5), _rand(V, K, seed=37, scale=0.1)
    tg = torch.randint(0, V, (M,), generator=torch.Generator().manual_seed(5)).to(DEV, torch.int32)
    nt = ops.ce_tiles(V)
    part, tl = torch.empty(M, nt, 2, device=DEV), torch.empty(M, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    ops.gemm(a, emb, L.ZO_EPI_CE | L.ZO_GEMM_B_KMAJOR, targets=tg, ce_part=part, ce_tgt=tl, err=err)
    loss, scratch = torch.empty(1, dtype=torch.float64, device=DEV), torch.empty(M, dtype=torch.float64, device=DEV)
    ops.ce_finalize(part, tl, M, nt, loss, scratch, err)
    logits = (a.float() @ emb.float().t()).double()
    assert err.item() == 0
    assert abs(loss.item() - torch.nn.functional.cross_entropy(logits, tg.long()).item()) < 1e-4


@pytest.mark.parametrize("M,N,K", [(512, 768, 256), (4096, 6144, 2048), (1024, 1000, 200)])
def test_gemm_split_equals_two_gemms(M, N, K):
    """zo_gemm_bf16_split over stacked rows == zo_gemm_bf16 on each half with
    its own B / bias, bit for bit, for every epilogue."""
    h = M // 2
    a = _rand(M, K, seed=41, scale=0.5)
    b1, b2 = _rand(K, N, seed=42, scale=0.1), _rand(K, N, seed=43, scale=0.1)
    c1, c2 = _rand(N, dtype=torch.float32, seed=44), _rand(N, dtype=torch.float32, seed=45)
    lib = L.lib()
    for epi, dt in ((L.ZO_EPI_BIAS_BF16, torch.bfloat16), (L.ZO_EPI_BIAS_GELU_BF16, torch.bfloat16),
                    (L.ZO_EPI_BIAS_RELU_BF16, torch.bfloat16), (L.ZO_EPI_BIAS_RESID_F32, torch.float32)):
        x0 = _rand(M, N, dtype=torch.float32, seed=46)
        got = x0.clone() if dt == torch.float32 else torch.empty(M, N, device=DEV, dtype=dt)
        want = x0.clone() if dt == torch.float32 else torch.empty(M, N, device=DEV, dtype=dt)
        L.check(lib.zo_gemm_bf16_split(a.data_ptr(), K, b1.data_ptr(), b2.data_ptr(), N, M, N, K, h, epi,
                                       c1.data_ptr(), c2.data_ptr(), got.data_ptr(), N, 0, 0, 0, 0, L.stream_ptr()))
        ops.gemm(a[:h], b1, epi, out=want[:h], bias=c1)
        ops.gemm(a[h:], b2, epi, out=want[h:], bias=c2)
        torch.cuda.synchronize()
        assert torch.equal(got, want), epi
    # CE epilogue: stacked rows share one [M/2] target vector
    tg = torch.randint(0, N, (h,), generator=torch.Generator().manual_seed(6)).to(DEV, torch.int32)
    nt = ops.ce_tiles(N)
    part, tl = torch.empty(M, nt, 2, device=DEV), torch.empty(M, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    L.check(lib.zo_gemm_bf16_split(a.data_ptr(), K, b1.data_ptr(), b2.data_ptr(), N, M, N, K, h, L.ZO_EPI_CE,
                                   c1.data_ptr(), c2.data_ptr(), 0, 0, tg.data_ptr(), part.data_ptr(), tl.data_ptr(),
                                   err.data_ptr(), L.stream_ptr()))
    p1, t1 = torch.empty(h, nt, 2, device=DEV), torch.empty(h, device=DEV)
    p2, t2 = torch.empty(h, nt, 2, device=DEV), torch.empty(h, device=DEV)
    ops.gemm(a[:h], b1, L.ZO_EPI_CE, bias=c1, targets=tg, ce_part=p1, ce_tgt=t1, err=err)
    ops.gemm(a[h:], b2, L.ZO_EPI_CE, bias=c2, targets=tg, ce_part=p2, ce_tgt=t2, err=err)
    torch.cuda.synchronize()
    assert torch.equal(part, torch.cat([p1, p2])) and torch.equal(tl, torch.cat([t1, t2]))
    with pytest.raises(Exception):      # the split must sit on a 256-row pair-tile boundary
        L.check(lib.zo_gemm_bf16_split(a.data_ptr(), K, b1.data_ptr(), b2.data_ptr(), N, M, N, K, 100,
                                       L.ZO_EPI_BIAS_BF16, c1.data_ptr(), c2.data_ptr(), got.data_ptr(), N,
                                       0, 0, 0, 0, L.stream_ptr()))


@pytest.mark.parametrize("d", [2048, 5120])
def test_layernorm_split_equals_two_layernorms(d):
    rows = 512
    x = _rand(rows, d, dtype=torch.float32, seed=47)
    g1, b1, g2, b2 = (_rand(d, dtype=torch.float32, seed=s) for s in (48, 49, 50, 51))
    got = torch.empty(rows, d, device=DEV, dtype=torch.bfloat16)
    want = torch.empty_like(got)
    L.check(L.lib().zo_layernorm_fwd_split(x.data_ptr(), d, g1.data_ptr(), b1.data_ptr(), g2.data_ptr(),
                                           b2.data_ptr(), rows, 200, d, got.data_ptr(), d, L.stream_ptr()))
    ops.layernorm(x[:200], g1, b1, want[:200])
    ops.layernorm(x[200:], g2, b2, want[200:])
    torch.cuda.synchronize()
    assert torch.equal(got, want)


# persistent CTA-pair schedule with partial last waves: 64 / 192 / 1576 tiles of
# 256 x 256 over the 74 pairs, a K=8192 case and ragged M / N / K
WAVE_SHAPES = [(2048, 2048, 2048), (2048, 6144, 2048), (2048, 2048, 8192), (1024, 4000, 1000), (512, 50272, 256)]


@pytest.mark.parametrize("M,N,K", WAVE_SHAPES)
def test_gemm_multiwave_epilogues(M, N, K):
    """Every epilogue matches fp32 torch over several (partial) waves of the
    persistent pair kernel and is bit-reproducible run to run."""
    a, b = _rand(M, K, seed=21, scale=0.5), _rand(K, N, seed=22, scale=0.05)
    bias = _rand(N, dtype=torch.float32, seed=23)
    ref = a.float() @ b.float()
    tol = dict(rtol=2e-3, atol=2e-3 * math.sqrt(K / 64))
    out = torch.full((M, N), float("nan"), device=DEV)
    ops.gemm(a, b, L.ZO_EPI_F32, out=out)
    torch.testing.assert_close(out, ref, **tol)
    out2 = torch.full((M, N), float("nan"), device=DEV)
    ops.gemm(a, b, L.ZO_EPI_F32, out=out2)
    assert torch.equal(out, out2)                # fixed accumulation order
    x = _rand(M, N, dtype=torch.float32, seed=24)
    xr = x + (ref + bias)
    ops.gemm(a, b, L.ZO_EPI_BIAS_RESID_F32, out=x, bias=bias)
    torch.testing.assert_close(x, xr, **tol)
    o16 = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    ops.gemm(a, b, L.ZO_EPI_BIAS_GELU_BF16, out=o16, bias=bias)
    torch.testing.assert_close(o16.float(), torch.nn.functional.gelu(ref + bias, approximate="tanh"),
                               rtol=1e-2, atol=1e-2)
    tg = torch.randint(0, N, (M,), generator=torch.Generator().manual_seed(4)).to(DEV, torch.int32)
    nt = ops.ce_tiles(N)
    part, tl = torch.empty(M, nt, 2, device=DEV), torch.empty(M, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    ops.gemm(a, b, L.ZO_EPI_CE, bias=bias, targets=tg, ce_part=part, ce_tgt=tl, err=err)
    loss, scratch = torch.empty(1, dtype=torch.float64, device=DEV), torch.empty(M, dtype=torch.float64, device=DEV)
    ops.ce_finalize(part, tl, M, nt, loss, scratch, err)
    cref = torch.nn.functional.cross_entropy((ref + bias).double(), tg.long())
    assert err.item() == 0 and abs(loss.item() - cref.item()) < 1e-3


@pytest.mark.parametrize("rows,d", [(64, 768), (513, 2048), (7, 6), (3, 12288), (65, 5120), (9, 9216), (4, 7168)])
def test_layernorm(rows, d):
    x = _rand(rows, d, dtype=torch.float32, seed=13) * 3 + 1
    g = _rand(d, dtype=torch.float32, seed=14)
    b = _rand(d, dtype=torch.float32, seed=15)
    out = torch.empty(rows, d, dtype=torch.bfloat16, device=DEV)
    ops.layernorm(x, g, b, out)
    ref = torch.nn.functional.layer_norm(x, (d,), g, b, eps=1e-5)
    torch.testing.assert_close(out.float(), ref, rtol=1e-2, atol=2e-2)


def _attn_ref(qkv, B, T, H, hd):
    d = H * hd
    q, k, v = qkv[:, :d].float(), qkv[:, d:2 * d].float(), qkv[:, 2 * d:3 * d].float()
    q = q.view(B, T, H, hd).transpose(1, 2)
    k = k.view(B, T, H, hd).transpose(1, 2)
    v = v.view(B, T, H, hd).transpose(1, 2)
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
    return o.transpose(1, 2).reshape(B * T, d)


@pytest.mark.parametrize("B,T,H,hd", [(1, 64, 12, 64), (2, 512, 4, 64), (1, 100, 2, 64), (2, 256, 2, 128),
                                      (1, 300, 3, 128), (1, 1024, 2, 128), (4, 8, 2, 8), (2, 6, 2, 3),
                                      (1, 33, 3, 32), (1, 300, 3, 64), (8, 512, 32, 64), (3, 1024, 5, 64),
                                      (1, 2048, 1, 64), (2, 130, 1, 64)])
def test_attention(B, T, H, hd):
    qkv = _rand(B * T, 3 * H * hd, seed=16)
    out = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device=DEV)
    ops.attention(qkv, B, T, H, hd, out)
    ref = _attn_ref(qkv, B, T, H, hd)
    torch.testing.assert_close(out.float(), ref, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("hd", [64, 128])
def test_attention_growing_scores(hd):
    """Scores whose row max keeps rising by far more than 2^8 along the keys:
    the hd-64 kernel's lazily raised running max must rescale O and l."""
    B, T, H = 2, 1024, 3
    qkv = _rand(B * T, 3 * H * hd, seed=17)
    d = H * hd
    ramp = torch.linspace(0.5, 12.0, T, device=DEV).repeat(B).unsqueeze(1)
    qkv[:, d:2 * d] = (qkv[:, d:2 * d].float() * ramp).bfloat16()      # later keys: larger |scores|
    qkv[:, :d] = (qkv[:, :d].float() * 4.0).bfloat16()
    out = torch.empty(B * T, d, dtype=torch.bfloat16, device=DEV)
    ops.attention(qkv, B, T, H, hd, out)
    ref = _attn_ref(qkv, B, T, H, hd)
    assert bool(torch.isfinite(out.float()).all())
    torch.testing.assert_close(out.float(), ref, rtol=2e-2, atol=2e-2)


def test_philox_distribution_and_slice_invariance():
    z = ops.philox_normals(1234567, 0, 1 << 22)
    zc = z.double().cpu().numpy()
    assert abs(zc.mean()) < 3e-3 and abs(zc.var() - 1) < 3e-3
    assert abs(((zc ** 3).mean())) < 1e-2 and abs((zc ** 4).mean() - 3) < 2e-2
    # slice invariance: any window is the same function of the global key
    z2 = ops.philox_normals(1234567, 1001, 4099)
    assert torch.equal(z[1001:1001 + 4099], z2)
    z3 = ops.philox_normals(7654321, 0, 1 << 10)
    assert not torch.equal(z[:1024], z3)
    # KS statistic against N(0,1)
    from scipy import stats
    ks = stats.kstest(zc[:200000], "norm").statistic
    assert ks < 5e-3


def test_philox_normals_finite_over_a_large_window():
    """u1 rounds to exactly 1.0 with probability 2^-24 per Box-Muller pair: a
    2^27-element window contains several such events; all outputs must be
    finite (a NaN here would poison theta through the folded update)."""
    for seed in (1, 0x123456789ABCDEF):
        z = ops.philox_normals(seed, 0, 1 << 27)
        assert bool(torch.isfinite(z).all())
        assert float(z.abs().max()) < 6.5
        del z


@pytest.mark.parametrize("n,off", [(1, 0), (7, 1), (4096, 0), (100003, 3), (1 << 22, 8)])
def test_planes_split_join_roundtrip(n, off):
    """hi / lo 16-bit planes of fp32 (transfer compression): split then join
    is the identity on the bits (incl. +-0, inf, NaN payloads, subnormals),
    hi equals the upper half-word, for aligned and unaligned buffers."""
    g = torch.Generator().manual_seed(n)
    bits = torch.randint(-2**31, 2**31 - 1, (n + off,), generator=g, dtype=torch.int64).to(torch.int32)
    special = torch.tensor([0, -2**31, 0x7F800000, -8388608, 0x7FC00001, 1, 0x00400000], dtype=torch.int32)
    bits[off:off + min(n, special.numel())] = special[:min(n, special.numel())]
    x = bits.view(torch.float32).to(DEV)[off:]
    hi = torch.empty(n + off, dtype=torch.int16, device=DEV)[off:]
    lo = torch.empty(n + off, dtype=torch.int16, device=DEV)[off:]
    ops.planes_split(x, hi, lo)
    y = torch.empty(n + off, dtype=torch.float32, device=DEV)[off:]
    ops.planes_join(hi, lo, y)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int32).cpu(), bits[off:])
    assert torch.equal(hi.cpu().to(torch.int32) & 0xFFFF, (bits[off:] >> 16) & 0xFFFF)


@pytest.mark.parametrize("tok_key0,d", [(0, 2048), (4096, 64), (2, 64), (0, 30)])
def test_embed_perturb_on_gather_matches_philox(tok_key0, d):
    """zo_embed_fwd (Philox mode): the 4-element vector path (4-aligned keys
    and buffers) gives the same bits as the scalar path at the same keys
    (forced by a misaligned output row), and both equal
    f32(tok[id] + eps z) + f32(pos[t] + eps z) with z from zo_philox_normals
    (reference in float64, one fused rounding)."""
    V, T, B, eps, seed = 97, 16, 3, 1e-3, 0x1234_5678_9ABC
    pos_key0 = tok_key0 + V * d
    g = torch.Generator().manual_seed(d)
    tok = torch.randn(V * d, generator=g).to(DEV)
    pos = torch.randn(T * d, generator=g).to(DEV)
    ids = torch.randint(0, V, (B * T,), generator=g, dtype=torch.int32).to(DEV)
    scal = torch.zeros(4, dtype=torch.int64, device=DEV)
    scal[0] = seed
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    outs = []
    for off in (0, 1):                 # off = 1: output not 16-byte aligned -> scalar path
        buf = torch.full((B * T * d + 4,), float("nan"), device=DEV)
        x = buf[off:off + B * T * d]
        L.check(L.lib().zo_embed_fwd(tok.data_ptr(), tok_key0, pos.data_ptr(), pos_key0, ids.data_ptr(), B, T, d,
                                     V, eps, scal.data_ptr(), L.ZO_Z_PHILOX, 0, 0, x.data_ptr(), d, err.data_ptr(),
                                     L.stream_ptr()))
        outs.append(x.view(B * T, d).clone())
    torch.cuda.synchronize()
    assert err.item() == 0
    assert torch.equal(outs[0], outs[1])
    zt = ops.philox_normals(seed, tok_key0, V * d).view(V, d).double()
    zp = ops.philox_normals(seed, pos_key0, T * d).view(T, d).double()
    e32 = float(torch.tensor(eps, dtype=torch.float32))
    a = (tok.view(V, d).double() + e32 * zt).float()[ids.long()]
    b = (pos.view(T, d).double() + e32 * zp).float().repeat(B, 1)
    torch.testing.assert_close(outs[0], a + b, rtol=0, atol=0)
