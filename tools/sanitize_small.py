"""Small invocations of every hand-written kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_small.py
    compute-sanitizer --tool racecheck python tools/sanitize_small.py
    compute-sanitizer --tool synccheck python tools/sanitize_small.py

GEMM: single-CTA (M=128) and CTA-pair (M>128, stacked split) kernels with every
epilogue incl. CE and the K-major tied head; attention: hd 64 (two-tile kernel,
odd (b,h) count, ragged T), hd 128, and the SIMT kernel; the ZO step (perturb /
update pass, perturb-on-gather embedding, LayerNorm, CE finalize, projected
gradient) at a hd-64 model shape, lazy + eager."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L, ops, zo  # noqa: E402
from paper_2507_03211_b200.engine import DeviceStore  # noqa: E402
from paper_2507_03211_b200.model import Batch, ModelConfig  # noqa: E402

DEV = "cuda"
g = torch.Generator(device=DEV).manual_seed(0)


def rnd(*s, dt=torch.bfloat16, sc=0.5):
    return (torch.randn(*s, device=DEV, generator=g) * sc).to(dt)


for M, N, K in [(128, 384, 192), (512, 512, 320)]:
    a, b, bias = rnd(M, K), rnd(K, N, sc=0.05), rnd(N, dt=torch.float32)
    for epi in (L.ZO_EPI_F32, L.ZO_EPI_BIAS_BF16, L.ZO_EPI_BIAS_GELU_BF16, L.ZO_EPI_BIAS_RELU_BF16,
                L.ZO_EPI_BIAS_RESID_F32):
        out = torch.zeros(M, N, device=DEV, dtype=torch.float32 if epi in (L.ZO_EPI_F32, L.ZO_EPI_BIAS_RESID_F32)
                          else torch.bfloat16)
        ops.gemm(a, b, epi, out=out, bias=bias)
    nt = ops.ce_tiles(N)
    tg = torch.randint(0, N, (M,), device=DEV, dtype=torch.int32)
    part, tl = torch.empty(M, nt, 2, device=DEV), torch.empty(M, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    ops.gemm(a, b, L.ZO_EPI_CE, bias=bias, targets=tg, ce_part=part, ce_tgt=tl, err=err)
    bt = rnd(N, K, sc=0.05)
    ops.gemm(a, bt, L.ZO_EPI_CE | L.ZO_GEMM_B_KMAJOR, targets=tg, ce_part=part, ce_tgt=tl, err=err)
    torch.cuda.synchronize()
    print(f"gemm {M}x{N}x{K} ok", flush=True)

for B, T, H, hd in [(1, 300, 3, 64), (2, 256, 2, 64), (1, 256, 2, 128), (2, 40, 2, 32)]:
    qkv = rnd(B * T, 3 * H * hd)
    out = torch.empty(B * T, H * hd, device=DEV, dtype=torch.bfloat16)
    ops.attention(qkv, B, T, H, hd, out)
    torch.cuda.synchronize()
    print(f"attention B={B} T={T} H={H} hd={hd} ok", flush=True)

cfg = ModelConfig(256, 128, 2, 2, 128, "f32")
store = DeviceStore(cfg, init_seed=3, device=DEV)
rs = np.random.default_rng(1)
batch = Batch(rs.integers(0, 256, (2, 128)).astype(np.int64), rs.integers(0, 256, (2, 128)).astype(np.int64))
sz = zo.StreamingZo(store, zo.ZoHyper(1e-3, 1e-4), graph=False)
for seed in (11, 12, 13):
    sz.step(batch, seed)
sz.flush()
zo.mezo_step(store, batch, zo.ZoHyper(1e-3, 1e-4), 14)
torch.cuda.synchronize()
print("zo steps ok", flush=True)
