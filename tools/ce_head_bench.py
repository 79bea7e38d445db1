"""LM-head GEMM at the stacked step's shape (M=4096, V=50272, d=2048):
CE epilogue (per-row max / sum-exp partials, logits never stored) vs the
plain bias epilogue writing bf16 logits, CUDA-event timed."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200 import ops  # noqa: E402

M, V, K = 4096, 50272, 2048
a = torch.randn(M, K, device="cuda").bfloat16() * 0.5
b = (torch.randn(K, V, device="cuda") * 0.02).bfloat16()
bias = torch.randn(V, device="cuda") * 0.1
tg = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
nt = ops.ce_tiles(V)
part, tl = torch.empty(M, nt, 2, device="cuda"), torch.empty(M, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
o16 = torch.empty(M, V, device="cuda", dtype=torch.bfloat16)


def t(f, n=20):
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


ce = t(lambda: ops.gemm(a, b, L.ZO_EPI_CE, bias=bias, targets=tg, ce_part=part, ce_tgt=tl, err=err))
bf = t(lambda: ops.gemm(a, b, L.ZO_EPI_BIAS_BF16, out=o16, bias=bias))
f32 = t(lambda: ops.gemm(a, b, L.ZO_EPI_F32, out=torch.empty(0, device="cuda") if False else o16.view(torch.float32)[:, :V // 2] if False else None, bias=None) if False else 0)
fl = 2 * M * V * K / 1e6
print(f"CE epilogue {ce:7.1f} us ({fl / ce:5.0f} TF)   bias->bf16 {bf:7.1f} us ({fl / bf:5.0f} TF)")
