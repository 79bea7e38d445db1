"""A/B of the stream-K tail policies at the stacked step's GEMM shapes."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200 import ops  # noqa: E402


def t(f, n=30):
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


for M, N, K in [(4096, 6144, 2048), (4096, 2048, 2048), (4096, 8192, 2048), (4096, 2048, 8192)]:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(K, N, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda")
    o = torch.zeros(M, N, device="cuda")
    ws = ops.gemm_workspace(M, N, K)
    dp = t(lambda: ops.gemm(a, b, L.ZO_EPI_BIAS_RESID_F32, out=o, bias=bias))
    sk = t(lambda: ops.gemm(a, b, L.ZO_EPI_BIAS_RESID_F32, out=o, bias=bias, workspace=ws)) if ws.numel() > 256 else float("nan")
    print(f"policy={os.environ.get('ZO_SK_POLICY', 'two-wave')} M={M} N={N} K={K} dp {dp:7.1f} us  sk {sk:7.1f} us", flush=True)
