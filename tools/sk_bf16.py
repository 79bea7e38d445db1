"""Stream-K vs data-parallel for bf16-output epilogues (QKV bias, FFN-up GELU)
at the stacked step's shapes; L2 flushed between launches."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200 import ops  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(f, n=30):
    f()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(n):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / n * 1e3


for M, N, K, epi in [(4096, 6144, 2048, L.ZO_EPI_BIAS_BF16), (4096, 8192, 2048, L.ZO_EPI_BIAS_GELU_BF16),
                     (4096, 2048, 2048, L.ZO_EPI_BIAS_BF16), (4096, 2048, 8192, L.ZO_EPI_BIAS_BF16)]:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = (torch.randn(K, N, device="cuda") * 0.05).bfloat16()
    bias = torch.randn(N, device="cuda")
    o = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    ws = ops.gemm_workspace(M, N, K)
    dp = t(lambda: ops.gemm(a, b, epi, out=o, bias=bias))
    sk = t(lambda: ops.gemm(a, b, epi, out=o, bias=bias, workspace=ws)) if ws.numel() > 256 else float("nan")
    print(f"policy={os.environ.get('ZO_SK_POLICY', 'two-wave')} M={M} N={N} K={K} epi={epi} dp {dp:7.1f} us  sk {sk:7.1f} us",
          flush=True)
