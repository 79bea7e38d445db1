"""GEMM microbenchmark: tcgen05 kernel per shape/epilogue, CUDA-event timed."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200 import ops  # noqa: E402

shapes = [(2048, 6144, 2048), (2048, 2048, 2048), (2048, 8192, 2048), (2048, 2048, 8192), (2048, 50272, 2048),
          (8192, 8192, 8192)]
epis = {"f32": L.ZO_EPI_F32, "bias": L.ZO_EPI_BIAS_BF16, "gelu": L.ZO_EPI_BIAS_GELU_BF16,
        "resid": L.ZO_EPI_BIAS_RESID_F32}
for M, N, K in shapes:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(K, N, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda")
    o32 = torch.zeros(M, N, device="cuda")
    o16 = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    for en, e in epis.items():
        out = o32 if e in (L.ZO_EPI_F32, L.ZO_EPI_BIAS_RESID_F32) else o16
        f = lambda: ops.gemm(a, b, e, out=out, bias=bias)  # noqa: E731
        f()
        torch.cuda.synchronize()
        s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            f()
        t.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(t) / 20
        print(f"M={M} N={N} K={K} {en:8s} {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.0f} TFLOP/s", flush=True)
    for _ in range(5):            # cuBLAS heuristics / workspace warm-up
        torch.matmul(a, b)
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        torch.matmul(a, b)
    t.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(t) / 20
    print(f"M={M} N={N} K={K} cuBLAS {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.0f} TFLOP/s", flush=True)
