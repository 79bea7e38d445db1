"""A/B: the same GEMM with B MN-major ([K, N], weights as stored) vs B
K-major ([N, K], ZO_GEMM_B_KMAJOR), CUDA-event timed, plus cuBLAS."""
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


for M, N, K in [(4096, 6144, 2048), (4096, 2048, 2048), (4096, 8192, 2048), (4096, 2048, 8192), (4096, 50272, 2048), (8192, 8192, 8192)]:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(K, N, device="cuda").bfloat16()
    bt = b.t().contiguous()
    o = torch.empty(M, N, device="cuda")
    mn = t(lambda: ops.gemm(a, b, L.ZO_EPI_F32, out=o))
    km = t(lambda: ops.gemm(a, bt, L.ZO_EPI_F32 | L.ZO_GEMM_B_KMAJOR, out=o))
    cb = t(lambda: torch.matmul(a, b))
    cbt = t(lambda: torch.matmul(a, bt.t()))
    fl = 2 * M * N * K / 1e6
    print(f"M={M} N={N} K={K}: MN-major {mn:7.1f} us ({fl/mn:5.0f} TF)  K-major {km:7.1f} us ({fl/km:5.0f} TF)  "
          f"cuBLAS {cb:7.1f} us ({fl/cb:5.0f} TF)  cuBLAS(B^T) {cbt:7.1f} us ({fl/cbt:5.0f} TF)", flush=True)
