"""zo_gemm_resid_ln vs the residual GEMM + separate LayerNorm at the stacked
step's O-proj / FFN-down shapes (CUDA events, 50 launches each, alternating).
ZO_B200_LIB selects a library variant (tools/build_variants.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_03211_b200 import _lib as L

lib = L.lib()
dev = "cuda"
torch.manual_seed(0)


def r(*s, dt=torch.bfloat16, sc=0.05):
    return (torch.randn(*s, device=dev) * sc).to(dt)


for (M, N, K) in [(4096, 2048, 2048), (4096, 2048, 8192)]:
    sp = M // 2
    a, b1, b2 = r(M, K, sc=0.5), r(K, N), r(K, N)
    bias1, bias2 = r(N, dt=torch.float32), r(N, dt=torch.float32)
    g1, be1, g2, be2 = (r(N, dt=torch.float32, sc=1.0) for _ in range(4))
    x = torch.randn(M, N, device=dev)
    h = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    stats = torch.empty(M, N // 128, 2, device=dev)
    ctr = torch.zeros(2 * (M // 256), dtype=torch.int32, device=dev)
    st = L.stream_ptr()

    def fused():
        L.check(lib.zo_gemm_resid_ln(a.data_ptr(), K, b1.data_ptr(), b2.data_ptr(), N, M, N, K, sp, bias1.data_ptr(),
                                     bias2.data_ptr(), x.data_ptr(), N, g1.data_ptr(), be1.data_ptr(), g2.data_ptr(),
                                     be2.data_ptr(), h.data_ptr(), N, stats.data_ptr(), ctr.data_ptr(), st))

    def gemm():
        L.check(lib.zo_gemm_bf16_split(a.data_ptr(), K, b1.data_ptr(), b2.data_ptr(), N, M, N, K, sp,
                                       L.ZO_EPI_BIAS_RESID_F32, bias1.data_ptr(), bias2.data_ptr(), x.data_ptr(), N,
                                       0, 0, 0, 0, st))

    def ln():
        L.check(lib.zo_layernorm_fwd_split(x.data_ptr(), N, g1.data_ptr(), be1.data_ptr(), g2.data_ptr(),
                                           be2.data_ptr(), M, sp, N, h.data_ptr(), N, st))

    def t(fn, n=50):
        for _ in range(5):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3

    for rep in range(2):
        tf, tg, tl = t(fused), t(gemm), t(ln)
        print(f"{M}x{N}x{K}: fused {tf:6.1f} us | gemm {tg:6.1f} + ln {tl:5.1f} = {tg + tl:6.1f} us")
