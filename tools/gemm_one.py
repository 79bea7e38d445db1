"""Run one GEMM shape/epilogue a few times (for ncu captures).

    python tools/gemm_one.py M N K epi [reps]      epi in f32|bias|gelu|resid
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200 import ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
epi = {"f32": L.ZO_EPI_F32, "bias": L.ZO_EPI_BIAS_BF16, "gelu": L.ZO_EPI_BIAS_GELU_BF16,
       "resid": L.ZO_EPI_BIAS_RESID_F32}[sys.argv[4]]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
a = torch.randn(M, K, device="cuda").bfloat16()
b = torch.randn(K, N, device="cuda").bfloat16()
bias = torch.randn(N, device="cuda")
out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi in (L.ZO_EPI_F32, L.ZO_EPI_BIAS_RESID_F32)
                  else torch.bfloat16)
for _ in range(reps):
    ops.gemm(a, b, epi, out=out, bias=bias)
torch.cuda.synchronize()
print("ok")
