"""One GEMM shape, data-parallel or stream-K tail (argv: M N K dp|sk), 5 launches (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200 import ops  # noqa: E402

M, N, K, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
a = torch.randn(M, K, device="cuda").bfloat16()
b = torch.randn(K, N, device="cuda").bfloat16()
bias = torch.randn(N, device="cuda")
o = torch.zeros(M, N, device="cuda")
ws = ops.gemm_workspace(M, N, K) if mode == "sk" else None
for _ in range(5):
    ops.gemm(a, b, L.ZO_EPI_BIAS_RESID_F32, out=o, bias=bias, workspace=ws)
torch.cuda.synchronize()
