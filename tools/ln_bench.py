"""LayerNorm microbenchmark at the stacked step's shape (4096 x 2048 fp32 ->
bf16), warm (inputs L2-resident after the first launch) and cold (a 256 MB
buffer written between launches), vs a torch copy of the same bytes."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import ops  # noqa: E402

rows, d = 4096, 2048
x = torch.randn(rows, d, device="cuda")
g, b = torch.randn(d, device="cuda"), torch.randn(d, device="cuda")
out = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
flush = torch.empty(64 << 20, device="cuda")


def t(f, cold, n=20):
    f()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(n):
        if cold:
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / n * 1e3


nbytes = rows * d * 6
for cold in (False, True):
    ln = t(lambda: ops.layernorm(x, g, b, out), cold)
    cp = t(lambda: out.copy_(x), cold)
    print(f"{'cold' if cold else 'warm'}: layernorm {ln:6.1f} us ({nbytes / ln / 1e3:5.0f} GB/s)   "
          f"torch fp32->bf16 copy {cp:6.1f} us ({nbytes / cp / 1e3:5.0f} GB/s)")
