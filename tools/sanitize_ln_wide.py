# compute-sanitizer driver for the wide-row LayerNorm kernel (d > 4096), plain and stacked-split
import sys; sys.path.insert(0, ".")
import torch
from paper_2507_03211_b200 import ops, _lib as L
for rows, d in [(37, 5120), (5, 9216), (3, 12288), (9, 7168)]:
    x = torch.randn(rows, d, device="cuda"); g = torch.randn(d, device="cuda"); b = torch.randn(d, device="cuda")
    out = torch.empty(rows, d, dtype=torch.bfloat16, device="cuda")
    ops.layernorm(x, g, b, out)
    g2 = torch.randn(d, device="cuda"); b2 = torch.randn(d, device="cuda")
    L.check(L.lib().zo_layernorm_fwd_split(x.data_ptr(), d, g.data_ptr(), b.data_ptr(), g2.data_ptr(), b2.data_ptr(), rows, rows // 2, d, out.data_ptr(), d, L.stream_ptr()))
torch.cuda.synchronize(); print("ok")
