import sys
import torch
sys.path.insert(0, ".")
from paper_2507_03211_b200 import ops  # noqa: E402
for B, T, H, hd in [(4, 512, 32, 64), (8, 512, 32, 64), (1, 2048, 40, 128), (4, 2048, 32, 64)]:
    qkv = torch.randn(B * T, 3 * H * hd, device="cuda").bfloat16()
    out = torch.empty(B * T, H * hd, device="cuda", dtype=torch.bfloat16)
    f = lambda: ops.attention(qkv, B, T, H, hd, out)  # noqa: E731
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        f()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    fl = 4 * B * H * T * T * hd / 2
    print(f"B={B} T={T} H={H} hd={hd}: {ms*1e3:.1f} us  {fl/ms/1e9:.0f} TFLOP/s (causal)")
