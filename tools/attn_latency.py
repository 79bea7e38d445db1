import sys
import torch
sys.path.insert(0, ".")
from paper_2507_03211_b200 import ops
for B, T, H in [(1, 128, 148), (1, 128, 296), (1, 256, 74), (1, 512, 37), (1, 1024, 18), (1, 2048, 9), (1, 128, 1), (1, 512, 1), (1, 2048, 1)]:
    hd = 64
    qkv = torch.randn(B * T, 3 * H * hd, device="cuda").bfloat16()
    out = torch.empty(B * T, H * hd, device="cuda", dtype=torch.bfloat16)
    f = lambda: ops.attention(qkv, B, T, H, hd, out)
    f(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            f()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    items = H * B * (T // 128)
    blocks = H * B * sum(range(1, T // 128 + 1))
    print(f"B={B} T={T} H={H}: {ms*1e3:7.1f} us  items={items} blocks={blocks} blocks/CTA~{blocks/min(items,148):.1f}")
