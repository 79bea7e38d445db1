"""clock64 timeline of CTA 0 of the hd-64 ping-pong attention kernel
(attn_pp_kernel): tile A's softmax warp 2, the MMA warp and the producer, from
a trace build:

    ZO_NVCC_EXTRA=-DZO_ATTN_TRACE python -c "from paper_2507_03211_b200 import build_lib as b; b.build(force=True)"
    mkdir -p build/alt && cp paper_2507_03211_b200/lib/libzo_b200.so build/alt/libzo_trace.so
    python -c "from paper_2507_03211_b200 import build_lib as b; b.build(force=True)"   # normal library back
"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ["ZO_B200_LIB"] = os.path.abspath("build/alt/libzo_trace.so")
from paper_2507_03211_b200 import _lib as L, ops  # noqa: E402
B, T, H, hd = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (8, 512, 32, 64)))
qkv = torch.randn(B * T, 3 * H * hd, device="cuda").bfloat16()
out = torch.empty(B * T, H * hd, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.attention(qkv, B, T, H, hd, out)
torch.cuda.synchronize()
dll = ctypes.CDLL(L.LIB_PATH)
buf = (ctypes.c_longlong * 4096)()
dll.zo_attn_trace_read(buf)
a = np.array(buf[:], dtype=np.int64)
t0 = min(v for v in a if v > 0)
rel = lambda v: int(v - t0) if v > 0 else -1  # noqa: E731
n_qt, n_pairs = (T + 127) // 128, (B * H + 1) // 2
items = n_qt * n_pairs
grid = min(items, 148)
print(f"B={B} T={T} H={H}: {items} items over {grid} CTAs; CTA 0 timeline (cycles)")
blk, m, kv = 0, 0, 0
for it in range(0, items, grid):
    qt = n_qt - 1 - it // n_pairs
    nkb = qt + 1
    print(f"item {it} qt={qt} ({nkb} blocks)")
    seq = [("S", 0, 0), ("S", 1, 0)]
    for j in range(nkb):
        if j + 1 < nkb:
            seq += [("S", 0, j + 1), ("S", 1, j + 1)]
        seq += [("PV", 0, j), ("PV", 1, j)]
    for kind, t, j in seq:
        r = a[1024 + 4 * m: 1024 + 4 * m + 3]
        if kind == "S":
            print(f"   MMA S {'AB'[t]}{j}: start {rel(r[0])} kv-ok {rel(r[1])} s-free {rel(r[2])}")
        else:
            print(f"   MMA PV {'AB'[t]}{j}: start {rel(r[0])} P-seen {rel(r[1])}")
        m += 1
    for j in range(nkb):
        r = a[blk * 8: blk * 8 + 8]
        print(f"   softmax A blk {j}: wait-S {rel(r[0])} S-ok {rel(r[1])} max {rel(r[2])} pv-ok {rel(r[3])} "
              f"exp+st {rel(r[4])} P-done {rel(r[5])}")
        blk += 1
    print(f"   softmax A end: PV-ok {rel(a[blk * 8 - 2])}")
    for j in range(nkb):
        for t in range(2):
            print(f"   TMA kv {kv} ({'AB'[t]}{j}): wait {rel(a[2048 + 2 * kv])} go {rel(a[2048 + 2 * kv + 1])}")
            kv += 1
