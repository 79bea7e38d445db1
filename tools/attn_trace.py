"""Per-CTA timeline of the tcgen05 attention kernel (clock64 stamps of CTA 0's
softmax warp 2, MMA warp and producer), from a trace build:

    ZO_NVCC_EXTRA=-DZO_ATTN_TRACE python -c "from paper_2507_03211_b200 import build_lib as b; b.build(force=True)"
    cp paper_2507_03211_b200/lib/libzo_b200.so build/alt/libzo_trace.so   # then rebuild the normal library

(the TR / TRW / TRP stamps in csrc/attention_tc.cu compile to nothing
without ZO_ATTN_TRACE; profiles/r01_attn_trace_cta0.txt is this tool's output
at the stacked step's shape)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ["ZO_B200_LIB"] = os.path.abspath("build/alt/libzo_trace.so")
from paper_2507_03211_b200 import _lib as L, ops
B, T, H, hd = 8, 512, 32, 64
qkv = torch.randn(B * T, 3 * H * hd, device="cuda").bfloat16()
out = torch.empty(B * T, H * hd, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.attention(qkv, B, T, H, hd, out)
torch.cuda.synchronize()
dll = ctypes.CDLL(L.LIB_PATH)
buf = (ctypes.c_longlong * 4096)()
print("rc", dll.zo_attn_trace_read(buf))
a = np.array(buf[:], dtype=np.int64)
t0 = min(v for v in a if v > 0)
rel = lambda v: (v - t0) if v > 0 else -1
items = 1024 // 148 + 1
n_qt, n_bh = 4, B * H
c = 0
for it_local in range(items):
    it = it_local * 148
    if it >= 1024: break
    qt = n_qt - 1 - it // n_bh
    nkb = qt + 1
    row = a[it_local * 32: it_local * 32 + 32]
    print(f"item {it_local} (qt={qt}, {nkb} blocks): start {rel(row[0])}  Qload {rel(a[3072 + it_local])}")
    for j in range(nkb):
        print(f"   blk {j}: pre-S {rel(row[1+3*j])} S-ready {rel(row[2+3*j])} P-done {rel(row[3+3*j])} | MMA: kv-wait {rel(a[1024+4*c])} kv-ok {rel(a[1024+4*c+1])} sfree {rel(a[1024+4*c+2])} P-seen {rel(a[1024+4*c+3])} | KV issued {rel(a[2048+c])}")
        c += 1
    print(f"   end: pre-PV {rel(row[20])} PV-ok {rel(row[21])} out-done {rel(row[22])}")
