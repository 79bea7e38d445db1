"""Quick timing probe of the resident ZO step (not the bench contract)."""
import sys
import time

import torch

from paper_2507_03211_b200 import zo
from paper_2507_03211_b200.engine import MINUS, PLUS, DeviceStore
from paper_2507_03211_b200.model import make_batch, opt_config

name = sys.argv[1] if len(sys.argv) > 1 else "opt-1.3b"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
T = int(sys.argv[3]) if len(sys.argv) > 3 else 512
cfg = opt_config(name, T)
t0 = time.time()
store = DeviceStore(cfg, init_seed=7, init="philox")
torch.cuda.synchronize()
print(f"{name} P={store.total_params/1e9:.3f}G init {time.time()-t0:.1f}s", flush=True)
h = zo.ZoHyper(1e-3, 1e-7)
sz = zo.StreamingZo(store, h)
batch = make_batch(cfg, B, 1)
wsp, wsn = zo._stage_batch(store, batch)
calls = sz.step_calls(wsp, wsn)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(c, n=5):
    store.run(c)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(n):
        store.run(c)
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / n


import paper_2507_03211_b200._lib as L
pert = store.perturb_call(store.model_table, L.ZO_PU_UPDATE | L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B, 1e-3, -1e-3)
fwd = store.forward_calls(PLUS, wsp, 1e-3)
tp = timed(pert)
tf = timed(fwd)
ts = timed(calls)
P = store.total_params
print(f"perturb+update {tp:.3f} ms = {P*12/tp/1e6:.0f} GB/s (12 B/param)")
gemm_flops = 2 * B * T * (cfg.n_blocks * 12 * cfg.d_model**2 + cfg.d_model * cfg.vocab_size)
print(f"forward {tf:.3f} ms = {gemm_flops/tf/1e9:.0f} TFLOP/s GEMM-only")
print(f"step {ts:.3f} ms -> {B*T/ts*1e3:.0f} tokens/s")
for i, (fn, args) in enumerate(fwd[:9]):
    t = timed([(fn, args)], 20)
    print(f"  op{i} {fn.__name__} {t*1e3:.1f} us")
