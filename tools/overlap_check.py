"""How much do the two directional forwards gain from running on two
streams?  Times (eager launches, CUDA events): perturb pass alone, one
forward alone, the step serialised on one stream, and the dual-stream step."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200 import zo  # noqa: E402
from paper_2507_03211_b200.engine import MINUS, PLUS, DeviceStore  # noqa: E402
from paper_2507_03211_b200.model import make_batch, opt_config  # noqa: E402

cfg = opt_config("opt-1.3b", 512)
store = DeviceStore(cfg, init_seed=7, init="philox")
sz = zo.StreamingZo(store, zo.ZoHyper(1e-3, 1e-7))
wsp, wsn = zo._stage_batch(store, make_batch(cfg, 4, 1))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(c, n=10):
    store.run(c)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(n):
        store.run(c)
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / n


pert = store.perturb_call(store.model_table, L.ZO_PU_UPDATE | L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B, 1e-3, -1e-3)
fwd_p = store.forward_calls(PLUS, wsp, 1e-3)
fwd_m = store.forward_calls(MINUS, wsn, -1e-3)
sz.dual_stream = False
serial = sz.step_calls(wsp, wsn)
sz.dual_stream = True
dual = sz.step_calls(wsp, wsn)
r = {"perturb": timed(pert), "fwd+": timed(fwd_p), "fwd-": timed(fwd_m), "fwd+ then fwd-": timed(fwd_p + fwd_m),
     "step serial": timed(serial), "step dual-stream": timed(dual)}
for k, v in r.items():
    print(f"{k:18s} {v:8.3f} ms")
