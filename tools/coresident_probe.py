"""Can the perturb pass hide under the forward's GEMMs?  Times (CUDA events)
the background perturb pass alone, the stacked forward GEMM sequence alone,
and both launched concurrently on two streams.  Env: ZO_PU_BG_CTAS (CTAs per
SM of the background pass), ZO_B200_LIB (library variant)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200 import zo  # noqa: E402
from paper_2507_03211_b200.engine import MINUS, PLUS, DeviceStore  # noqa: E402
from paper_2507_03211_b200.model import make_batch, opt_config  # noqa: E402

cfg = opt_config("opt-1.3b", 512)
store = DeviceStore(cfg, init_seed=7, init="philox")
sz = zo.StreamingZo(store, zo.ZoHyper(1e-3, 1e-7), overlap="stacked")
wsp, wsn = zo._stage_batch(store, make_batch(cfg, 4, 1))
ws = store.stacked_workspace(4, 512)
store.set_pending(1e-7 * 3.0, 7, True)
nb = len(store.layouts)
table = store.range_table(0, nb)
flags = L.ZO_PU_UPDATE | L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B
P, F = torch.cuda.Stream(), torch.cuda.Stream()
pert = store.perturb_bg_call(table, flags, 1e-3, -1e-3, stream=P)
fwd = [c for c in store.forward_calls_stacked(ws, 1e-3, stream=F) if c[0].__name__ == "zo_gemm_bf16_split"]


def run_timed(calls, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    store.run(calls)
    e1.record(stream)
    return e0, e1


def once(mode):
    torch.cuda.synchronize()
    store.block_done.zero_()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(torch.cuda.current_stream())
    P.wait_event(t0)
    F.wait_event(t0)
    out = {}
    if mode in ("pert", "both"):
        out["pert"] = run_timed(pert, P)
    if mode in ("fwd", "both"):
        out["fwd"] = run_timed(fwd, F)
    torch.cuda.synchronize()
    r = {k: a.elapsed_time(b) for k, (a, b) in out.items()}
    if mode == "both":
        r["union"] = max(t0.elapsed_time(b) for (_, b) in out.values())
    return r


for mode in ("pert", "fwd", "both"):
    once(mode)
    rs = [once(mode) for _ in range(3)]
    avg = {k: sum(r[k] for r in rs) / len(rs) for k in rs[0]}
    gflop = sum(2.0 * a[5] * a[6] * a[7] for _, a in fwd) / 1e9
    extra = f" GEMM {gflop / avg['fwd']:.0f} TFLOP/s" if "fwd" in avg else ""
    extra += f" perturb {store.total_params * 12 / avg['pert'] / 1e6:.0f} GB/s" if "pert" in avg else ""
    print(f"bg_ctas={os.environ.get('ZO_PU_BG_CTAS', '1')} lib={os.path.basename(L.LIB_PATH)} {mode:5s} "
          + " ".join(f"{k}={v:.3f}ms" for k, v in avg.items()) + extra, flush=True)
