"""Perturb/update kernel microbenchmark at the OPT-1.3B shape (CUDA events)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200.engine import DeviceStore  # noqa: E402
from paper_2507_03211_b200.model import opt_config  # noqa: E402

cfg = opt_config(sys.argv[1] if len(sys.argv) > 1 else "opt-1.3b", 512)
st = DeviceStore(cfg, init="philox")
P = st.total_params
st.set_seed(11)
st.set_pending(1e-7 * 3.0, 7, True)
cases = {
    "update+2 shadows (12 B/param)": (L.ZO_PU_UPDATE | L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B, 12),
    "update+1 shadow (10 B/param)": (L.ZO_PU_UPDATE | L.ZO_PU_SHADOW_A, 10),
    "2 shadows, no update (8 B/param)": (L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B, 8),
    "update only (8 B/param)": (L.ZO_PU_UPDATE, 8),
}
for name, (flags, bpp) in cases.items():
    calls = st.perturb_call(st.model_table, flags, 1e-3, -1e-3)
    st.run(calls)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        st.run(calls)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{name:36s} {ms:7.3f} ms  {P * bpp / ms / 1e6:7.0f} GB/s", flush=True)
