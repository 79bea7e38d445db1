"""Does the HBM/ALU-bound perturb pass overlap the tensor-core-bound forward?"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import _lib as L  # noqa: E402
from paper_2507_03211_b200 import zo  # noqa: E402
from paper_2507_03211_b200.engine import MINUS, PLUS, DeviceStore  # noqa: E402
from paper_2507_03211_b200.model import make_batch, opt_config  # noqa: E402

cfg = opt_config("opt-1.3b", 512)
st = DeviceStore(cfg, init="philox")
st.set_seed(5)
st.set_pending(0.0, 0, False)
batch = make_batch(cfg, 4, 1)
wsp, wsn = zo._stage_batch(st, batch)
main = torch.cuda.current_stream()
side = torch.cuda.Stream()
fwd = st.forward_calls(PLUS, wsp, 1e-3)
pert = st.perturb_call(st.model_table, L.ZO_PU_SHADOW_B, 0.0, -1e-3, sa=None, sb=MINUS, stream=side)


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(main)
    for _ in range(n):
        fn()
    e.record(main)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


def both():
    ev = torch.cuda.Event()
    ev.record(main)
    side.wait_event(ev)
    st.run(pert)
    st.run(fwd)
    ev2 = torch.cuda.Event()
    ev2.record(side)
    main.wait_event(ev2)


def pert_only():
    ev = torch.cuda.Event()
    ev.record(main)
    side.wait_event(ev)
    st.run(pert)
    ev2 = torch.cuda.Event()
    ev2.record(side)
    main.wait_event(ev2)


tf = t(lambda: st.run(fwd))
tp = t(pert_only)
tb = t(both)
print(f"forward alone {tf:.3f} ms, perturb(1 shadow, no update) alone {tp:.3f} ms, concurrent {tb:.3f} ms "
      f"(serial sum {tf + tp:.3f})")

# the two directional forwards concurrently on two streams
fwdn = st.forward_calls(MINUS, wsn, -1e-3, stream=side)
st.run(st.perturb_call(st.model_table, L.ZO_PU_SHADOW_A | L.ZO_PU_SHADOW_B, 1e-3, -1e-3))
torch.cuda.synchronize()


def two_fwd_serial():
    st.run(fwd)
    st.run(st.forward_calls(MINUS, wsn, -1e-3))


def two_fwd_concurrent():
    ev = torch.cuda.Event()
    ev.record(main)
    side.wait_event(ev)
    st.run(fwd)
    st.run(fwdn)
    ev2 = torch.cuda.Event()
    ev2.record(side)
    main.wait_event(ev2)


ts = t(two_fwd_serial)
tc = t(two_fwd_concurrent)
print(f"two forwards serial {ts:.3f} ms, concurrent on 2 streams {tc:.3f} ms")
