"""PCIe numbers behind the offload rows: pinned H2D / D2H GB/s for one
OPT-13B-shape transformer block (fp32, 1.26 GB), alone and concurrently on
two streams (the U / O streams of scheduler.OffloadedZo), and the
reference's T_comm model (comm.py:250-256) evaluated with the measured
bandwidth for n = 1 (no peers on this box)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200.model import model_layout, opt_config  # noqa: E402
from paper_2507_03211_b200.scheduler import sliced_upload_time  # noqa: E402

n = model_layout(opt_config("opt-13b", 2048))[1].elem_count
host = torch.empty(n, dtype=torch.float32, pin_memory=True)
host2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
dev = torch.empty(n, dtype=torch.float32, device="cuda")
dev2 = torch.empty(n, dtype=torch.float32, device="cuda")
su, so = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def both():
    ev = torch.cuda.Event()
    ev.record()
    su.wait_event(ev)
    so.wait_event(ev)
    with torch.cuda.stream(su):
        dev.copy_(host, non_blocking=True)
    with torch.cuda.stream(so):
        host2.copy_(dev2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(su)
    torch.cuda.current_stream().wait_stream(so)


t_h2d = timed(lambda: dev.copy_(host, non_blocking=True))
t_d2h = timed(lambda: host2.copy_(dev2, non_blocking=True))
t_both = timed(both)
nb = n * 4
out = {"block_bytes": nb, "h2d_gbs": nb / t_h2d / 1e9, "d2h_gbs": nb / t_d2h / 1e9,
       "bidirectional_gbs_each_way": nb / t_both / 1e9, "pcie_gen5_x16_spec_gbs": 64.0,
       "tcomm_model_s_n1": sliced_upload_time(n, 1, nb / t_h2d / 4, 1.0), "measured_h2d_s": t_h2d}
print(json.dumps(out))
