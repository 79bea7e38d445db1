"""Where the e2e step's host time goes (StreamingZo.step at the bench shape):
per-phase perf_counter timings of the public step call, and the device-idle
gap between consecutive steps (CUDA events at each step's first and last op)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import zo  # noqa: E402
from paper_2507_03211_b200.engine import init_model  # noqa: E402
from paper_2507_03211_b200 import ZoHyper, iteration_seeds, make_batch, opt_config  # noqa: E402

cfg = opt_config("opt-1.3b", 512)
store = init_model(cfg, 7, init="philox")
sz = zo.StreamingZo(store, ZoHyper(1e-3, 1e-7))
N = 12
seeds = iteration_seeds(1234, N)
batches = [make_batch(cfg, 4, j) for j in range(N)]
for j in range(3):
    sz.step(batches[j], seeds[j])
torch.cuda.synchronize()

phases = {}
orig = {name: getattr(zo, name) for name in ("_stage_batch", "_write_scal", "_finish_record")}


def wrap(name):
    f = orig[name]

    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        phases[name] = phases.get(name, 0.0) + time.perf_counter() - t
        return r
    return g


for name in orig:
    setattr(zo, name, wrap(name))
rep = sz._replay


def rep_t(*a):
    t = time.perf_counter()
    rep(*a)
    phases["_replay"] = phases.get("_replay", 0.0) + time.perf_counter() - t


sz._replay = rep_t
t0 = time.perf_counter()
for j in range(3, N):
    sz.step(batches[j], seeds[j])
wall = (time.perf_counter() - t0) / (N - 3)
n = N - 3
print(f"wall per step {wall * 1e3:.3f} ms")
for k, v in phases.items():
    print(f"  {k:16s} {v / n * 1e3:8.3f} ms")

# device-only replay (no per-step sync) for comparison
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
wsp, wsn = zo._stage_batch(store, batches[0])
s.record()
for j in range(n):
    orig["_write_scal"](store, seeds[j], True)
    rep(wsp, wsn)
e.record()
torch.cuda.synchronize()
print(f"device-timed replay per step {s.elapsed_time(e) / n:.3f} ms")
t = time.perf_counter()
for _ in range(50):
    torch.cuda.synchronize()
print(f"empty synchronize {(time.perf_counter() - t) / 50 * 1e6:.1f} us")

# per-step device windows inside the synchronous public step loop
sz._replay = rep
evs = []
for j in range(n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sz.step(batches[j], seeds[j])
    b.record()
    evs.append((a, b))
torch.cuda.synchronize()
busy = [a.elapsed_time(b) for a, b in evs]
gaps = [evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(n - 1)]
print("device window per sync'd step (ms):", " ".join(f"{x:.3f}" for x in busy))
print("device gap between steps (ms):     ", " ".join(f"{x:.3f}" for x in gaps))
