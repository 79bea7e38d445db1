"""Host-side cost of StreamingZo.step at the bench config: wall per step vs
device time per step, and a cProfile of the host path (what runs between
the previous step's sync and the next graph launch)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_03211_b200 import zo
from paper_2507_03211_b200.engine import DeviceStore
from paper_2507_03211_b200.model import ModelConfig, make_batch
from paper_2507_03211_b200.rng import iteration_seeds

plan = sys.argv[1] if len(sys.argv) > 1 else "fill"
cfg = ModelConfig(50272, 2048, 32, 24, 512, "f32")
store = DeviceStore(cfg, init_seed=7, device="cuda:0", init="philox")
api = zo.StreamingZo(store, zo.ZoHyper(1e-3, 1e-7), overlap=plan)
n = 30
seeds = iteration_seeds(1234, n)
batches = [make_batch(cfg, 4, 42 * 1_000_003 + j) for j in range(n)]
for j in range(5):
    api.step(batches[j], seeds[j])
torch.cuda.synchronize()
t0 = time.perf_counter()
for j in range(5, 15):
    api.step(batches[j], seeds[j])
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / 10 * 1e3
# device time of the same graph replays back to back (no host round trip)
ws = store.workspace(0, 4, 512), store.workspace(1, 4, 512)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for j in range(10):
    api._replay(*ws)
e1.record()
torch.cuda.synchronize()
dev = e0.elapsed_time(e1) / 10
print(f"plan {plan}: e2e wall {wall:.3f} ms/step, back-to-back replay {dev:.3f} ms/step, gap {wall - dev:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for j in range(15, 30):
    api.step(batches[j], seeds[j])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
