"""Run the ZO step at the larger BASELINE.json shapes on ONE GPU (evidence
for configs #3-#5; the bench line is config #2).

    python tools/run_config.py resident opt-13b 2048 1      # 13B, T=2048, B=1, both directions
    python tools/run_config.py offload  opt-66b 2048 1      # ZO2 schedule, host master, 3 slots
    python tools/run_config.py sharded  opt-13b 2048 1      # same schedule, fp32 master in HBM (1 rank)
    python tools/run_config.py offload:20 opt-13b 2048 1    # 20 of 40 blocks resident, the rest streamed
    python tools/run_config.py resident opt-175b/4 2048 1   # 4 decoder blocks of the OPT-175B shape
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_03211_b200 import zo  # noqa: E402
from paper_2507_03211_b200.engine import DeviceStore  # noqa: E402
from paper_2507_03211_b200.model import make_batch, opt_config  # noqa: E402
from paper_2507_03211_b200.rng import iteration_seeds  # noqa: E402


def main():
    mode, name, T, B = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
    if "/" in name:          # "<shape>/<n>": n decoder blocks of that shape (per-block rates of 66B / 175B)
        import dataclasses

        base, nb = name.split("/")
        cfg = dataclasses.replace(opt_config(base, T), n_blocks=int(nb)).validate()
    else:
        cfg = opt_config(name, T)
    hyper = zo.ZoHyper(1e-3, 1e-7)
    t0 = time.time()
    if mode == "resident":
        store = DeviceStore(cfg, init_seed=7, init="philox")
        rt = zo.StreamingZo(store, hyper)
    elif mode == "sharded":
        from paper_2507_03211_b200.scheduler import OffloadedZo
        from paper_2507_03211_b200.sharded import ShardStore
        shards = ShardStore(cfg, None, 7, init="philox")
        rt = OffloadedZo(shards, hyper, batch=B, trace=True)
    else:   # "offload", "offload:K" (K blocks resident) or "offload:budget=GB" (plan_residency),
        # optionally ":split16" (hi / lo plane transfer compression)
        from paper_2507_03211_b200.scheduler import HostStore, OffloadedZo, plan_residency
        parts = mode.split(":")
        compress = "split16" if "split16" in parts[1:] else "none"
        rest = [p for p in parts[1:] if p != "split16"]
        arg = rest[0] if rest else "0"
        if arg.startswith("budget="):
            k, slots = plan_residency(cfg, int(float(arg.split("=")[1]) * 1e9), compress=compress)
        else:
            k, slots = int(arg), (6 if int(arg) else 3)
        host = HostStore(cfg, 7, init="philox")
        rt = OffloadedZo(host, hyper, batch=B, trace=True, resident_blocks=k, n_slots=max(slots, 2),
                         compress=compress)
    torch.cuda.synchronize()
    init_s = time.time() - t0
    seeds = iteration_seeds(1234, steps)
    walls = []
    for j, s in enumerate(seeds):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = rt.step(make_batch(cfg, B, 99 * 1_000_003 + j + 1), s)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t)
    med = sorted(walls[1:])[len(walls[1:]) // 2] if len(walls) > 1 else walls[0]
    out = {"mode": mode, "model": name, "params": cfg.param_count(), "seq": T, "batch": B,
           "init_s": round(init_s, 1), "step_ms": [round(w * 1e3, 2) for w in walls],
           "median_step_ms": round(med * 1e3, 2), "tokens_per_s": B * T / med,
           "loss_pos": r.loss_pos, "loss_neg": r.loss_neg, "g": r.g,
           "peak_device_gb": round(torch.cuda.max_memory_allocated() / 1e9, 2)}
    if mode != "resident":
        tl = rt.last_timeline
        busy = {k: sum(e["end"] - e["start"] for e in tl if e["op"] == k) for k in ("upload", "compute", "offload")}
        out["stream_busy_ms"] = {k: round(v, 2) for k, v in busy.items()}
        out["makespan_ms"] = round(rt.makespan(), 2)
        if hasattr(rt, "pcie_bytes_per_step"):
            out["pcie_gb_per_step"] = [round(b / 1e9, 2) for b in rt.pcie_bytes_per_step()]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
