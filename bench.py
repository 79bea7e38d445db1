#!/usr/bin/env python
"""Benchmark of the B200-native ZO training step (DistZO2 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

Workload (BASELINE.json configs[1]): OPT-1.3B-shaped zosim model (V=50272,
d=2048, H=32, 24 blocks, T=512), synthetic tokens, random-init weights, ZO-SGD
with eps=1e-3, lr=1e-7, batch 4 sequences per PertP group.
  N=1   both directions on one GPU (the lazy-update MeZO/ZO2 step, Alg. 2)
  N=2   Perturbation Parallelism: rank 0 the +eps forward, rank 1 the -eps
  N=2k  2D mesh, k groups x 2 directions, batch 4 per group (weak scaling)
One step = fused update(j-1)+perturb(j) pass + forward(s) + loss + g.

Prints ONE JSON line (rank 0).  `value` is device-timed tokens/s with inputs
resident; `e2e` is the same metric through the public API
(StreamingZo.step / strategies) with host batches copied in and the step
record read back every step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

EPS, LR = 1e-3, 1e-7
MODEL, SEQ, BATCH_PER_GROUP = "opt-1.3b", 512, 4
BASE_SEED, DATA_SEED = 1234, 99


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default=MODEL)
    ap.add_argument("--arch", default="zosim", choices=["zosim", "opt"],
                    help="zosim: the reference's architecture at OPT dims (the headline); opt: real OPT "
                         "(ReLU, tied head, position offset) -- a comparison row")
    ap.add_argument("--seq", type=int, default=SEQ)
    ap.add_argument("--batch", type=int, default=BATCH_PER_GROUP, help="sequences per PertP group")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the public-API pass (profiling runs)")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly instead of replaying a CUDA graph")
    ap.add_argument("--overlap", default="stacked", choices=["none", "blocks", "background", "stacked", "stacked_bg"],
                    help="none: the two forwards on two streams; blocks: per-block perturb passes on a side stream ahead of the +eps forward; "
                         "background: one co-resident perturb pass gated per block by device counters; "
                         "stacked: both directions as one launch per layer over stacked activations")
    return ap.parse_args()


def _config(args):
    from paper_2507_03211_b200.model import opt_config, real_opt_config

    return real_opt_config(args.model, args.seq) if args.arch == "opt" else opt_config(args.model, args.seq)


def _plan(args):
    return {"none": False, "blocks": "blocks", "background": "background", "stacked": "stacked",
            "stacked_bg": "stacked_bg"}[args.overlap]


def _plan_text(args, world):
    if world > 1 or args.overlap == "none":
        return "one launch; timed alone in a serialised replay"
    if args.overlap == "stacked":
        return "one launch; both directions' forwards stacked into one launch per layer"
    if args.overlap == "blocks":
        return "timed run: one launch per block on a side stream ahead of the +eps forward; timed alone in a serialised replay"
    return ("timed run: block 0 full-width, the rest as one co-resident background launch gating each block's "
            "forward by a device counter; timed alone in a serialised replay")


# ----------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md recipe)
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            for line in out.strip().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == 7:
                    self.rows.append(parts)

    def summary(self) -> dict:
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _traffic():
    """DRAM bytes per launch (perturb) / per step (all GEMM launches) from the
    committed ncu capture of this bench (profiles/ncu_traffic.json, written by
    tools/traffic_from_ncu.py from a `--metrics dram__bytes_*` launch list)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops_sustained"]), float(p["bf16_tflops"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1400.0, 1590.0, "fallback"


# ----------------------------------------------------------------------------
# CPU reference sample (oracle port of zosim, bounded)
# ----------------------------------------------------------------------------
def cpu_reference_sample(cfg, batch: int, rows_frac: float = 0.125, param_frac: float = 0.25) -> dict:
    """Time the reference's CPU algorithm (oracle/zo_oracle.py, a bit-exact
    restatement of zosim) on a bounded sample of ONE step and extrapolate:
      - z draw + perturb/restore/update arithmetic: 4 z passes per parameter
        (zo.py:154-167) timed on `param_frac` of one transformer block;
      - 2 forwards of one transformer block at the full (B, T);
      - 2 LM-head forwards + CE on `rows_frac` of the rows.
    Step time = P * t_param + N * t_block_fwd + t_head / rows_frac."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import zo_oracle as O

    d, V, T, N = cfg.d_model, cfg.vocab_size, cfg.seq_len, cfg.n_blocks
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(0)
    with threadpool_limits(limits=cores):
        pblk = 12 * d * d + 13 * d
        n = int(pblk * param_frac)
        base = (0.02 * rng.standard_normal(n)).astype(np.float32)
        t0 = time.perf_counter()
        gen = np.random.Generator(np.random.PCG64(7))
        for sc in (+EPS, -EPS, 0.0):      # +eps, -2eps (-> -eps), restore
            z = gen.standard_normal(n)
            O.perturbed(base, sc, z)
        z = gen.standard_normal(n)
        O.updated(base, 0.5, LR, z)
        t_param = (time.perf_counter() - t0) / n
        blk = (0.02 * rng.standard_normal(pblk)).astype(np.float32)
        x = rng.standard_normal((batch, T, d)).astype(np.float32)
        t0 = time.perf_counter()
        for _ in range(2):
            O.block_forward("transformer", blk, V, d, T, cfg.n_heads, x)
        t_block = time.perf_counter() - t0
        rows = max(1, int(batch * T * rows_frac))
        head = (0.02 * rng.standard_normal(2 * d + d * V + V)).astype(np.float32)
        xh = rng.standard_normal((1, rows, d)).astype(np.float32)
        tg = rng.integers(0, V, (1, rows))
        t0 = time.perf_counter()
        for _ in range(2):
            O.cross_entropy(O.block_forward("head", head, V, d, T, cfg.n_heads, xh), tg)
        t_head = (time.perf_counter() - t0) * (batch * T / rows)
    P = cfg.param_count()
    step = P * t_param + N * t_block + t_head
    return {"step_s": step, "tokens_per_s": batch * T / step, "cores": cores,
            "sample": (f"zosim oracle port (numpy, BLAS {cores} threads, z on 1 core): 4 z passes on "
                       f"{param_frac:g} of one transformer block, 2 forwards of 1/{N} blocks at B={batch},T={T}, "
                       f"2 LM-head forwards+CE on {rows_frac:g} of rows; extrapolated to P={P}")}


def reference_arm(args, rank, world):
    from paper_2507_03211_b200.model import opt_config

    if rank != 0:
        return
    cfg = _config(args)
    n_groups = max(1, args.gpus // 2)
    batch = args.batch * n_groups
    for _ in range(args.warmup):
        cpu_reference_sample(cfg, batch, rows_frac=0.03125, param_frac=0.0625)
    samples = [cpu_reference_sample(cfg, batch, rows_frac=0.03125, param_frac=0.0625) for _ in range(args.steps)]
    vals = [s["tokens_per_s"] for s in samples]
    v = statistics.median(vals)
    ms = 1e3 * statistics.median([s["step_s"] for s in samples])
    line = {"metric": "OPT ZO fine-tune tokens/s (zosim arch, OPT-1.3B shape)", "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.model} ZO-SGD step, seq {args.seq}, batch {args.batch}/group",
                       "global_batch": batch, "seq_len": args.seq, "strategy": "mezo (CPU reference)"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": samples[0]["cores"], "kind": "port",
                             "sample": samples[0]["sample"]},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2507_03211_b200 import _lib as L
    from paper_2507_03211_b200 import zo
    from paper_2507_03211_b200.engine import MINUS, PLUS, DeviceStore
    from paper_2507_03211_b200.model import make_batch, opt_config
    from paper_2507_03211_b200.rng import iteration_seeds

    torch.cuda.set_device(local_rank)
    dev = torch.device(f"cuda:{local_rank}")
    cfg = _config(args)
    B, T = args.batch, args.seq
    M = B * T
    hyper = zo.ZoHyper(EPS, LR)
    if world == 1:
        strategy, n_groups, dirs = "mezo-lazy (both directions, 1 GPU)", 1, (PLUS, MINUS)
    else:
        if world % 2:
            raise SystemExit("world size must be 1 or even (PertP pairs)")
        n_groups = world // 2
        strategy = "pertp" if world == 2 else f"2d ({n_groups} groups x 2 directions)"
        dirs = (PLUS if rank % 2 == 0 else MINUS,)
    store = DeviceStore(cfg, init_seed=7, device=dev, init="philox", directions=dirs)
    seeds = iteration_seeds(BASE_SEED, args.warmup + args.steps)
    group = rank // 2
    batches = [make_batch(cfg, B * n_groups, DATA_SEED * 1_000_003 + j).shard(n_groups, group)
               for j in range(1, args.warmup + args.steps + 1)]

    if world == 1:
        runner = zo.StreamingZo(store, hyper, overlap=_plan(args))
        wss = [store.workspace(PLUS, B, T), store.workspace(MINUS, B, T)]
        step_calls = {"none": runner.step_calls, "blocks": runner.overlapped_step_calls,
                      "background": runner.background_step_calls,
                      "stacked": runner.stacked_step_calls,
                      "stacked_bg": runner.stacked_bg_step_calls}[args.overlap](wss[0], wss[1])
    else:
        from paper_2507_03211_b200.strategies import TwoDRunner
        runner = TwoDRunner(store, hyper, rank=rank, world=world, batch=B, seq=T)
        wss = runner.ws_list
        step_calls = runner.step_calls()
    ids_dev = torch.stack([torch.from_numpy(b.token_ids.reshape(-1).astype(np.int32)) for b in batches]).to(dev)
    tgt_dev = torch.stack([torch.from_numpy(b.targets.reshape(-1).astype(np.int32)) for b in batches]).to(dev)

    pert_set = {i for i, (fn, _) in enumerate(step_calls) if fn.__name__ == "zo_perturb_update"}
    gemm_idx = [i for i, (fn, _) in enumerate(step_calls) if fn.__name__.startswith("zo_gemm_bf16")]
    streams = {int(torch.cuda.current_stream().cuda_stream): torch.cuda.current_stream()}
    if hasattr(store, "_side"):
        streams[int(store._side.cuda_stream)] = store._side
    n_launch = sum(2 if fn.__name__ == "zo_ce_finalize" else 1 for fn, _ in step_calls if fn.__name__.startswith("zo_"))
    if world > 1:
        n_launch += 0   # collectives are NCCL kernels, not ours

    def gemm_flops(fn, args_):
        if fn.__name__ == "zo_gemm_bf16_split":          # (A, lda, B, B2, ldb, M, N, K, ...)
            return 2.0 * args_[5] * args_[6] * args_[7]
        return 2.0 * args_[4] * args_[5] * args_[6]

    pert_ev, gemm_ev, all_ev = [], [], []   # all_ev: every library call of the instrumented replay
    gemm_shape_ev = []

    def one_step(j, instrument=False):
        for ws in wss:
            ws.ids.copy_(ids_dev[j])
            ws.tgt.copy_(tgt_dev[j])
        store.scal[0:1].fill_(zo._u64_as_i64(seeds[j]))
        store.scal[3:4].fill_(1 if j > 0 else 0)
        if world == 1 and not instrument and not args.no_graph and j > 0:
            runner._replay(wss[0], wss[1])         # the captured step (same launches)
            return
        for i, (fn, a) in enumerate(step_calls):
            timed = instrument and fn.__name__.startswith("zo_")
            if timed:
                st_ = streams.get(int(a[-1]) if a and isinstance(a[-1], int) else -1,
                                  torch.cuda.current_stream())
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st_)
            rc = fn(*a)
            if rc:
                L.check(rc)
            if timed:
                e1.record(st_)
                if i in pert_set:
                    pert_ev.append((j, e0, e1))
                elif i in gemm_set:
                    gemm_ev.append((e0, e1, gemm_flops(fn, a)))
                all_ev.append((fn.__name__, e0, e1))
                if i in gemm_set and fn.__name__ == "zo_gemm_bf16_split":      # per-shape split of the GEMM time
                    gemm_shape_ev.append((f"{a[5]}x{a[6]}x{a[7]}", e0, e1))
        if hasattr(runner, "post_step"):
            runner.post_step()

    gemm_set = set(gemm_idx)
    if world > 1:
        import torch.distributed as dist
    for j in range(args.warmup):
        one_step(j)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st = torch.cuda.Event(enable_timing=True)
    en = torch.cuda.Event(enable_timing=True)
    # uninstrumented timed region (the `value`)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        st.record()
        nvtx = bool(os.environ.get("ZO_NVTX"))      # ncu --nvtx-include zo_step/ selects the timed steps
        for j in range(args.warmup, args.warmup + args.steps):
            if nvtx:
                torch.cuda.nvtx.range_push("zo_step")
            one_step(j)
            if nvtx:
                torch.cuda.nvtx.range_pop()
        en.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = st.elapsed_time(en) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # instrumented pass over the same steps: per-kernel CUDA-event durations.
    # Kernels of concurrent streams would overlap their event windows, so the
    # instrumented replay runs the two directional forwards serialised.
    if world == 1 and args.overlap != "stacked":      # instrument a single-stream plan
        if args.overlap == "stacked_bg":
            runner.overlap = "stacked"
            step_calls[:] = runner.stacked_step_calls(wss[0], wss[1])
        else:
            runner.dual_stream = False
            step_calls[:] = runner.step_calls(wss[0], wss[1])
        pert_set.clear()
        pert_set.update(i for i, (fn, _) in enumerate(step_calls) if fn.__name__ == "zo_perturb_update")
        gemm_set.clear()
        gemm_set.update(i for i, (fn, _) in enumerate(step_calls) if fn.__name__.startswith("zo_gemm_bf16"))
    for j in range(args.warmup, args.warmup + args.steps):
        one_step(j, instrument=True)
    if world == 1:
        runner.dual_stream = True
        runner.overlap = _plan(args) or None
    torch.cuda.synchronize()
    per_step = {}
    for jj, a, b in pert_ev:
        per_step[jj] = per_step.get(jj, 0.0) + a.elapsed_time(b)
    p_ms = list(per_step.values())
    g_tot = sum(a.elapsed_time(b) for a, b, _ in gemm_ev)
    breakdown = {}
    for name, a, b in all_ev:
        breakdown[name] = breakdown.get(name, 0.0) + a.elapsed_time(b) / args.steps
    g_flops = sum(f for _, _, f in gemm_ev)
    gemm_shapes = {}
    for name, a, b in gemm_shape_ev:
        gemm_shapes.setdefault(name, []).append(a.elapsed_time(b) * 1e3)
    gemm_shapes = {k: {"n_per_step": len(v) // args.steps, "median_us": round(statistics.median(v), 1)}
                   for k, v in gemm_shapes.items()}
    rec = store.record.cpu().numpy()

    # e2e through the public API: host batch -> device, record -> host, every step
    e2e_ms = None
    h2d = d2h = 0
    if args.no_e2e:
        e2e_ms = ms
    elif world == 1:
        runner2 = zo.StreamingZo(store, hyper, overlap=_plan(args), graph=not args.no_graph)
        for j in range(args.warmup):
            runner2.step(batches[j], seeds[j])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for j in range(args.warmup, args.warmup + args.steps):
            runner2.step(batches[j], seeds[j])
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        h2d = 2 * M * 4              # ids + targets (int32), shared by both directional workspaces
        d2h = 3 * 8 + 2 * 4          # ZoStep record (f64 x3) + 2 error flags (int32)
    else:
        e2e_ms, h2d, d2h = runner.e2e(batches, seeds, args.warmup, args.steps)

    if rank != 0:
        return
    hbm, tf_sus, tf_burst, peak_kind = _peaks()
    traffic = _traffic() if (args.model, T, B, args.arch) == (MODEL, SEQ, BATCH_PER_GROUP, "zosim") else {}
    P = store.total_params
    bytes_per_param = 12 if world == 1 else 10
    pert_avg = statistics.mean(p_ms)
    pert_gbs = P * bytes_per_param / (pert_avg * 1e-3) / 1e9
    gemm_tfs = g_flops / (g_tot * 1e-3) / 1e12
    tokens = B * n_groups * T
    value = tokens / (ms * 1e-3)
    step_ms_per_rank = ms
    gemm_share = g_tot / args.steps / step_ms_per_rank
    pert_share = pert_avg / step_ms_per_rank
    roof_gemm = {"bound": "tensor", "kernel": "gemm_tcgen05_kernel (all QKV/O/FFN/LM-head launches)",
                 "achieved": gemm_tfs, "peak": tf_sus, "unit": "TFLOP/s", "frac": gemm_tfs / tf_sus,
                 "traffic": traffic.get("gemm_bytes_per_step") if world == 1 else None,
                 "traffic_unit": "DRAM bytes per step, all GEMM launches (ncu)",
                 "peak_kind": f"{peak_kind} sustained bf16", "share_of_step": gemm_share,
                 "algorithmic": "2*M*N*K per launch, M=B*T"}
    roof_pert = {"bound": "hbm", "kernel": "perturb_update_kernel", "achieved": pert_gbs, "peak": hbm,
                 "unit": "GB/s", "frac": pert_gbs / hbm,
                 "traffic": traffic.get("perturb_bytes_per_launch") if world == 1 else None,
                 "traffic_algorithmic": P * bytes_per_param, "peak_kind": f"{peak_kind} HBM copy",
                 "share_of_step": pert_share,
                 "algorithmic": f"{bytes_per_param} B/param x {P} params per step "
                                f"({_plan_text(args, world)})"}
    dominant = roof_gemm if gemm_share >= pert_share else roof_pert
    other = roof_pert if dominant is roof_gemm else roof_gemm
    line = {
        "metric": "OPT ZO fine-tune tokens/s (zosim arch, OPT-1.3B shape)" if args.arch == "zosim"
        else "OPT ZO fine-tune tokens/s (real OPT arch, comparison row)",
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic tokens, random-init (Philox) weights",
        "config": {"workload": f"{args.model} ZO-SGD step ({args.arch} arch), seq {T}, batch {B} per PertP group",
                   "global_batch": B * n_groups, "seq_len": T, "parallelism": strategy, "eps": EPS, "lr": LR,
                   "params": P, "l2": "inputs > L2 (fp32 master 4 B/param + bf16 shadows stream every step)",
                   "perturb_plan": args.overlap,
                   "launch": "eager" if (args.no_graph or world > 1) else "CUDA graph replay per step"},
        "roofline": dominant, "roofline_other": other,
        "perturb_kernel_gbs": pert_gbs,
        "breakdown_ms_per_step": {k: round(v, 4) for k, v in sorted(breakdown.items(), key=lambda kv: -kv[1])},
        "gemm_us_by_shape": gemm_shapes,
        "clocks": clk.summary(),
        "gpu_launches": n_launch * args.steps,
        "e2e": {"value": tokens / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "last_step": {"loss_pos": float(rec[0]), "loss_neg": float(rec[1]), "g": float(rec[2])},
    }
    if world == 1 and not args.no_cpu_baseline and args.arch == "zosim":
        s = cpu_reference_sample(cfg, B)
        line["cpu_baseline"] = {"value": s["tokens_per_s"], "unit": "tokens/s", "cores": s["cores"], "kind": "port",
                                "sample": s["sample"]}
    print(json.dumps(line), flush=True)


def main():
    args = _args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if os.environ.get("ZO_BENCH_SHARE_GPU"):
        local_rank = 0          # test mode: all ranks on one GPU (timings meaningless)
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        backend = os.environ.get("ZO_DIST_BACKEND", "nccl")   # gloo only for single-GPU tests
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        else:
            dist.init_process_group(backend)
    try:
        ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
