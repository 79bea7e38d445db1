#!/usr/bin/env python
"""Benchmark of the B200-native ZO training step (DistZO2 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

Headline workload (BASELINE.json configs[1]): OPT-1.3B-shaped zosim model
(V=50272, d=2048, H=32, 24 blocks, T=512), synthetic tokens, random-init
weights, ZO-SGD with eps=1e-3, lr=1e-7.  Every GPU evaluates
2 x ``--batch`` (default 4) sequences' forwards per step (weak scaling):
  N=1   both directions on one GPU, batch 4 (the lazy MeZO / ZO2 step, Alg. 2)
  N=2   Perturbation Parallelism: rank 0 the +eps forward, rank 1 the -eps
        forward of the same 8 sequences
  N=2k  2D mesh, k groups x 2 directions, 8 sequences per group
One step = fused update(j-1)+perturb(j) pass + forward(s) + loss + g.

Offload leg (configs #4 / #5 at the OPT-13B shape, T=2048, 1 sequence per
group; ``--offload-model`` for 66B / 175B): the fp32 master lives in pinned
host memory and every transformer block streams through the GPU each step.
  N=1   the 1-GPU ZO2 schedule (full-block H2D / D2H, both directions): the
        baseline of the north star's >= 3x target
  N>=2  the 2D mesh + sliced offload: per-rank NUMA-local host slices (1/N of
        every block over each rank's own PCIe link), the direction-aware bf16
        exchange over NVLink, split16 transfer compression
It reports tokens/s, per-rank PCIe / NVLink GB/s and the per-block time
against the reference's T_comm model (comm.py:250-256).

Prints ONE JSON line (rank 0).  `value` is device-timed tokens/s with inputs
resident; `e2e` is the same metric through the public API
(StreamingZo.step / MeshZo.step) with host batches copied in and the step
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
MODEL, SEQ, BATCH = "opt-1.3b", 512, 4
BASE_SEED, DATA_SEED = 1234, 99
NVLINK_GBS = 900.0          # NVLink 5, per direction (spec; no measured figure exists for this box)


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
    ap.add_argument("--batch", type=int, default=BATCH,
                    help="sequences per directional forward (N=1); a 2-rank PertP group runs 2x this")
    ap.add_argument("--plan", default="fill", choices=["stacked", "fill", "none"],
                    help="N=1 step plan: both directions as one launch per layer (stacked), the same with the "
                         "perturb pass filling idle SMs from a low-priority stream (fill), or two streams")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly instead of replaying a CUDA graph")
    ap.add_argument("--no-e2e", action="store_true", help="skip the public-API pass (profiling runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-full", action="store_true", help="skip the one full (unsampled) CPU reference step")
    ap.add_argument("--offload", default="on", choices=["on", "off"])
    ap.add_argument("--offload-timeout", type=float, default=900.0,
                    help="seconds after which a still-running offload leg is reported as an error")
    ap.add_argument("--offload-data-plane", default="collective", choices=["collective", "copy_engine"],
                    help="N>1 offload leg: block slices over NCCL collectives or pulled by the copy engines (CUDA IPC)")
    ap.add_argument("--offload-model", default="opt-13b")
    ap.add_argument("--offload-seq", type=int, default=2048)
    ap.add_argument("--offload-steps", type=int, default=3)
    ap.add_argument("--offload-warmup", type=int, default=1)
    ap.add_argument("--offload-compress", default="auto", choices=["auto", "none", "split16"],
                    help="auto: none for the 1-GPU ZO2 baseline, split16 for the sliced mesh")
    return ap.parse_args()


def _config(args):
    """--model <shape> or <shape>/<n>: n decoder blocks of that shape (per-block
    rates of shapes whose full model does not fit one GPU, e.g. opt-175b/4)."""
    import dataclasses

    from paper_2507_03211_b200.model import opt_config, real_opt_config

    name, _, nb = args.model.partition("/")
    cfg = real_opt_config(name, args.seq) if args.arch == "opt" else opt_config(name, args.seq)
    return dataclasses.replace(cfg, n_blocks=int(nb)).validate() if nb else cfg


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


def _host_info() -> dict:
    info = {"cpu_count": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return info


# ----------------------------------------------------------------------------
# CPU reference (oracle port of zosim): a bounded sample, and one full step
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
    return {"step_s": step, "tokens_per_s": batch * T / step, "cores": cores, "extrapolated": True,
            "fractions": {"params": param_frac / N, "forward_blocks": 1.0 / N, "head_rows": rows_frac},
            "sample": (f"zosim oracle port (numpy, BLAS {cores} threads, z on 1 core): 4 z passes on "
                       f"{param_frac:g} of one transformer block, 2 forwards of 1/{N} blocks at B={batch},T={T}, "
                       f"2 LM-head forwards+CE on {rows_frac:g} of rows; extrapolated to P={P}")}


def cpu_reference_full_step(cfg, batch: int) -> dict:
    """ONE full, unsampled eager step of the reference's algorithm on the
    host, in the reference's own op order (zo.py:136-168): reset, +eps over
    every block (z regenerated block by block from one PCG64 stream),
    forward + loss; reset, -2eps, forward + loss; reset, +eps (restore); g;
    reset, update -- four z passes over all P parameters and two full
    forwards, arithmetic from the oracle restatement.  Weights are drawn
    cheaply (same shapes; the cost does not depend on their values)."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import zo_oracle as O

    cores = os.cpu_count() or 1
    V, d, T, H, N = cfg.vocab_size, cfg.d_model, cfg.seq_len, cfg.n_heads, cfg.n_blocks
    kinds = O.block_kinds(N)
    sizes = [V * d + T * d] + [12 * d * d + 13 * d] * N + [2 * d + d * V + V]      # model.py:60-63
    rng = np.random.default_rng(1)
    blocks = [(0.02 * rng.standard_normal(n, dtype=np.float32)).astype(np.float32) for n in sizes]
    ids = rng.integers(0, V, (batch, T))
    tg = rng.integers(0, V, (batch, T))
    seed = O.iteration_seeds(BASE_SEED, 1)[0]
    with threadpool_limits(limits=cores):
        t0 = time.perf_counter()
        losses = []
        for scale in (+EPS, -EPS):
            gen = np.random.Generator(np.random.PCG64(seed))
            x = ids
            for kind, b in zip(kinds, blocks):
                pert = O.perturbed(b, scale, gen.standard_normal(b.size))
                x = O.block_forward(kind, pert, V, d, T, H, x)
            losses.append(O.cross_entropy(x, tg))
        gen = np.random.Generator(np.random.PCG64(seed))      # +eps closing the cycle: restore (z still drawn)
        for b in blocks:
            gen.standard_normal(b.size)
        g = O.zo_grad(losses[0], losses[1], EPS)
        gen = np.random.Generator(np.random.PCG64(seed))
        blocks = [O.updated(b, g, LR, gen.standard_normal(b.size)) for b in blocks]
        wall = time.perf_counter() - t0
    return {"step_s": wall, "tokens_per_s": batch * T / wall, "cores": cores, "extrapolated": False,
            "sample": f"one full eager step (4 z passes over P={sum(sizes)}, 2 full forwards at B={batch},T={T})"}


def reference_arm(args, rank, world):
    if rank != 0:
        return
    cfg = _config(args)
    batch = args.batch if world == 1 else 2 * args.batch * (world // 2)
    for _ in range(args.warmup):
        cpu_reference_sample(cfg, batch, rows_frac=0.03125, param_frac=0.0625)
    samples, walls = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        samples.append(cpu_reference_sample(cfg, batch, rows_frac=0.03125, param_frac=0.0625))
        walls.append(time.perf_counter() - t0)
    vals = [s["tokens_per_s"] for s in samples]
    v = statistics.median(vals)
    # each timed "step" is the bounded sample; ms_per_step is its measured wall time (so steps x
    # ms_per_step is the run's real duration), the full step it extrapolates to is reported beside it
    ms = 1e3 * statistics.median(walls)
    full_s = statistics.median([s["step_s"] for s in samples])
    line = {"metric": f"OPT ZO fine-tune tokens/s (zosim arch, {args.model} shape)", "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference", "extrapolated": True,
            "extrapolated_step_s": full_s,
            "step_definition": "one bounded sample of the CPU reference step (fractions in cpu_baseline); value = "
                               "the full step's tokens/s extrapolated from it",
            "config": {"workload": f"{args.model} ZO-SGD step, seq {args.seq}, global batch {batch}",
                       "global_batch": batch, "seq_len": args.seq, "strategy": "mezo (CPU reference)"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": samples[0]["cores"], "kind": "port",
                             "extrapolated": True, "fractions": samples[0]["fractions"],
                             "sample": samples[0]["sample"], "host": _host_info()},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# our arm: the resident headline step
# ----------------------------------------------------------------------------
MIX_CEILING_GBS = 5652.0   # read 4 B + write 4 + 2 + 2 B per element, no arithmetic (profiles/r02/mix_probe/)


def _kernel_kind(name: str) -> str:
    if name.startswith("zo_gemm"):
        return "gemm"
    return {"zo_perturb_update": "perturb", "zo_attn_causal_fwd": "attention",
            "zo_layernorm_fwd": "layernorm", "zo_layernorm_fwd_split": "layernorm"}.get(name, "other")


def ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2507_03211_b200 import _lib as L
    from paper_2507_03211_b200 import zo
    from paper_2507_03211_b200.engine import MINUS, PLUS, DeviceStore
    from paper_2507_03211_b200.model import make_batch
    from paper_2507_03211_b200.rng import iteration_seeds

    torch.cuda.set_device(local_rank)
    dev = torch.device(f"cuda:{local_rank}")
    cfg = _config(args)
    T = args.seq
    hyper = zo.ZoHyper(EPS, LR)
    if world == 1:
        strategy, n_groups, dirs, B = "mezo-lazy (both directions, 1 GPU)", 1, (PLUS, MINUS), args.batch
    else:
        if world % 2:
            raise SystemExit("world size must be 1 or even (PertP pairs)")
        n_groups = world // 2
        strategy = "pertp" if world == 2 else f"2d ({n_groups} groups x 2 directions)"
        dirs = (PLUS if rank % 2 == 0 else MINUS,)
        B = 2 * args.batch             # one direction per rank: the same forward rows per GPU as N=1
    M = B * T
    store = DeviceStore(cfg, init_seed=7, device=dev, init="philox", directions=dirs)
    seeds = iteration_seeds(BASE_SEED, args.warmup + args.steps)
    group = rank // 2
    batches = [make_batch(cfg, B * n_groups, DATA_SEED * 1_000_003 + j).shard(n_groups, group)
               for j in range(1, args.warmup + args.steps + 1)]

    if world == 1:
        runner = zo.StreamingZo(store, hyper, overlap=args.plan if args.plan in ("stacked", "fill") else False,
                                graph=not args.no_graph)
        wss = [store.workspace(PLUS, B, T), store.workspace(MINUS, B, T)]
        step_calls = runner._plan(wss[0], wss[1])
    else:
        from paper_2507_03211_b200.fabric import TorchFabric
        from paper_2507_03211_b200.strategies import MeshZo

        fabric = TorchFabric()
        runner = MeshZo(store, hyper, fabric, "2d", B, T, graph=not args.no_graph)
        wss = list(runner.ws.values())
        step_calls = runner.step_calls()
    ids_dev = torch.stack([torch.from_numpy(b.token_ids.reshape(-1).astype(np.int32)) for b in batches]).to(dev)
    tgt_dev = torch.stack([torch.from_numpy(b.targets.reshape(-1).astype(np.int32)) for b in batches]).to(dev)
    n_launch = sum(2 if fn.__name__ == "zo_ce_finalize" else 1 for fn, _ in step_calls if fn.__name__.startswith("zo_"))
    streams = {int(torch.cuda.current_stream().cuda_stream): torch.cuda.current_stream()}
    for st_ in store.plan_streams():
        streams[int(st_.cuda_stream)] = st_

    use_graph = not args.no_graph and (world == 1 or runner.graph)     # (a gloo mesh cannot be captured)

    def one_step(j, instrument=None):
        for ws in wss:
            ws.ids.copy_(ids_dev[j])
            ws.tgt.copy_(tgt_dev[j])
        store.scal[0:1].fill_(zo._u64_as_i64(seeds[j]))
        store.scal[3:4].fill_(1 if j > 0 else 0)
        if instrument is None and use_graph and j > 0:
            if world == 1:
                runner._replay(wss[0], wss[1])        # the captured step (same launches)
            else:
                runner.replay()
            return
        for fn, a in step_calls:
            timed = instrument is not None and fn.__name__.startswith("zo_")
            if timed:
                st_ = streams.get(int(a[-1]) if a and isinstance(a[-1], int) else -1, torch.cuda.current_stream())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st_)
            rc = fn(*a)
            if rc:
                L.check(rc)
            if timed:
                e1.record(st_)
                instrument.append((fn.__name__, a, e0, e1))

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

    # instrumented eager replay of the same steps on ONE stream (event windows
    # never overlap): per-kernel CUDA-event durations for the roofline rows
    if world == 1 and args.plan != "stacked":
        runner.dual_stream = False
        if args.plan == "fill":
            runner.overlap = "stacked"          # per-kernel windows: the same launches, serialised
        step_calls = runner._plan(wss[0], wss[1])
    events = []
    for j in range(args.warmup, args.warmup + args.steps):
        one_step(j, instrument=events)
    runner.dual_stream = True
    torch.cuda.synchronize()
    rec = store.record.cpu().numpy()
    by_kind, breakdown, gemm_shapes = {}, {}, {}
    for name, a, e0, e1 in events:
        t_ms = e0.elapsed_time(e1)
        breakdown[name] = breakdown.get(name, 0.0) + t_ms / args.steps
        k = _kernel_kind(name)
        d = by_kind.setdefault(k, {"ms": 0.0, "work": 0.0})
        d["ms"] += t_ms
        if name == "zo_gemm_bf16_split":            # (A, lda, B, B2, ldb, M, N, K, ...)
            d["work"] += 2.0 * a[5] * a[6] * a[7]
            gemm_shapes.setdefault(f"{a[5]}x{a[6]}x{a[7]}", []).append(t_ms * 1e3)
        elif name == "zo_gemm_bf16":                # (A, lda, B, ldb, M, N, K, ...)
            d["work"] += 2.0 * a[4] * a[5] * a[6]
            gemm_shapes.setdefault(f"{a[4]}x{a[5]}x{a[6]}", []).append(t_ms * 1e3)
        elif k == "attention":                      # (qkv, ldq, B, T, H, hd, ...): causal 2*B*T^2*d
            d["work"] += 2.0 * a[2] * a[3] * a[3] * a[4] * a[5]
        elif name == "zo_layernorm_fwd_split":      # (x, ldx, g, b, g2, b2, rows, split, d, ...): 4 B in + 2 B out
            d["work"] += 6.0 * a[6] * a[8]
        elif name == "zo_layernorm_fwd":            # (x, ldx, g, b, rows, d, ...)
            d["work"] += 6.0 * a[4] * a[5]
    gemm_shapes = {k: {"n_per_step": len(v) // args.steps, "median_us": round(statistics.median(v), 1)}
                   for k, v in gemm_shapes.items()}

    # e2e through the public API: host batch -> device, record -> host, every step
    e2e_ms, h2d, d2h = ms, 0, 0
    api = None
    if not args.no_e2e:
        if world == 1:
            api = zo.StreamingZo(store, hyper, overlap=args.plan if args.plan in ("stacked", "fill") else False,
                                 graph=not args.no_graph)
        else:
            api = MeshZo(store, hyper, fabric, "2d", B, T, graph=not args.no_graph)
        for j in range(args.warmup):
            api.step(batches[j], seeds[j])
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for j in range(args.warmup, args.warmup + args.steps):
            api.step(batches[j], seeds[j])
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        h2d = 2 * M * 4 + (16 if world == 1 else 0)   # ids + targets (int32, shared by the workspaces) + seed / pending
        d2h = 3 * 8 + len(wss) * 4           # ZoStep record (f64 x3) + error flags (int32)
    P = store.total_params
    pert_bytes = store.perturb_bytes(dirs)
    api = None
    del runner, store, wss, api
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    if rank != 0:
        if args.offload == "on":
            _guarded_offload(args, rank, world, local_rank, None)
        return
    hbm, tf_sus, tf_burst, peak_kind = _peaks()
    headline = (args.model, T, args.batch, args.arch, world) == (MODEL, SEQ, BATCH, "zosim", 1)
    traffic = _traffic() if headline else {}
    tokens = B * n_groups * T
    value = tokens / (ms * 1e-3)

    def roof(kind, bound, unit, peak, work_unit, algorithmic, kernel, traffic_v=None):
        d = by_kind.get(kind, {"ms": 0.0, "work": 0.0})
        if not d["ms"]:
            return None
        ach = d["work"] / (d["ms"] * 1e-3) / work_unit
        return {"bound": bound, "kernel": kernel, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                "traffic": traffic_v, "share_of_step": d["ms"] / args.steps / ms, "algorithmic": algorithmic}

    r_gemm = roof("gemm", "tensor", "TFLOP/s", tf_sus, 1e12, "2*M*N*K per launch, M = rows of the launch",
                  "gemm_tcgen05_pair_kernel (all QKV / O / FFN / LM-head launches)",
                  traffic.get("gemm_bytes_per_step"))
    if r_gemm:
        r_gemm["traffic_unit"] = "DRAM bytes per step, all GEMM launches (ncu)"
        r_gemm["peak_kind"] = f"{peak_kind} sustained bf16"
    d = by_kind["perturb"]
    pert_ms = d["ms"] / args.steps
    r_pert = {"bound": "hbm", "kernel": "perturb_update_kernel", "achieved": pert_bytes / (pert_ms * 1e-3) / 1e9,
              "peak": hbm, "unit": "GB/s", "frac": pert_bytes / (pert_ms * 1e-3) / 1e9 / hbm,
              "traffic": traffic.get("perturb_bytes_per_step", traffic.get("perturb_bytes_per_launch")),
              "traffic_algorithmic": pert_bytes,
              "peak_kind": f"{peak_kind} HBM copy", "share_of_step": pert_ms / ms,
              # the pure-memory ceiling of this exact R4/W4/W2/W2 mix, measured on this pool's B200s
              # (tools/mix_probe.cu, profiles/r02/mix_probe/): the pass's own bandwidth roof
              "mix_ceiling_gbs": MIX_CEILING_GBS,
              "frac_of_mix_ceiling": pert_bytes / (pert_ms * 1e-3) / 1e9 / MIX_CEILING_GBS,
              "algorithmic": (f"R+W fp32 master (8 B) + the bf16 / fp32 shadows this rank writes, per parameter "
                              f"(embedding: no shadow, 8 B): {pert_bytes} B over {P} params, one launch per step")}
    r_attn = roof("attention", "tensor", "TFLOP/s", tf_sus, 1e12, "2*B*T^2*d per launch (causal halves of QK^T, PV)",
                  "attn_pp_kernel (tcgen05, hd 64; attn_tc_kernel<128> at hd 128)")
    r_ln = roof("layernorm", "hbm", "GB/s", hbm, 1e9, "4 B read + 2 B write per element", "layernorm_warp_kernel")
    dominant = max([r for r in (r_gemm, r_pert) if r], key=lambda r: r["share_of_step"])
    line = {
        "metric": f"OPT ZO fine-tune tokens/s ({args.arch} arch, {args.model} shape)",
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic tokens, random-init (Philox) weights",
        "config": {"workload": f"{args.model} ZO-SGD step ({args.arch} arch), seq {T}, {B} sequences per "
                               f"directional forward per GPU", "global_batch": B * n_groups, "seq_len": T,
                   "parallelism": strategy, "eps": EPS, "lr": LR, "params": P,
                   "l2": "inputs > L2 (fp32 master 4 B/param + bf16 shadows stream every step)",
                   "plan": args.plan if world == 1 else "mesh (one direction per rank)",
                   "launch": "CUDA graph replay per step" if use_graph else "eager"},
        "roofline": dominant,
        "roofline_other": {"perturb": r_pert, "gemm": r_gemm, "attention": r_attn, "layernorm": r_ln},
        "perturb_kernel_gbs": r_pert["achieved"],
        "breakdown_ms_per_step": {k: round(v, 4) for k, v in sorted(breakdown.items(), key=lambda kv: -kv[1])},
        "gemm_us_by_shape": gemm_shapes,
        "clocks": clk.summary(),
        "gpu_launches": n_launch * args.steps,
        "e2e": {"value": tokens / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "last_step": {"loss_pos": float(rec[0]), "loss_neg": float(rec[1]), "g": float(rec[2])},
    }
    if args.offload == "on":
        line["offload"] = _guarded_offload(args, rank, world, local_rank, line)
    if world == 1 and not args.no_cpu_baseline and args.arch == "zosim":
        s = cpu_reference_sample(cfg, B)
        line["cpu_baseline"] = {"value": s["tokens_per_s"], "unit": "tokens/s", "cores": s["cores"], "kind": "port",
                                "extrapolated": True, "fractions": s["fractions"], "sample": s["sample"],
                                "host": _host_info()}
        if not args.no_cpu_full:
            f = cpu_reference_full_step(cfg, B)
            line["cpu_baseline"]["full_step"] = {"value": f["tokens_per_s"], "unit": "tokens/s",
                                                 "step_s": f["step_s"], "cores": f["cores"],
                                                 "extrapolated": False, "sample": f["sample"]}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# our arm: the offload leg (configs #4 / #5 at a shape every box can hold)
# ----------------------------------------------------------------------------
def _guarded_offload(args, rank, world, local_rank, line) -> dict:
    """The offload leg must not cost the headline line: an exception becomes
    {"error": ...}, and a leg still running after --offload-timeout seconds
    (e.g. a collective that never completes) makes rank 0 print the line with
    {"error": "timeout"} and every rank exit."""
    import threading

    def expire():
        if line is not None:
            line["offload"] = {"error": f"offload leg did not finish within {args.offload_timeout} s"}
            print(json.dumps(line), flush=True)
        os._exit(0)

    t = threading.Timer(args.offload_timeout, expire)
    t.daemon = True
    t.start()
    try:
        return offload_leg(args, rank, world, local_rank)
    except Exception as e:                       # noqa: BLE001 (reported in the line)
        return {"error": f"{type(e).__name__}: {e}"[:400]}
    finally:
        t.cancel()


def offload_leg(args, rank, world, local_rank) -> dict | None:
    affinity = os.sched_getaffinity(0)          # the NUMA binding below is undone on return
    try:
        return _offload_leg(args, rank, world, local_rank)
    finally:
        os.sched_setaffinity(0, affinity)


def _offload_leg(args, rank, world, local_rank) -> dict | None:
    import torch

    from paper_2507_03211_b200.model import make_batch, opt_config
    from paper_2507_03211_b200.rng import iteration_seeds
    from paper_2507_03211_b200.scheduler import HostStore, OffloadedZo
    from paper_2507_03211_b200.zo import ZoHyper

    dev = torch.device(f"cuda:{local_rank}")
    cfg = opt_config(args.offload_model, args.offload_seq)
    T = args.offload_seq
    hyper = ZoHyper(EPS, LR)
    steps, warm = args.offload_steps, args.offload_warmup
    seeds = iteration_seeds(BASE_SEED, warm + steps)
    t_setup = time.perf_counter()
    if world == 1:
        compress = "none" if args.offload_compress == "auto" else args.offload_compress
        host = HostStore(cfg, init_seed=7, init="philox", device=dev, numa=True)
        rt = OffloadedZo(host, hyper, batch=1, device=dev, trace=True, compress=compress)
        schedule = ("ZO2 on 1 GPU: every transformer block's full fp32 master H2D and back D2H per step, both "
                    "directions on the GPU (scheduler.py:285-322)" + (", split16" if compress == "split16" else ""))
        n_groups, group, numa = 1, 0, host.numa
    else:
        from paper_2507_03211_b200.fabric import TorchFabric
        from paper_2507_03211_b200.sharded import ShardStore

        compress = "split16" if args.offload_compress == "auto" else args.offload_compress
        fabric = TorchFabric(data_plane=args.offload_data_plane)
        host = ShardStore(cfg, fabric, init_seed=7, init="philox", device=dev, where="host")
        rt = OffloadedZo(host, hyper, batch=1, device=dev, fabric=fabric, strategy="2d", redistribute="bf16",
                         compress=compress, trace=True)
        schedule = (f"2D mesh ({world // 2} groups x 2 directions) + sliced offload: per-rank NUMA-local pinned "
                    f"slices (1/{world} of every block over each rank's PCIe link, comm.py:314-342), "
                    f"direction-aware bf16 exchange over NVLink ({args.offload_data_plane} data plane), "
                    f"compress={compress}")
        n_groups, group, numa = world // 2, rank // 2, host.numa
    t_setup = time.perf_counter() - t_setup
    batches = [make_batch(cfg, n_groups, DATA_SEED * 1_000_003 + j).shard(n_groups, group)
               for j in range(1, warm + steps + 1)]
    for j in range(warm):
        rt.step(batches[j], seeds[j])
    rt.phase_stats.clear()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for j in range(warm, warm + steps):
        rt.step(batches[j], seeds[j])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    stats = {k: dict(v) for k, v in rt.phase_stats.items()}
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    nb = len(rt.wids)
    P_blk = cfg.d_model * cfg.d_model * 12 + 13 * cfg.d_model

    def gbs(k):
        s = stats.get(k)
        return None if not s or not s["ms"] else s["bytes"] / (s["ms"] * 1e-3) / 1e9

    def per_block(k):
        s = stats.get(k)
        return None if not s or not s["n"] else s["ms"] / s["n"]

    h2d_gbs, nvl = gbs("h2d"), gbs("nvlink_exchange") or gbs("nvlink_allgather")
    b_pcie = 2 if compress == "split16" else 4
    b_nvl = 2 if world > 1 else 4
    # the reference's model (comm.py:250-256) at the measured PCIe rate and the NVLink spec
    t_model = None
    if h2d_gbs:
        w = -(-P_blk // world)
        t_model = 1e3 * (w * b_pcie / (h2d_gbs * 1e9) + (P_blk - w) * b_nvl / (NVLINK_GBS * 1e9))
    measured_block = (per_block("h2d") or 0.0) + (per_block("nvlink_exchange") or per_block("nvlink_allgather") or 0.0)
    rt.flush()
    out = {
        "workload": f"{args.offload_model} (zosim arch) ZO-SGD step, seq {T}, 1 sequence per PertP group, fp32 master "
                    f"in pinned host memory, all {nb} transformer blocks streamed every step",
        "schedule": schedule, "n_gpus": world, "global_batch": n_groups, "seq_len": T,
        "tokens_per_s": n_groups * T / (ms * 1e-3), "ms_per_step": ms, "steps": steps, "warmup": warm,
        "setup_s": t_setup, "compress": compress,
        "pcie_bytes_per_step_per_rank": {"h2d": rt.pcie_bytes_per_step()[0], "d2h": rt.pcie_bytes_per_step()[1]},
        "h2d_gbs_per_rank": h2d_gbs, "d2h_gbs_per_rank": gbs("d2h"),
        "nvlink_rx_gbs_per_rank": nvl, "nvlink_peak_gbs": NVLINK_GBS,
        "nvlink_frac": (nvl / NVLINK_GBS) if nvl else None,
        "per_block_ms": {k: per_block(k) for k in ("h2d", "nvlink_exchange", "nvlink_allgather", "compute", "d2h")
                         if per_block(k) is not None},
        "per_block_upload_ms": measured_block, "t_comm_model_ms": t_model,
        "t_comm_model": "ceil(M/N)*b_pcie/BW_pcie(measured h2d) + (M-ceil(M/N))*b_nvl/900 GB/s (comm.py:250-256)",
        "numa": numa,
    }
    del rt, host
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


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
