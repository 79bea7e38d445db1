"""Training-run driver and its artefacts: the reference's ``RunConfig`` /
``run`` / ``write_outputs`` (src/zosim/bench.py:53-207, 337-346) over the
B200 runtime.

``run(config)`` trains ``hyper.steps`` iterations under one strategy and
returns a ``RunReport`` with the reference's fields; with ``report_dir`` set
it writes ``report.json``, ``steps.jsonl`` and ``timeline.json`` in the
reference's format (bench.py:337-346).

  mezo   eager Alg. 1 on one GPU (zo.mezo_step)
  zo2    Alg. 2/3 with the fp32 master in pinned host memory
         (scheduler.OffloadedZo); the timeline is the last step's CUDA-event
         upload / compute / offload intervals (milliseconds from step start)
  pertp / ddp / 2d
         one process per GPU under torch.distributed (``torchrun``);
         ``mesh.workers`` must equal the world size; rank 0 reports

Differences from the reference, all measurement-side: step walls are real
seconds of the GPU step (each step ends with the ZoStep read-back, which
synchronises), ``peak_device_bytes`` is torch's allocator high-water mark on
the device, and ``comm_bytes`` counts real host<->device and fabric bytes.
"""

from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError
from .model import Batch, ModelConfig, make_batch
from .rng import RngStateManager, iteration_seeds

STRATEGIES = ("mezo", "zo2", "pertp", "ddp", "2d")     # bench.py:33
ORDERINGS = ("pertp_inner", "ddp_inner")


@dataclass(frozen=True)
class MeshConfig:
    """bench.py:37-49."""

    workers: int = 1
    n_b: int = 1
    n_p: int = 2
    ordering: str = "pertp_inner"

    @classmethod
    def from_dict(cls, d: dict) -> "MeshConfig":
        try:
            return cls(**d)
        except TypeError as e:
            raise ConfigurationError(f"bad mesh config: {e}") from e


@dataclass
class RunConfig:
    """bench.py:55-150 minus the simulator's topology / compute_time knobs
    (real hardware replaces the cost model).  ``device_capacity_blocks`` keeps
    the reference's meaning of a device capacity in block footprints, used as
    the zo2 runtime's HBM budget: what fits stays resident, the rest streams."""

    model: ModelConfig
    hyper: object                  # zo.ZoHyper
    strategy: str = "mezo"
    mesh: MeshConfig = field(default_factory=MeshConfig)
    batch_size: int = 4
    seed: int = 1234
    init_seed: int = 7
    data_seed: int = 99
    init: str = "host"             # "host" (zosim's numpy draws) or "philox" (random-init at scale)
    device_capacity_blocks: float | None = None   # zo2: HBM budget in transformer-block footprints
    offload_compress: str = "none"                 # zo2: "split16" = hi plane over PCIe, lo plane in HBM
    report_dir: str | None = None

    def validate(self) -> "RunConfig":
        """bench.py:69-103: the same checks and messages."""
        self.model.validate()
        self.hyper.validate()
        if self.strategy not in STRATEGIES:
            raise ConfigurationError(f"strategy must be one of {STRATEGIES}, got {self.strategy!r}")
        if self.mesh.ordering not in ORDERINGS:
            raise ConfigurationError(f"ordering must be one of {ORDERINGS}")
        k = self.mesh.workers
        if self.strategy in ("mezo", "zo2") and k != 1:
            raise ConfigurationError(f"strategy {self.strategy} runs on 1 worker, mesh has {k}")
        if self.strategy == "pertp" and k != 2:
            raise ConfigurationError(f"pertp needs exactly 2 workers, mesh has {k}")
        if self.strategy == "ddp":
            if k < 1:
                raise ConfigurationError("ddp needs at least 1 worker")
            if self.batch_size % k != 0:
                raise ConfigurationError(f"batch_size {self.batch_size} not divisible by {k} workers")
        if self.strategy == "2d":
            if self.mesh.n_p != 2:
                raise ConfigurationError(f"the mesh's direction dimension is fixed at 2, got {self.mesh.n_p}")
            if k != self.mesh.n_b * 2:
                raise ConfigurationError(f"2d mesh needs workers = n_b x 2 = {self.mesh.n_b * 2}, got {k}")
            if self.batch_size % self.mesh.n_b != 0:
                raise ConfigurationError(f"batch_size {self.batch_size} not divisible by {self.mesh.n_b} groups")
        if self.batch_size < 1:
            raise ConfigurationError("batch_size must be >= 1")
        if self.init not in ("host", "philox"):
            raise ConfigurationError(f"init must be 'host' or 'philox', got {self.init!r}")
        if self.offload_compress not in ("none", "split16"):
            raise ConfigurationError(f"offload_compress must be 'none' or 'split16', got {self.offload_compress!r}")
        return self

    @classmethod
    def from_dict(cls, d: dict) -> "RunConfig":
        from .zo import ZoHyper

        d = dict(d)
        for k in ("topology", "compute_time"):   # simulator-only knobs
            d.pop(k, None)
        try:
            cfg = cls(model=ModelConfig.from_dict(d.pop("model")), hyper=ZoHyper(**d.pop("hyper")),
                      mesh=MeshConfig.from_dict(d.pop("mesh", {})), **d)
        except TypeError as e:
            raise ConfigurationError(f"bad run config: {e}") from e
        return cfg.validate()

    @classmethod
    def from_file(cls, path, overrides: dict | None = None) -> "RunConfig":
        try:
            with open(path) as f:
                d = json.load(f)
        except OSError as e:
            raise ConfigurationError(f"cannot read config {path}: {e}") from e
        except json.JSONDecodeError as e:
            raise ConfigurationError(f"config {path} is not valid JSON: {e}") from e
        return cls.from_dict(_merge(d, overrides or {}))

    def to_dict(self) -> dict:
        return {
            "model": self.model.to_dict(),
            "hyper": {"epsilon": self.hyper.epsilon, "lr": self.hyper.lr, "steps": self.hyper.steps},
            "strategy": self.strategy,
            "mesh": {"workers": self.mesh.workers, "n_b": self.mesh.n_b, "n_p": self.mesh.n_p,
                     "ordering": self.mesh.ordering},
            "batch_size": self.batch_size,
            "seed": self.seed,
            "init_seed": self.init_seed,
            "data_seed": self.data_seed,
            "init": self.init,
            "device_capacity_blocks": self.device_capacity_blocks,
            "offload_compress": self.offload_compress,
        }


def _merge(base: dict, overrides: dict) -> dict:
    out = dict(base)
    for key, val in overrides.items():
        if isinstance(val, dict) and isinstance(out.get(key), dict):
            out[key] = _merge(out[key], val)
        else:
            out[key] = val
    return out


@dataclass
class RunReport:
    """bench.py:167-191."""

    strategy: str
    workers: int
    steps: list
    tokens_per_sec: float
    tokens_per_sec_total: float
    wall_time: float
    peak_device_bytes: int
    peak_by_tag: dict
    comm_bytes: dict
    timeline: list
    final_checksum: str

    def to_dict(self) -> dict:
        return {
            "strategy": self.strategy,
            "workers": self.workers,
            "tokens_per_sec": self.tokens_per_sec,
            "tokens_per_sec_total": self.tokens_per_sec_total,
            "wall_time": self.wall_time,
            "peak_device_bytes": self.peak_device_bytes,
            "peak_by_tag": self.peak_by_tag,
            "comm_bytes": self.comm_bytes,
            "final_checksum": self.final_checksum,
            "steps": len(self.steps),
        }


def throughput(step_walls: list, tokens_per_step: int) -> float:
    """bench.py:194-197: median step wall with the first 2 steps dropped
    (when more than 3 were run)."""
    walls = step_walls[2:] if len(step_walls) > 3 else step_walls
    med = float(np.median(walls))
    return tokens_per_step / med if med > 0 else float("inf")


def batch_for(config: RunConfig, iteration: int) -> Batch:
    """bench.py:199-200."""
    return make_batch(config.model, config.batch_size, config.data_seed * 1_000_003 + iteration)


def run(config: RunConfig) -> RunReport:
    """bench.py:203-227."""
    config.validate()
    runner = {"mezo": _run_mezo, "zo2": _run_zo2, "pertp": _run_mesh, "ddp": _run_mesh, "2d": _run_mesh}
    t0 = time.perf_counter()
    report = runner[config.strategy](config)
    report.wall_time = time.perf_counter() - t0
    if config.report_dir and _is_rank0():
        write_outputs(report, config)
    return report


def _is_rank0() -> bool:
    import torch.distributed as dist

    return not dist.is_initialized() or dist.get_rank() == 0


def _device():
    import torch

    return torch.device("cuda", torch.cuda.current_device())


def _tokens_per_step(config: RunConfig) -> int:
    return config.batch_size * config.model.seq_len


def _run_mezo(config: RunConfig) -> RunReport:
    import torch

    from .engine import DeviceStore
    from .zo import mezo_step

    dev = _device()
    torch.cuda.reset_peak_memory_stats(dev)
    store = DeviceStore(config.model, init_seed=config.init_seed, device=dev, init=config.init)
    mgr = RngStateManager()
    steps, walls = [], []
    for j, seed in enumerate(iteration_seeds(config.seed, config.hyper.steps), 1):
        batch = batch_for(config, j)
        t = time.perf_counter()
        steps.append(mezo_step(store, batch, config.hyper, seed, mgr, iteration=j))
        walls.append(time.perf_counter() - t)
    tps = _tokens_per_step(config)
    peak = int(torch.cuda.max_memory_allocated(dev))
    return RunReport("mezo", 1, steps, throughput(walls, tps), tps * len(steps) / sum(walls), sum(walls),
                     peak, {"device": peak}, {}, [], store.checksum())


def _run_zo2(config: RunConfig) -> RunReport:
    import torch

    from .scheduler import HostStore, OffloadedZo

    dev = _device()
    torch.cuda.reset_peak_memory_stats(dev)
    host = HostStore(config.model, init_seed=config.init_seed, init=config.init, device=dev)
    k, slots = 0, 3
    if config.device_capacity_blocks is not None:
        # the reference's capacity knob (bench.py:262-264) as a real HBM budget:
        # keep what fits resident, stream the rest (scheduler.plan_residency)
        from .model import model_layout
        from .scheduler import plan_residency

        per = [bl for bl in model_layout(config.model) if bl.kind == "transformer"][0].elem_count * 8
        k, slots = plan_residency(config.model, int(config.device_capacity_blocks * per),
                                  compress=config.offload_compress)
        slots = max(slots, 2)
    rt = OffloadedZo(host, config.hyper, config.batch_size, device=dev, trace=True, resident_blocks=k,
                     n_slots=slots, compress=config.offload_compress)
    steps, walls = [], []
    for j, seed in enumerate(iteration_seeds(config.seed, config.hyper.steps), 1):
        batch = batch_for(config, j)
        t = time.perf_counter()
        steps.append(rt.step(batch, seed))
        walls.append(time.perf_counter() - t)
    rt.flush()
    bpp = 2 if config.offload_compress == "split16" else 4      # PCIe bytes per streamed parameter
    comm = {"host_upload_bytes": rt.uploaded_params * bpp, "host_offload_bytes": rt.offloaded_params * bpp}
    tps = _tokens_per_step(config)
    peak = int(torch.cuda.max_memory_allocated(dev))
    return RunReport("zo2", 1, steps, throughput(walls, tps), tps * len(steps) / sum(walls), sum(walls),
                     peak, {"device": peak}, comm, rt.last_timeline, host.checksum())


def _run_mesh(config: RunConfig) -> RunReport:
    """pertp / ddp / 2d: this process is one rank (bench.py:292-334 runs the
    ranks as threads; here they are torchrun processes, one per GPU)."""
    import torch
    import torch.distributed as dist

    from .engine import MINUS, PLUS, DeviceStore
    from .fabric import TorchFabric
    from .strategies import MeshLayout, MeshZo

    if not dist.is_initialized():
        raise ConfigurationError(f"strategy {config.strategy} needs torch.distributed (launch with torchrun)")
    fabric = TorchFabric()
    k = config.mesh.workers
    if fabric.k != k:
        raise ConfigurationError(f"mesh has {k} workers, world size is {fabric.k}")
    strategy = config.strategy
    if strategy == "2d" and config.mesh.ordering != "pertp_inner":
        raise ConfigurationError("the GPU mesh runs the pertp_inner ordering (ddp_inner is numerically identical)")
    mesh = MeshLayout(strategy, k, fabric.rank)
    n_shards = {"pertp": 1, "ddp": k, "2d": config.mesh.n_b}[strategy]
    shard_of = {"pertp": 0, "ddp": fabric.rank, "2d": mesh.group}[strategy]
    dev = _device()
    torch.cuda.reset_peak_memory_stats(dev)
    dirs = (PLUS, MINUS) if strategy == "ddp" else mesh.dirs
    store = DeviceStore(config.model, init_seed=config.init_seed, device=dev, init=config.init, directions=dirs)
    B = config.batch_size // n_shards
    mz = MeshZo(store, config.hyper, fabric, strategy, B, config.model.seq_len)
    steps, walls = [], []
    for j, seed in enumerate(iteration_seeds(config.seed, config.hyper.steps), 1):
        batch = batch_for(config, j).shard(n_shards, shard_of)
        t = time.perf_counter()
        steps.append(mz.step(batch, seed))
        walls.append(time.perf_counter() - t)
    mz.flush()
    tps = _tokens_per_step(config)
    peak = int(torch.cuda.max_memory_allocated(dev))
    checksum = store.checksum()
    return RunReport(strategy, k, steps, throughput(walls, tps), tps * len(steps) / sum(walls), sum(walls),
                     peak, {"block": peak}, dict(fabric.bytes_by_tag), [], checksum)


def write_outputs(report: RunReport, config: RunConfig) -> None:
    """bench.py:337-346."""
    out = config.report_dir
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "report.json"), "w") as f:
        json.dump({"config": config.to_dict(), **report.to_dict()}, f, indent=1)
    with open(os.path.join(out, "steps.jsonl"), "w") as f:
        for s in report.steps:
            f.write(s.to_json() + "\n")
    with open(os.path.join(out, "timeline.json"), "w") as f:
        json.dump(report.timeline, f, indent=1)
