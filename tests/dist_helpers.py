"""Worker functions for multi-process tests (spawned; must be importable)."""

import os
import socket


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def init(rank, world, port, backend="gloo"):
    import datetime

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))


def fabric_worker(rank, world, port, q):
    """CPU: ordered collectives + the mesh-gather layout."""
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.strategies import MeshLayout

    init(rank, world, port)
    fab = TorchFabric()
    out = {}
    out["gather"] = fab.all_gather(rank, 10.0 + rank, tag="loss")
    out["bcast"] = fab.broadcast(rank, 42 if rank == 0 else None, tag="seed")
    vals = [0.1, 0.2, 0.3, 1e16, -1e16, 0.7, 0.9, 1.1][:world]
    out["mean"] = fab.all_reduce_mean(rank, vals[rank], tag="grad")
    # device-gather layout: each rank fills its own slot(s) of [L+, L-]
    for strat in (["ddp", "2d"] + (["pertp"] if world == 2 else [])):
        mesh = MeshLayout(strat, world, rank)
        local = torch.zeros(2, dtype=torch.float64)
        lp, ln = 2.0 + 0.01 * (rank // (1 if strat == "ddp" else 2)), 2.0 - 0.013 * (rank // (1 if strat == "ddp" else 2))
        if 0 in mesh.dirs:
            local[0] = lp
        if 1 in mesh.dirs:
            local[1] = ln
        gathered = torch.zeros(2 * world, dtype=torch.float64)
        fab.all_gather_tensor(gathered, local, tag="loss")
        out[strat] = mesh.grad_host(gathered.tolist(), 1e-3)
    out["bytes"] = dict(fab.bytes_by_tag)
    dist.destroy_process_group()
    q.put((rank, out))


def exchange_worker(rank, world, port, width, q):
    """CPU: the direction-aware slice exchange -- rank q ends up with slice k
    of direction dir_of[q] from every rank k (gloo path)."""
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200.fabric import TorchFabric

    init(rank, world, port)
    fab = TorchFabric()
    dir_of = [q % 2 for q in range(world)]
    bufs = {d: torch.full((world * width,), float("nan"), dtype=torch.bfloat16) for d in (0, 1)}
    for d in (0, 1):      # this rank's slice of each direction: value = 100 d + rank + i / 64
        bufs[d][rank * width:(rank + 1) * width] = (100 * d + rank + torch.arange(width) / 64).bfloat16()
    fab.exchange_slices(bufs, dir_of[rank], dir_of, width, tag="param")
    out = bufs[dir_of[rank]].float().tolist()
    nbytes = dict(fab.bytes_by_tag)
    dist.destroy_process_group()
    q.put((rank, out, nbytes))


def gpu_strategy_worker(rank, world, port, strategy, name, steps, oracle, q):
    """GPU (all ranks on cuda:0, gloo collectives): run the eager strategy
    step of the drop-in API and report records + the master hash."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200 import ops
    from paper_2507_03211_b200.engine import DeviceStore
    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import RngStateManager, iteration_seeds
    from paper_2507_03211_b200.strategies import ddp_step, mesh_assignments, pertp_step, twod_step
    from paper_2507_03211_b200.zo import ZoHyper

    torch.cuda.set_device(0)
    init(rank, world, port)
    fab = TorchFabric()
    v, d, h, n, t, bsz = {"tiny": (16, 16, 2, 2, 8, 4), "mid": (64, 32, 4, 2, 16, 4)}[name]
    cfg = ModelConfig(v, d, h, n, t, "f32")
    store = DeviceStore(cfg, init_seed=7)
    hyper = ZoHyper(1e-3, 1e-2)
    mgr = RngStateManager("oracle" if oracle else "philox")
    recs = []
    for j, s in enumerate(iteration_seeds(5, steps), 1):
        batch = make_batch(cfg, bsz, 200 + j)
        seed_arg = s if rank == 0 else None
        if strategy == "pertp":
            r = pertp_step(fab, rank, store, batch, hyper, seed_arg, mgr, iteration=j)
        elif strategy == "ddp":
            r = ddp_step(fab, rank, store, batch.shard(world, rank), hyper, seed_arg, mgr, iteration=j)
        else:
            ordering = strategy.split(":")[1] if ":" in strategy else "pertp_inner"
            a = mesh_assignments(world // 2)[rank]
            r = twod_step(fab, rank, a, store, batch.shard(world // 2, a.group), hyper, seed_arg,
                          ordering=ordering, mgr=mgr, iteration=j)
        recs.append((r.loss_pos, r.loss_neg, r.g))
    hsh = int(ops.hash_u64(store.theta).item())
    theta = store.theta.cpu().numpy() if rank == 0 else None
    log = [c["kind"] + ":" + c["tag"] + ":" + str(c["participants"]) for c in fab.collective_log]
    dist.destroy_process_group()
    q.put((rank, recs, hsh, theta, log, dict(fab.bytes_by_tag)))


def run(fn, world, *args, timeout=240):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    import queue
    import time

    t_end = time.monotonic() + timeout
    try:
        while len(out) < world:
            try:
                item = q.get(timeout=2)
                out[item[0]] = item
                continue
            except queue.Empty:
                pass
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead:       # a worker raised: fail now instead of waiting out the timeout
                raise RuntimeError(f"worker process exited with {dead} (see its traceback above)")
            if time.monotonic() > t_end:
                raise TimeoutError(f"multi-process run did not finish within {timeout} s")
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    return [out[r] for r in range(world)]


DEEP = (64, 32, 4, 5, 16)


def sliced_offload_worker(rank, world, port, strategy, steps, q):
    """OffloadedZo with sliced H2D + all-gather / own-slice D2H (gloo, one GPU)."""
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import iteration_seeds
    from paper_2507_03211_b200.scheduler import HostStore, OffloadedZo
    from paper_2507_03211_b200.zo import ZoHyper

    torch.cuda.set_device(0)
    init(rank, world, port)
    fab = TorchFabric()
    cfg = ModelConfig(*DEEP, "f32")
    path = f"/dev/shm/zo_b200_test_{port}"
    if rank == 0:
        host = HostStore(cfg, 7, shared=path)
    fab.barrier()
    if rank != 0:
        host = HostStore(cfg, 7, init="attach", shared=path)
    rt = OffloadedZo(host, ZoHyper(1e-3, 1e-2), batch=4 // world, fabric=fab, strategy=strategy)
    recs = []
    for j, s in enumerate(iteration_seeds(9, steps), 1):
        r = rt.step(make_batch(cfg, 4, 40 + j).shard(world, rank), s)
        recs.append((r.loss_pos, r.loss_neg, r.g))
    rt.flush()
    torch.cuda.synchronize()
    fab.barrier()                     # every rank has written its slices back
    theta = host.theta.numpy().copy()
    host.close()
    fab.barrier()
    if rank == 0:
        os.unlink(path)
    dist.destroy_process_group()
    q.put((rank, recs, theta))


def gpu_strategy_worker_theta(rank, world, port, strategy, steps, q):
    """Resident eager strategy step on the DEEP config (reference for the
    sliced offload test)."""
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200.engine import DeviceStore
    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import iteration_seeds
    from paper_2507_03211_b200.strategies import ddp_step
    from paper_2507_03211_b200.zo import ZoHyper

    torch.cuda.set_device(0)
    init(rank, world, port)
    fab = TorchFabric()
    cfg = ModelConfig(*DEEP, "f32")
    store = DeviceStore(cfg, 7)
    recs = []
    for j, s in enumerate(iteration_seeds(9, steps), 1):
        r = ddp_step(fab, rank, store, make_batch(cfg, 4, 40 + j).shard(world, rank), ZoHyper(1e-3, 1e-2),
                     s if rank == 0 else None, iteration=j)
        recs.append((r.loss_pos, r.loss_neg, r.g))
    theta = store.theta.cpu().numpy()
    dist.destroy_process_group()
    q.put((rank, recs, theta))


def fullsize_mesh_worker(rank, world, port, steps, q):
    """The lazy 2D-mesh step (MeshZo, what bench.py runs at N > 1) at the
    OPT-1.3B headline size, one direction per rank, all ranks on cuda:0."""
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200 import ops
    from paper_2507_03211_b200.engine import MINUS, PLUS, DeviceStore
    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import make_batch, opt_config
    from paper_2507_03211_b200.rng import iteration_seeds
    from paper_2507_03211_b200.strategies import MeshZo
    from paper_2507_03211_b200.zo import ZoHyper

    torch.cuda.set_device(0)
    init(rank, world, port)
    fab = TorchFabric()
    cfg = opt_config("opt-1.3b", 512)
    store = DeviceStore(cfg, 7, init="philox", directions=(PLUS,) if rank % 2 == 0 else (MINUS,))
    groups = world // 2
    mz = MeshZo(store, ZoHyper(1e-3, 1e-7), fab, "2d", 4, 512)
    recs = []
    for j, s in enumerate(iteration_seeds(1234, steps)):
        r = mz.step(make_batch(cfg, 4 * groups, 99 * 1_000_003 + j + 1).shard(groups, rank // 2), s)
        recs.append((r.loss_pos, r.loss_neg, r.g))
    mz.flush()
    h = int(ops.hash_u64(store.theta).item())
    dist.destroy_process_group()
    q.put((rank, recs, h))


def sliced_dir_worker(rank, world, port, redistribute, steps, sharded, compress, strategy, q):
    """OffloadedZo on the 2D mesh (one direction per rank) with the fp32
    all-gather or the direction-aware bf16 exchange, over a
    shared host master or an HBM-sharded one (gloo, one GPU)."""
    _sliced_dir(rank, world, port, redistribute, steps, sharded, compress, strategy, q, "collective")


def sliced_dir_ce_worker(rank, world, port, redistribute, steps, sharded, strategy, q):
    """The same over the copy-engine data plane (CUDA IPC pulls)."""
    _sliced_dir(rank, world, port, redistribute, steps, sharded, "none", strategy, q, "copy_engine")


def _sliced_dir(rank, world, port, redistribute, steps, sharded, compress, strategy, q, data_plane):
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import iteration_seeds
    from paper_2507_03211_b200.scheduler import HostStore, OffloadedZo
    from paper_2507_03211_b200.sharded import ShardStore
    from paper_2507_03211_b200.zo import ZoHyper

    torch.cuda.set_device(0)
    init(rank, world, port)
    fab = TorchFabric(data_plane=data_plane)
    fab.CE_MIN_BYTES = 0           # the test model's slices are small: exercise the copy engines anyway
    cfg = ModelConfig(*DEEP, "f32")
    path = f"/dev/shm/zo_b200_test_{port}"
    if sharded:
        host = ShardStore(cfg, fab, 7)
    else:
        if rank == 0:
            host = HostStore(cfg, 7, shared=path)
        fab.barrier()
        if rank != 0:
            host = HostStore(cfg, 7, init="attach", shared=path)
    groups = world // 2 if strategy == "2d" else world
    rt = OffloadedZo(host, ZoHyper(1e-3, 1e-2), batch=4 // groups, fabric=fab, strategy=strategy,
                     redistribute=redistribute, compress=compress)
    fab.bytes_by_tag.clear()
    recs = []
    for j, s in enumerate(iteration_seeds(9, steps), 1):
        r = rt.step(make_batch(cfg, 4, 40 + j).shard(groups, rank // (world // groups)), s)
        recs.append((r.loss_pos, r.loss_neg, r.g))
    nbytes = dict(fab.bytes_by_tag)
    nbytes["pcie"] = rt.pcie_bytes_per_step()
    nbytes["ce_exchanges"] = fab.ce_exchanges
    rt.flush()
    torch.cuda.synchronize()
    fab.barrier()
    if sharded:
        theta = host.gather_master()
    else:
        theta = host.theta.numpy().copy()
        host.close()
        fab.barrier()
        if rank == 0:
            os.unlink(path)
    dist.destroy_process_group()
    q.put((rank, recs, theta, nbytes))


def verify_offload_worker(rank, world, port, q):
    """Sliced offload with the divergence guard: a clean step passes; a step
    in which rank 1's copy of a block is corrupted after its update raises
    ConsistencyError on every rank before anything is written back."""
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200.errors import ConsistencyError
    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import iteration_seeds
    from paper_2507_03211_b200.scheduler import OffloadedZo
    from paper_2507_03211_b200.sharded import ShardStore
    from paper_2507_03211_b200.zo import ZoHyper

    torch.cuda.set_device(0)
    init(rank, world, port)
    fab = TorchFabric()
    cfg = ModelConfig(*DEEP, "f32")
    shards = ShardStore(cfg, fab, 7)
    rt = OffloadedZo(shards, ZoHyper(1e-3, 1e-2), batch=4 // world, fabric=fab, strategy="mezo", verify=True,
                     mode="serial")
    seeds = iteration_seeds(9, 2)
    rt.step(make_batch(cfg, 4, 41).shard(world, rank), seeds[0])
    clean = True
    if rank == 1:
        orig = rt._perturb

        def corrupt(bid, slot, flags, stream):
            orig(bid, slot, flags, stream)
            if bid in rt.wids:
                with torch.cuda.stream(stream):
                    slot.theta[0:1].add_(1e-3)
        rt._perturb = corrupt
    raised = False
    try:
        rt.step(make_batch(cfg, 4, 42).shard(world, rank), seeds[1])
    except ConsistencyError:
        raised = True
    dist.destroy_process_group()
    q.put((rank, clean, raised))


def sharded_worker(rank, world, port, strategy, steps, init_kind, q):
    """OffloadedZo over an HBM-sharded fp32 master (sharded.ShardStore):
    upload = own shard slice + all-gather, offload = own slice back (gloo,
    all ranks on one GPU)."""
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import iteration_seeds
    from paper_2507_03211_b200.scheduler import OffloadedZo
    from paper_2507_03211_b200.sharded import ShardStore
    from paper_2507_03211_b200.zo import ZoHyper

    torch.cuda.set_device(0)
    init(rank, world, port)
    fab = TorchFabric()
    cfg = ModelConfig(*DEEP, "f32")
    shards = ShardStore(cfg, fab, 7, init=init_kind)
    init_master = shards.gather_master()
    rt = OffloadedZo(shards, ZoHyper(1e-3, 1e-2), batch=4 // world, fabric=fab, strategy=strategy)
    recs = []
    for j, s in enumerate(iteration_seeds(9, steps), 1):
        r = rt.step(make_batch(cfg, 4, 40 + j).shard(world, rank), s)
        recs.append((r.loss_pos, r.loss_neg, r.g))
    rt.flush()
    torch.cuda.synchronize()
    theta = shards.gather_master()
    nbytes = shards.shard_bytes
    dist.destroy_process_group()
    q.put((rank, recs, theta, init_master, nbytes))


def gpu_strategy_edge_worker(rank, world, port, case, q):
    """Edge contracts of the strategies (pkg/tests/test_strategies.py:114-232,
    321-326) on the GPU path, all ranks on cuda:0 with gloo."""
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200 import zo
    from paper_2507_03211_b200.engine import DeviceStore
    from paper_2507_03211_b200.errors import ConfigurationError, ConsistencyError
    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import RngStateManager, iteration_seeds
    from paper_2507_03211_b200.strategies import ddp_step, mesh_assignments, pertp_step, twod_step

    torch.cuda.set_device(0)
    init(rank, world, port)
    fab = TorchFabric()
    cfg = ModelConfig(16, 16, 2, 2, 8, "f32")
    hyper = zo.ZoHyper(1e-3, 1e-2)
    store = DeviceStore(cfg, init_seed=7)
    out = {}
    try:
        if case == "divergence":
            pertp_step(fab, rank, store, make_batch(cfg, 4, 3), hyper, 11 if rank == 0 else None)
            if rank == 1:
                store.theta[5] += 1e-3          # silent corruption on one replica
            try:
                pertp_step(fab, rank, store, make_batch(cfg, 4, 4), hyper, 12 if rank == 0 else None, iteration=2)
                out["raised"] = None
            except ConsistencyError:
                out["raised"] = "ConsistencyError"
        elif case == "traffic":
            for j, s in enumerate(iteration_seeds(1, 3), 1):
                ddp_step(fab, rank, store, make_batch(cfg, 8, j).shard(world, rank), hyper,
                         s if rank == 0 else None, RngStateManager(), iteration=j)
            out["bytes"] = dict(fab.bytes_by_tag)
        elif case == "k1":
            batch = make_batch(cfg, 4, 3)
            r = ddp_step(fab, rank, store, batch.shard(1, 0), hyper, 21)
            ref = DeviceStore(cfg, init_seed=7)
            rr = zo.mezo_step(ref, batch, hyper, 21)
            out["same"] = (r.g == rr.g) and bool(torch.equal(store.theta, ref.theta))
        elif case == "wrong_count":
            for name, fn in (("pertp", lambda: pertp_step(fab, rank, store, make_batch(cfg, 4, 3), hyper, 1)),
                             ("twod", lambda: twod_step(fab, rank, mesh_assignments(2)[0], store,
                                                        make_batch(cfg, 4, 1), hyper, 1))):
                try:
                    fn()
                    out[name] = None
                except ConfigurationError:
                    out[name] = "ConfigurationError"
    finally:
        dist.destroy_process_group()
    q.put((rank, out))


def mesh_golden_worker(rank, world, port, strategy, precision, teacher, golden_path, q):
    """The lazy mesh step (MeshZo, the production multi-GPU path) in oracle-z
    mode on the golden ``dist`` case (all ranks on cuda:0, gloo): records per
    step, and with ``teacher`` the reference's g fed back as g_prev, the
    flushed master's SHA-256 (the reference's ParamStore.checksum)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200.engine import MINUS, PLUS, DeviceStore
    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import RngStateManager
    from paper_2507_03211_b200.strategies import MeshZo
    from paper_2507_03211_b200.zo import ZoHyper

    torch.cuda.set_device(0)
    init(rank, world, port)
    fab = TorchFabric()
    gd = np.load(golden_path)
    cfg = ModelConfig(16, 16, 2, 2, 8, "f32")
    seeds = [int(np.uint64(s)) for s in gd["dist/seeds"].tolist()]
    kind, ordering = (strategy.split(":") + ["pertp_inner"])[:2]
    key = {"pertp": "dist/pertp", "ddp": f"dist/ddp{world}", "2d": f"dist/2d_{ordering}"}[kind]
    ref = gd[key]
    ref_mine = ref if kind == "pertp" else ref[rank]
    groups = {"pertp": 1, "ddp": world, "2d": world // 2}[kind]
    dirs = (PLUS, MINUS) if kind == "ddp" else ((PLUS,) if rank % 2 == 0 else (MINUS,))
    store = DeviceStore(cfg, init_seed=7, directions=dirs, precision=precision)
    gidx = rank if kind == "ddp" else rank // 2
    mz = MeshZo(store, ZoHyper(1e-3, 1e-2), fab, "2d" if kind == "pertp" else kind, 4 // groups, 8,
                mgr=RngStateManager("oracle"))
    recs = []
    for j, s in enumerate(seeds, 1):
        r = mz.step(make_batch(cfg, 4, 200 + j).shard(groups, gidx), s)
        recs.append((r.loss_pos, r.loss_neg, r.g))
        if teacher:
            mz.g_prev = float(ref_mine[j - 1][2])
    mz.flush()
    sha = store.checksum()
    theta = store.theta.cpu().numpy()
    dist.destroy_process_group()
    q.put((rank, recs, [tuple(map(float, x)) for x in ref_mine], sha, str(gd[key + "_sha"]), theta))


def nccl_world1_worker(rank, world, port, q):
    """(test_gpu_nccl) NCCL at world size 1: the captured mesh step and the
    sliced offload runtime over an NCCL fabric vs the single-GPU paths."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200 import zo
    from paper_2507_03211_b200.engine import DeviceStore
    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import iteration_seeds
    from paper_2507_03211_b200.scheduler import OffloadedZo
    from paper_2507_03211_b200.sharded import ShardStore
    from paper_2507_03211_b200.strategies import MeshZo

    torch.cuda.set_device(0)
    init(rank, world, port, backend="nccl")
    fab = TorchFabric()
    out = {"backend": fab.backend}
    cfg = ModelConfig(64, 32, 4, 3, 16, "f32")
    h = zo.ZoHyper(1e-3, 1e-2)
    seeds = iteration_seeds(71, 5)
    ref, mesh = DeviceStore(cfg, 7), DeviceStore(cfg, 7)
    sz = zo.StreamingZo(ref, h, overlap=False, graph=False)
    mz = MeshZo(mesh, h, fab, "ddp", 2, 16, graph=True)
    same = True
    for j, s in enumerate(seeds, 1):
        b = make_batch(cfg, 2, 900 + j)
        a, c = sz.step(b, s), mz.step(b, s)
        same &= (a.loss_pos, a.loss_neg, a.g) == (c.loss_pos, c.loss_neg, c.g)
    sz.flush()
    mz.flush()
    out["mesh_graph"] = bool(mz._graphs.get(True))       # the public step replays the I/O-carrying graph
    out["mesh_same"] = bool(same and torch.equal(ref.theta, mesh.theta))
    # sliced offload over the NCCL fabric, host-pinned per-rank slices (N = 1: the whole block)
    host = ShardStore(cfg, fab, 7, where="host")
    rt = OffloadedZo(host, h, batch=2, fabric=fab, strategy="mezo", trace=True)
    ref2 = DeviceStore(cfg, 7)
    sz2 = zo.StreamingZo(ref2, h, overlap=False, graph=False)
    same = True
    for j, s in enumerate(seeds, 1):
        b = make_batch(cfg, 2, 900 + j)
        a, c = sz2.step(b, s), rt.step(b, s)
        same &= (a.loss_pos, a.loss_neg, a.g) == (c.loss_pos, c.loss_neg, c.g)
    sz2.flush()
    rt.flush()
    out["offload_same"] = bool(same and np.array_equal(host.gather_master(), ref2.theta.cpu().numpy()))
    out["phases"] = sorted(rt.phase_stats)
    dist.destroy_process_group()
    q.put((rank, out))


def mesh_plan_worker(rank, world, port, strategy, overlap, steps, q):
    """MeshZo lazy steps (gloo, ranks sharing cuda:0) under one step plan:
    records and the flushed master, for the fill == serial check."""
    import torch
    import torch.distributed as dist

    from paper_2507_03211_b200 import ops
    from paper_2507_03211_b200.engine import DeviceStore
    from paper_2507_03211_b200.fabric import TorchFabric
    from paper_2507_03211_b200.model import ModelConfig, make_batch
    from paper_2507_03211_b200.rng import iteration_seeds
    from paper_2507_03211_b200.strategies import MeshZo
    from paper_2507_03211_b200.zo import ZoHyper

    torch.cuda.set_device(0)
    init(rank, world, port)
    fab = TorchFabric()
    cfg = ModelConfig(*DEEP, "f32")
    store = DeviceStore(cfg, 7)
    n_groups = world // 2 if strategy == "2d" else (1 if strategy == "pertp" else world)
    B = 2
    mz = MeshZo(store, ZoHyper(1e-3, 1e-2), fab, strategy, B, cfg.seq_len, overlap=overlap)
    recs = []
    for j, s in enumerate(iteration_seeds(13, steps), 1):
        b = make_batch(cfg, B * n_groups, 70 + j).shard(n_groups, mz.mesh.group)
        r = mz.step(b, s)
        recs.append((r.loss_pos, r.loss_neg, r.g))
    mz.flush()
    h = int(ops.hash_u64(store.theta).item())
    dist.destroy_process_group()
    q.put((rank, recs, h))
