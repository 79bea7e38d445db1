"""Generate the golden fixtures from the REAL reference (zosim).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports ``zosim`` from /root/reference/pkg/src (read-only, never copied),
runs the reference's own public API on small seeded cases and writes
``tests/golden/golden.npz``.  The fixtures pin ``oracle/zo_oracle.py``
(tests/test_oracle_golden.py) and, through the oracle, the GPU parity tests.
The GPU box never reads /root/reference; it only sees the committed npz.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

# (name, vocab, d, heads, n_blocks, seq, dtype, batch, steps)
CASES = [
    ("tiny32", 16, 16, 2, 2, 8, "f32", 4, 3),
    ("tiny64", 16, 16, 2, 2, 8, "f64", 4, 3),
    ("ragged32", 7, 6, 2, 1, 6, "f32", 2, 2),
    ("mid32", 64, 32, 4, 2, 16, "f32", 2, 3),
    ("wide32", 96, 64, 4, 1, 32, "f32", 2, 2),
]


def main():
    sys.path.insert(0, REF_SRC)
    import zosim
    from zosim import (ModelConfig, StreamingZo, ZoHyper, init_model, iteration_seeds,
                       make_batch, mezo_step, zo_grad, loss, Batch)
    from zosim.comm import LinkTopology, SliceLayout, sliced_upload_time
    from zosim.fabric import WorkerFabric
    from zosim.scheduler import OffloadedZo
    from zosim.strategies import ddp_step, mesh_assignments, pertp_step, twod_step

    out = {}
    meta = {"numpy": np.__version__, "zosim": zosim.__version__, "cases": []}
    hyper = ZoHyper(epsilon=1e-3, lr=1e-2, steps=4)

    for name, v, d, h, n, t, dt, bsz, steps in CASES:
        cfg = ModelConfig(v, d, h, n, t, dt)
        meta["cases"].append({"name": name, "vocab": v, "d": d, "heads": h, "n_blocks": n,
                              "seq": t, "dtype": dt, "batch": bsz, "steps": steps})
        store = init_model(cfg, 7)
        for b in store.blocks:
            out[f"{name}/init/{b.block_id}"] = b.buf.copy()
        seeds = iteration_seeds(17, steps)
        out[f"{name}/seeds"] = np.array(seeds, dtype=np.int64)
        # z of the first iteration, per block (pins numpy's PCG64 ziggurat)
        gen = np.random.Generator(np.random.PCG64(seeds[0]))
        for b in store.blocks:
            out[f"{name}/z0/{b.block_id}"] = gen.standard_normal(b.elem_count)
        # the eager MeZO trajectory
        recs = []
        for j, s in enumerate(seeds, 1):
            batch = make_batch(cfg, bsz, 100 + j)
            out[f"{name}/ids/{j}"] = batch.token_ids.copy()
            out[f"{name}/tgt/{j}"] = batch.targets.copy()
            if j == 1:
                logits = zosim.forward(store, batch.token_ids)
                out[f"{name}/logits1"] = logits
                out[f"{name}/loss1"] = np.float64(loss(logits, batch))
            r = mezo_step(store, batch, hyper, s, iteration=j)
            recs.append((r.loss_pos, r.loss_neg, r.g))
            if j == 1:
                for b in store.blocks:
                    out[f"{name}/after1/{b.block_id}"] = b.buf.copy()
        out[f"{name}/mezo"] = np.array(recs, dtype=np.float64)
        for b in store.blocks:
            out[f"{name}/final/{b.block_id}"] = b.buf.copy()
        out[f"{name}/final_sha"] = np.array(store.checksum())
        # ZOPK checkpoint bytes of the trained store (model.py:381-401)
        import tempfile
        from zosim import save_checkpoint
        with tempfile.TemporaryDirectory() as td:
            p = os.path.join(td, "ck.zopk")
            save_checkpoint(store, p)
            out[f"{name}/ckpt"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8).copy()

        # lazy streaming and the offload scheduler (must match eager)
        lazy = init_model(cfg, 7)
        sz = StreamingZo(lazy, hyper)
        srecs = []
        for j, s in enumerate(seeds, 1):
            r = sz.step(make_batch(cfg, bsz, 100 + j), s)
            srecs.append((r.loss_pos, r.loss_neg, r.g))
        for b in lazy.blocks:
            out[f"{name}/lazy_unflushed/{b.block_id}"] = b.buf.copy()
        sz.flush()
        out[f"{name}/streaming"] = np.array(srecs, dtype=np.float64)
        out[f"{name}/streaming_sha"] = np.array(lazy.checksum())
        if n >= 1:
            off = init_model(cfg, 7)
            rt = OffloadedZo(off, hyper)
            orecs = []
            for j, s in enumerate(seeds, 1):
                r = rt.step(make_batch(cfg, bsz, 100 + j), s)
                orecs.append((r.loss_pos, r.loss_neg, r.g))
            rt.flush()
            out[f"{name}/offload"] = np.array(orecs, dtype=np.float64)
            out[f"{name}/offload_sha"] = np.array(off.checksum())

    # distributed strategies on the tiny f32 case
    cfg = ModelConfig(16, 16, 2, 2, 8, "f32")
    seeds = iteration_seeds(5, 3)
    out["dist/seeds"] = np.array(seeds, dtype=np.int64)

    def run_fabric(k, fn):
        fab = WorkerFabric(k)
        stores = [init_model(cfg, 7) for _ in range(k)]
        res = fab.run(lambda rank: fn(fab, rank, stores[rank]))
        return res, stores, fab

    def pertp(fab, rank, store):
        mgr = zosim.RngStateManager()
        return [pertp_step(fab, rank, store, make_batch(cfg, 4, 200 + j), hyper,
                           s if rank == 0 else None, mgr, iteration=j)
                for j, s in enumerate(seeds, 1)]

    res, stores, _ = run_fabric(2, pertp)
    out["dist/pertp"] = np.array([(r.loss_pos, r.loss_neg, r.g) for r in res[0]])
    out["dist/pertp_sha"] = np.array(stores[0].checksum())

    for k in (2, 4):
        def ddp(fab, rank, store, k=k):
            mgr = zosim.RngStateManager()
            return [ddp_step(fab, rank, store, make_batch(cfg, 4, 200 + j).shard(k, rank), hyper,
                             s if rank == 0 else None, mgr, iteration=j)
                    for j, s in enumerate(seeds, 1)]
        res, stores, _ = run_fabric(k, ddp)
        out[f"dist/ddp{k}"] = np.array([[(r.loss_pos, r.loss_neg, r.g) for r in rr] for rr in res])
        out[f"dist/ddp{k}_sha"] = np.array(stores[0].checksum())

    for ordering in ("pertp_inner", "ddp_inner"):
        assigns = mesh_assignments(2)

        def twod(fab, rank, store, ordering=ordering):
            mgr = zosim.RngStateManager()
            a = assigns[rank]
            return [twod_step(fab, rank, a, store, make_batch(cfg, 4, 200 + j).shard(2, a.group),
                              hyper, s if rank == 0 else None, ordering=ordering, mgr=mgr, iteration=j)
                    for j, s in enumerate(seeds, 1)]
        res, stores, _ = run_fabric(4, twod)
        out[f"dist/2d_{ordering}"] = np.array([[(r.loss_pos, r.loss_neg, r.g) for r in rr] for rr in res])
        out[f"dist/2d_{ordering}_sha"] = np.array(stores[0].checksum())

    # comm: slice layouts and the T_comm model
    lay = []
    for total, nn in ((10, 3), (7, 4), (3, 8), (1000, 8), (7087872, 8), (1, 1), (5, 5)):
        for s in SliceLayout.build(0, total, nn).slices:
            lay.append((total, nn, s.owner, s.offset, s.length))
    out["comm/layouts"] = np.array(lay, dtype=np.int64)
    topo = LinkTopology(host_bw=4e8, peer_bw=2.4e9, latency=0.0, devices=8)
    out["comm/tcomm"] = np.array([(m, nn, sliced_upload_time(m, nn, topo))
                                  for m in (1000, 7087872, 50358272) for nn in (1, 2, 4, 8)])

    # known answers
    out["kat/zo_grad"] = np.array([zo_grad(1.2, 0.8, 0.1), zo_grad(1.5, 1.5, 0.1)])
    b = Batch(np.zeros((2, 3), dtype=np.int64), np.zeros((2, 3), dtype=np.int64))
    out["kat/ce_uniform4"] = np.float64(loss(np.zeros((2, 3, 4)), b))
    out["kat/iteration_seeds_1234"] = np.array(iteration_seeds(1234, 8), dtype=np.int64)

    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT, **out)
    h = hashlib.sha256(open(OUT, "rb").read()).hexdigest()[:16]
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, sha256 {h}); keys={len(out)}")


if __name__ == "__main__":
    main()
