"""Measured gaps of the f32 parity mode and of the bf16 production path
against the real reference's recorded trajectories (tests/golden) and, for
the OPT-125M shape, against the oracle's eager step."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import zo_oracle as O  # noqa: E402
from paper_2507_03211_b200 import zo  # noqa: E402
from paper_2507_03211_b200.engine import DeviceStore  # noqa: E402
from paper_2507_03211_b200.model import Batch, ModelConfig, opt_config  # noqa: E402
from paper_2507_03211_b200.rng import RngStateManager  # noqa: E402

g = dict(np.load("tests/golden/golden.npz"))
meta = json.loads(str(g["meta"]))
out = {}
for c in meta["cases"]:
    if c["dtype"] != "f32":
        continue
    cfg = ModelConfig(c["vocab"], c["d"], c["heads"], c["n_blocks"], c["seq"], "f32")
    for prec in ("f32", "bf16"):
        store = DeviceStore(cfg, init_seed=7, precision=prec)
        sz = zo.StreamingZo(store, zo.ZoHyper(1e-3, 1e-2), mgr=RngStateManager("oracle"))
        ref = g[f"{c['name']}/streaming"]
        dl, dg = 0.0, 0.0
        for j, s in enumerate(g[f"{c['name']}/seeds"].tolist(), 1):
            r = sz.step(Batch(g[f"{c['name']}/ids/{j}"], g[f"{c['name']}/tgt/{j}"]), int(s))
            dl = max(dl, abs(r.loss_pos - ref[j - 1][0]), abs(r.loss_neg - ref[j - 1][1]))
            dg = max(dg, abs(r.g - ref[j - 1][2]) / max(1.0, abs(ref[j - 1][2])))
        sz.flush()
        th = store.theta.cpu().numpy()
        fin = np.concatenate([g[f"{c['name']}/final/{b}"] for b in range(c["n_blocks"] + 2)])
        out[f"{c['name']}/{prec}"] = {"max_dloss": dl, "max_rel_dg": dg,
                                      "max_dtheta": float(np.abs(th.astype(np.float64) - fin).max())}
cfg = opt_config("opt-125m", 64)
om = O.Model(cfg.vocab_size, cfg.d_model, cfg.n_heads, cfg.n_blocks, cfg.seq_len, init_seed=7)
seed = O.iteration_seeds(1234, 1)[0]
ids, tg = O.synthetic_batch(cfg.vocab_size, cfg.seq_len, 1, O.bench_batch_seed(99, 1))
lp, ln, gg = O.mezo_step(om, ids, tg, 1e-3, 1e-2, seed)
for prec in ("f32", "bf16"):
    st = DeviceStore(cfg, init_seed=7, precision=prec)
    r = zo.mezo_step(st, Batch(ids, tg), zo.ZoHyper(1e-3, 1e-2), seed, mgr=RngStateManager("oracle"))
    out[f"opt-125m-shape/{prec}"] = {"max_dloss": max(abs(r.loss_pos - lp), abs(r.loss_neg - ln)),
                                     "max_rel_dg": abs(r.g - gg) / max(1.0, abs(gg))}
print(json.dumps(out, indent=1))
