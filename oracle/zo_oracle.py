"""CPU oracle for the DistZO2 zeroth-order training step.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2507_03211_b200`` may import
this module: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it, and only as the checker
or the timed CPU baseline, never as the thing measured or shipped.

What it is: a numpy restatement of the reference package ``zosim``
(``/root/reference/pkg/src/zosim``) for the hot path named in
BASELINE.json's north star: parameter layout, initialisation, synthetic
batches, the pure forward + loss, the perturb / restore / update arithmetic,
the eager (MeZO, Alg. 1) and lazy (ZO2, Alg. 2) step orders, the three
distribution strategies' scalar arithmetic, and the sliced-transfer layout.
Each function cites the reference file:line it follows.

Third-party arithmetic at the boundary: the Gaussian direction z is
``numpy.random.Generator(PCG64(seed)).standard_normal`` (numpy's ziggurat,
f64).  The reference pins only ``numpy>=1.24`` (pkg/pyproject.toml:8-11);
this image has numpy 2.3.5 and the golden fixtures record the version they
were generated with.

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference in
the build container and writes fixtures; ``tests/test_oracle_golden.py``
checks this restatement against them bit for bit (f32 and f64).

Data model: a model is a list of 1-D numpy arrays ("block buffers"), one per
block in reference order (embedding, N transformer blocks, head), each laid
out by ``tensor_spec`` (the layout fixes the z draw order).
"""

from __future__ import annotations

import numpy as np

LN_EPS = 1e-5          # src/zosim/model.py:28
INIT_STD = 0.02        # src/zosim/model.py:29
KINDS = ("embedding", "transformer", "head")


# --------------------------------------------------------------------------
# layout (src/zosim/model.py:60-63, 81-101)
# --------------------------------------------------------------------------

def tensor_spec(vocab: int, d: int, seq: int, kind: str):
    """Ordered (name, shape) list of one block; model.py:81-101."""
    if kind == "embedding":
        return [("tok_emb", (vocab, d)), ("pos_emb", (seq, d))]
    if kind == "transformer":
        out = []
        for nm, shp in (("ln1_g", (d,)), ("ln1_b", (d,)),
                        ("wq", (d, d)), ("bq", (d,)), ("wk", (d, d)), ("bk", (d,)),
                        ("wv", (d, d)), ("bv", (d,)), ("wo", (d, d)), ("bo", (d,)),
                        ("ln2_g", (d,)), ("ln2_b", (d,)),
                        ("w1", (d, 4 * d)), ("b1", (4 * d,)),
                        ("w2", (4 * d, d)), ("b2", (d,))):
            out.append((nm, shp))
        return out
    if kind == "head":
        return [("lnf_g", (d,)), ("lnf_b", (d,)), ("w_out", (d, vocab)), ("b_out", (vocab,))]
    raise ValueError(kind)


def block_kinds(n_blocks: int):
    return ["embedding"] + ["transformer"] * n_blocks + ["head"]


def views(buf: np.ndarray, spec):
    """name -> view into the flat block buffer (model.py:119-130)."""
    out, off = {}, 0
    for name, shape in spec:
        n = int(np.prod(shape))
        out[name] = buf[off:off + n].reshape(shape)
        off += n
    return out


def param_count(vocab, d, n_blocks, seq) -> int:
    """model.py:60-63."""
    return (vocab * d + seq * d) + n_blocks * (12 * d * d + 13 * d) + (2 * d + d * vocab + vocab)


# --------------------------------------------------------------------------
# init, batches, seeds (model.py:203-229, 270-274; rng.py:35-42)
# --------------------------------------------------------------------------

def init_blocks(vocab, d, n_blocks, seq, init_seed, dtype=np.float32):
    """Per-block PCG64(SeedSequence([init_seed, block_id])) stream; gains 1,
    biases 0, weights 0.02*N(0,1) cast to dtype.  model.py:203-229."""
    blocks = []
    for bid, kind in enumerate(block_kinds(n_blocks)):
        spec = tensor_spec(vocab, d, seq, kind)
        size = sum(int(np.prod(s)) for _, s in spec)
        buf = np.zeros(size, dtype=dtype)
        gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(init_seed), bid])))
        v = views(buf, spec)
        for name, shape in spec:
            if name.endswith("_g"):
                v[name][...] = 1.0
            elif name.startswith("b") or name.endswith("_b"):
                v[name][...] = 0.0
            else:
                n = int(np.prod(shape))
                v[name][...] = (INIT_STD * gen.standard_normal(n)).astype(dtype).reshape(shape)
        blocks.append(buf)
    return blocks


def synthetic_batch(vocab, seq, batch_size, seed):
    """ids/targets from PCG64(SeedSequence([seed, 0xDA7A])); model.py:270-274."""
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), 0xDA7A])))
    ids = gen.integers(0, vocab, size=(batch_size, seq + 1))
    return ids[:, :-1], ids[:, 1:]


def bench_batch_seed(data_seed: int, iteration: int) -> int:
    """bench.py:195-196."""
    return data_seed * 1_000_003 + iteration


def iteration_seeds(base_seed: int, steps: int):
    """rng.py:35-42."""
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(base_seed), 0x5EED])))
    return [int(s) for s in gen.integers(0, 2**63 - 1, size=steps)]


def z_stream(seed: int, sizes):
    """The direction z of one iteration, split per block in block order
    (zo.py:96, rng.py:11-13: per-block draws concatenate to one stream)."""
    gen = np.random.Generator(np.random.PCG64(int(seed)))
    return [gen.standard_normal(int(n)) for n in sizes]


# --------------------------------------------------------------------------
# forward + loss (model.py:280-372)
# --------------------------------------------------------------------------

def _ln(x, g, b):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + LN_EPS) * g + b


def _gelu_tanh(x):
    c = np.sqrt(np.asarray(2.0 / np.pi, dtype=x.dtype))
    return 0.5 * x * (1.0 + np.tanh(c * (x + 0.044715 * x ** 3)))


def block_forward(kind, buf, vocab, d, seq, n_heads, x):
    """One pure block forward; model.py:298-346 (pre-LN, exact causal
    softmax, tanh GELU; head = LN_f then the untied projection)."""
    p = views(buf, tensor_spec(vocab, d, seq, kind))
    if kind == "embedding":
        ids = np.asarray(x)
        return p["tok_emb"][ids] + p["pos_emb"][: ids.shape[1]][None, :, :]
    if kind == "transformer":
        bsz, t, _ = x.shape
        hd = d // n_heads

        def heads(a):
            return a.reshape(bsz, t, n_heads, hd).transpose(0, 2, 1, 3)

        h = _ln(x, p["ln1_g"], p["ln1_b"])
        q = heads(h @ p["wq"] + p["bq"])
        k = heads(h @ p["wk"] + p["bk"])
        v = heads(h @ p["wv"] + p["bv"])
        s = q @ k.transpose(0, 1, 3, 2) / np.sqrt(np.asarray(hd, dtype=x.dtype))
        causal = np.triu(np.ones((t, t), dtype=bool), k=1)
        s = np.where(causal, np.asarray(-np.inf, dtype=x.dtype), s)
        e = np.exp(s - s.max(axis=-1, keepdims=True))
        a = (e / e.sum(axis=-1, keepdims=True)) @ v
        x = x + (a.transpose(0, 2, 1, 3).reshape(bsz, t, d) @ p["wo"] + p["bo"])
        h2 = _ln(x, p["ln2_g"], p["ln2_b"])
        return x + (_gelu_tanh(h2 @ p["w1"] + p["b1"]) @ p["w2"] + p["b2"])
    h = _ln(x, p["lnf_g"], p["lnf_b"])
    return h @ p["w_out"] + p["b_out"]


def model_forward(blocks, vocab, d, seq, n_heads, n_blocks, ids):
    x = ids
    for kind, buf in zip(block_kinds(n_blocks), blocks):
        x = block_forward(kind, buf, vocab, d, seq, n_heads, x)
    return x


def cross_entropy(logits, targets) -> float:
    """Mean CE over every position, in f64; model.py:357-372."""
    l64 = np.asarray(logits).astype(np.float64, copy=False)
    if not np.isfinite(l64).all():
        raise FloatingPointError("non-finite logits")
    m = l64.max(axis=-1, keepdims=True)
    lse = m[..., 0] + np.log(np.exp(l64 - m).sum(axis=-1))
    picked = np.take_along_axis(l64, np.asarray(targets)[..., None], axis=-1)[..., 0]
    return float((lse - picked).mean())


# --------------------------------------------------------------------------
# perturb / update arithmetic (zo.py:80-130)
# --------------------------------------------------------------------------

def perturbed(base: np.ndarray, scale: float, z: np.ndarray) -> np.ndarray:
    """The value a block holds while perturbed by cumulative ``scale``:
    dtype(f64(base) + (scale*z)), always from the unperturbed base
    (zo.py:97-107).  scale == 0 returns the base itself (restore)."""
    if scale == 0.0:
        return base.copy()
    out = np.empty_like(base)
    np.add(base, scale * z, out=out, casting="same_kind")
    return out


def updated(buf: np.ndarray, g: float, lr: float, z: np.ndarray) -> np.ndarray:
    """theta - (lr*g)*z with the product formed first; zo.py:124-125."""
    out = np.empty_like(buf)
    np.subtract(buf, (lr * g) * z, out=out, casting="same_kind")
    return out


def zo_grad(lp: float, ln: float, eps: float) -> float:
    """zo.py:80-84."""
    if eps == 0:
        raise ZeroDivisionError("epsilon must be nonzero")
    return (lp - ln) / (2.0 * eps)


# --------------------------------------------------------------------------
# step drivers
# --------------------------------------------------------------------------

class Model:
    """Dimensions + block buffers; a tiny stand-in for zosim.ParamStore."""

    def __init__(self, vocab, d, n_heads, n_blocks, seq, init_seed=7, dtype=np.float32, blocks=None):
        self.vocab, self.d, self.n_heads, self.n_blocks, self.seq = vocab, d, n_heads, n_blocks, seq
        self.dtype = dtype
        self.blocks = blocks if blocks is not None else init_blocks(vocab, d, n_blocks, seq, init_seed, dtype)

    @property
    def sizes(self):
        return [b.size for b in self.blocks]

    def copy(self):
        return Model(self.vocab, self.d, self.n_heads, self.n_blocks, self.seq,
                     dtype=self.dtype, blocks=[b.copy() for b in self.blocks])

    def forward(self, ids, blocks=None):
        return model_forward(blocks if blocks is not None else self.blocks,
                             self.vocab, self.d, self.seq, self.n_heads, self.n_blocks, ids)

    def loss_at(self, scale, zs, ids, tgts):
        pert = [perturbed(b, scale, z) for b, z in zip(self.blocks, zs)]
        return cross_entropy(self.forward(ids, pert), tgts)


def mezo_step(model: Model, ids, tgts, eps, lr, seed, zs=None):
    """Alg. 1 / zo.py:136-168: L+ at base+eps z, L- at base-eps z (both from
    the unperturbed base), restore, g, then theta -= (lr g) z in place.
    Returns (loss_pos, loss_neg, g)."""
    zs = zs if zs is not None else z_stream(seed, model.sizes)
    lp = model.loss_at(+eps, zs, ids, tgts)
    ln = model.loss_at(-eps, zs, ids, tgts)
    g = zo_grad(lp, ln, eps)
    model.blocks = [updated(b, g, lr, z) for b, z in zip(model.blocks, zs)]
    return lp, ln, g


class LazyZo:
    """Alg. 2 / zo.py:245-293 (StreamingZo) and scheduler.py:243-283
    (OffloadedZo): the update of iteration j is applied to each block just
    before it is perturbed in iteration j+1; ``flush`` applies the last one.
    Numerically identical to repeated ``mezo_step`` after the flush."""

    def __init__(self, model: Model, eps, lr):
        self.model, self.eps, self.lr = model, eps, lr
        self.pending = None        # (g, zs) of the last iteration

    def step(self, ids, tgts, seed):
        m = self.model
        zs = z_stream(seed, m.sizes)
        if self.pending is not None:
            g_prev, zs_prev = self.pending
            m.blocks = [updated(b, g_prev, self.lr, z) for b, z in zip(m.blocks, zs_prev)]
        lp = m.loss_at(+self.eps, zs, ids, tgts)
        ln = m.loss_at(-self.eps, zs, ids, tgts)
        g = zo_grad(lp, ln, self.eps)
        self.pending = (g, zs)
        return lp, ln, g

    def flush(self):
        if self.pending is None:
            raise RuntimeError("flush with no pending update")
        g, zs = self.pending
        self.model.blocks = [updated(b, g, self.lr, z) for b, z in zip(self.model.blocks, zs)]
        self.pending = None


def ordered_mean(values):
    """Ascending-rank sum then divide; fabric.py:105-113."""
    total = 0.0
    for v in values:
        total += v
    return total / len(values)


def ddp_grads(model: Model, ids, tgts, eps, k, seed):
    """Per-shard projected gradients of one ZO-DDP iteration
    (strategies.py:128-151): shard r = contiguous rows (model.py:261-267)."""
    zs = z_stream(seed, model.sizes)
    step = ids.shape[0] // k
    out = []
    for r in range(k):
        sl = slice(r * step, (r + 1) * step)
        lp = model.loss_at(+eps, zs, ids[sl], tgts[sl])
        ln = model.loss_at(-eps, zs, ids[sl], tgts[sl])
        out.append((lp, ln, zo_grad(lp, ln, eps)))
    return out, zs


def ddp_step(model: Model, ids, tgts, eps, lr, k, seed):
    """strategies.py:128-151: g = ordered mean of the shard g's."""
    per, zs = ddp_grads(model, ids, tgts, eps, k, seed)
    g = ordered_mean([p[2] for p in per])
    model.blocks = [updated(b, g, lr, z) for b, z in zip(model.blocks, zs)]
    return per, g


def twod_step(model: Model, ids, tgts, eps, lr, n_groups, seed, ordering="pertp_inner"):
    """strategies.py:154-222.  Both orderings reduce to the ordered mean of
    per-group central differences; pertp_inner sums group gradients, the
    ddp_inner ordering sums zo_grad(plus_i, minus_i) in the same order."""
    per, zs = ddp_grads(model, ids, tgts, eps, n_groups, seed)
    total = 0.0
    for lp, ln, gi in per:
        total += gi if ordering == "pertp_inner" else zo_grad(lp, ln, eps)
    g = total / n_groups
    model.blocks = [updated(b, g, lr, z) for b, z in zip(model.blocks, zs)]
    return per, g


# --------------------------------------------------------------------------
# sliced transfer layout + byte semantics (comm.py:106-119, 250-256, 314-342)
# --------------------------------------------------------------------------

def slice_layout(total: int, n: int):
    """[(owner, offset, length)]: ceil-width slices, last may be short or
    empty; comm.py:106-119."""
    width = -(-total // n)
    out, off = [], 0
    for owner in range(n):
        length = max(min(width, total - off), 0)
        out.append((owner, off, length))
        off += length
    return out


def sliced_upload_time(total: int, n: int, host_bw: float, peer_bw: float) -> float:
    """T_comm = ceil(M/n)/BW_host + (M - ceil(M/n))/BW_peer; comm.py:250-256."""
    width = -(-total // n)
    return width / host_bw + (total - width) / peer_bw


def sliced_upload(host_buf: np.ndarray, n: int):
    """Phase 1 owners pull their slice from the host, phase 2 peers fill the
    rest from the owner; comm.py:314-328."""
    layout = slice_layout(host_buf.size, n)
    reps = [np.empty_like(host_buf) for _ in range(n)]
    for owner, off, ln in layout:
        reps[owner][off:off + ln] = host_buf[off:off + ln]
    for owner, off, ln in layout:
        for dst in range(n):
            if dst != owner:
                reps[dst][off:off + ln] = reps[owner][off:off + ln]
    return reps


def sliced_offload(reps, host_buf: np.ndarray):
    """Own slice back to the host after a byte-identity check; comm.py:331-342."""
    if len({r.tobytes() for r in reps}) != 1:
        raise ValueError("device replicas diverged")
    for owner, off, ln in slice_layout(host_buf.size, len(reps)):
        host_buf[off:off + ln] = reps[owner][off:off + ln]
