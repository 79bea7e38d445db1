"""Model configuration, parameter layout, initialisation and synthetic batches.

Mirrors src/zosim/model.py: the same ``ModelConfig`` fields and validation,
the same per-block tensor order (which fixes the direction-z draw order and
the global element keys), the same ``init_model`` / ``make_batch`` seed
schemes.  Parameters live on the GPU (engine.DeviceStore); this module is
pure host-side bookkeeping.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass

import numpy as np

from .errors import ConfigurationError, DimensionError

EMBEDDING, TRANSFORMER, HEAD = "embedding", "transformer", "head"
LN_EPS = 1e-5
INIT_STD = 0.02
DTYPES = ("f32", "f64")


@dataclass(frozen=True)
class ModelConfig:
    """src/zosim/model.py:34-78.  ``dtype`` is the master dtype the reference
    computes in; the B200 build keeps an fp32 master either way (f64 masters
    are accepted for API compatibility and stored as fp32)."""

    vocab_size: int
    d_model: int
    n_heads: int
    n_blocks: int
    seq_len: int
    dtype: str = "f64"

    def validate(self) -> "ModelConfig":
        for name in ("vocab_size", "d_model", "n_heads", "n_blocks", "seq_len"):
            v = getattr(self, name)
            if not isinstance(v, int) or v < 1:
                raise ConfigurationError(f"{name} must be a positive integer, got {v!r}")
        if self.d_model % self.n_heads != 0:
            raise ConfigurationError(f"d_model={self.d_model} must be divisible by n_heads={self.n_heads}")
        if self.dtype not in DTYPES:
            raise ConfigurationError(f"dtype must be one of {sorted(DTYPES)}, got {self.dtype!r}")
        return self

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def param_count(self) -> int:
        d, v, s = self.d_model, self.vocab_size, self.seq_len
        return (v * d + s * d) + self.n_blocks * (12 * d * d + 13 * d) + (2 * d + d * v + v)

    arch = "zosim"

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, d: dict) -> "ModelConfig":
        try:
            if d.get("arch") == "opt":
                return OPTConfig(**d).validate()
            return cls(**d).validate()
        except TypeError as e:
            raise ConfigurationError(f"bad model config: {e}") from e

    @classmethod
    def from_json(cls, path) -> "ModelConfig":
        with open(path) as f:
            return cls.from_dict(json.load(f))


@dataclass(frozen=True)
class OPTConfig(ModelConfig):
    """Real OPT (HF ``OPTForCausalLM`` with do_layer_norm_before=True, i.e.
    every size except 350m).  Differences from
    the zosim architecture (model.py:81-101, 286-289, 339-344):
      * ReLU FFN instead of tanh-GELU;
      * learned positions with ``max_positions + 2`` rows, position t reads
        row t + 2 (OPTLearnedPositionalEmbedding's offset);
      * the LM head is tied to the token embedding and has no bias, so the
        head block holds only the final LayerNorm.
    Linear weights are kept in the (d_in, d_out) layout of the zosim blocks;
    the HF loader (opt.py) transposes nn.Linear's (out, in)."""

    max_positions: int = 2048
    arch: str = "opt"

    def validate(self) -> "OPTConfig":
        super().validate()
        if self.arch != "opt":
            raise ConfigurationError(f"OPTConfig.arch must be 'opt', got {self.arch!r}")
        if not isinstance(self.max_positions, int) or self.seq_len > self.max_positions:
            raise ConfigurationError(f"seq_len={self.seq_len} exceeds max_positions={self.max_positions}")
        return self

    def param_count(self) -> int:
        d, v = self.d_model, self.vocab_size
        return (v * d + (self.max_positions + 2) * d) + self.n_blocks * (12 * d * d + 13 * d) + 2 * d


# Real OPT family (facebook/opt-*; 350m is post-LN with a projected
# embedding and is not covered)
REAL_OPT_SHAPES = {
    "opt-125m": dict(d_model=768, n_heads=12, n_blocks=12),
    "opt-1.3b": dict(d_model=2048, n_heads=32, n_blocks=24),
    "opt-2.7b": dict(d_model=2560, n_heads=32, n_blocks=32),
    "opt-6.7b": dict(d_model=4096, n_heads=32, n_blocks=32),
    "opt-13b": dict(d_model=5120, n_heads=40, n_blocks=40),
    "opt-30b": dict(d_model=7168, n_heads=56, n_blocks=48),
    "opt-66b": dict(d_model=9216, n_heads=72, n_blocks=64),
    "opt-175b": dict(d_model=12288, n_heads=96, n_blocks=96),
}


def real_opt_config(name: str, seq_len: int, dtype: str = "f32", vocab_size: int = 50272,
                    max_positions: int = 2048) -> OPTConfig:
    return OPTConfig(vocab_size=vocab_size, seq_len=seq_len, dtype=dtype, max_positions=max_positions,
                     **REAL_OPT_SHAPES[name]).validate()


# OPT-family shapes on the zosim architecture (SURVEY.md section 8 shape sheet)
OPT_SHAPES = {
    "opt-125m": dict(vocab_size=50272, d_model=768, n_heads=12, n_blocks=12),
    "opt-1.3b": dict(vocab_size=50272, d_model=2048, n_heads=32, n_blocks=24),
    "opt-13b": dict(vocab_size=50272, d_model=5120, n_heads=40, n_blocks=40),
    "opt-66b": dict(vocab_size=50272, d_model=9216, n_heads=72, n_blocks=64),
    "opt-175b": dict(vocab_size=50272, d_model=12288, n_heads=96, n_blocks=96),
}


def opt_config(name: str, seq_len: int, dtype: str = "f32") -> ModelConfig:
    return ModelConfig(seq_len=seq_len, dtype=dtype, **OPT_SHAPES[name]).validate()


def block_tensor_spec(config: ModelConfig, kind: str):
    """Ordered (name, shape) list of one block (model.py:81-101); for
    OPTConfig the real-OPT variant (positions table with the offset rows,
    head = final LayerNorm only)."""
    d, v, s = config.d_model, config.vocab_size, config.seq_len
    opt = config.arch == "opt"
    if kind == EMBEDDING:
        return [("tok_emb", (v, d)), ("pos_emb", ((config.max_positions + 2) if opt else s, d))]
    if kind == TRANSFORMER:
        return [("ln1_g", (d,)), ("ln1_b", (d,)), ("wq", (d, d)), ("bq", (d,)), ("wk", (d, d)), ("bk", (d,)),
                ("wv", (d, d)), ("bv", (d,)), ("wo", (d, d)), ("bo", (d,)), ("ln2_g", (d,)), ("ln2_b", (d,)),
                ("w1", (d, 4 * d)), ("b1", (4 * d,)), ("w2", (4 * d, d)), ("b2", (d,))]
    if kind == HEAD:
        if opt:
            return [("lnf_g", (d,)), ("lnf_b", (d,))]
        return [("lnf_g", (d,)), ("lnf_b", (d,)), ("w_out", (d, v)), ("b_out", (v,))]
    raise ConfigurationError(f"unknown block kind {kind!r}")


def block_kinds(config: ModelConfig):
    return [EMBEDDING] + [TRANSFORMER] * config.n_blocks + [HEAD]


class BlockLayout:
    """Tensor offsets of one block inside the flat master and its global key
    range [key0, key0 + elem_count)."""

    def __init__(self, block_id: int, kind: str, spec, key0: int):
        self.block_id, self.kind, self.key0 = block_id, kind, key0
        self.names = [n for n, _ in spec]
        self.shapes = {n: tuple(s) for n, s in spec}
        self.offsets = {}
        off = 0
        for n, s in spec:
            self.offsets[n] = off
            off += int(np.prod(s))
        self.elem_count = off

    def key(self, name: str) -> int:
        return self.key0 + self.offsets[name]

    def size(self, name: str) -> int:
        return int(np.prod(self.shapes[name]))


def model_layout(config: ModelConfig):
    out, key = [], 0
    for bid, kind in enumerate(block_kinds(config)):
        bl = BlockLayout(bid, kind, block_tensor_spec(config, kind), key)
        out.append(bl)
        key += bl.elem_count
    return out


def init_block_host(config: ModelConfig, layout: BlockLayout, init_seed: int, dtype=np.float32) -> np.ndarray:
    """One block's initial values exactly as zosim draws them
    (model.py:203-229): PCG64(SeedSequence([init_seed, block_id])), gains 1,
    biases 0, weights INIT_STD * N(0,1) cast to the config dtype."""
    cdt = np.float32 if config.dtype == "f32" else np.float64
    buf = np.zeros(layout.elem_count, dtype=cdt)
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(init_seed), layout.block_id])))
    for name in layout.names:
        o, n = layout.offsets[name], layout.size(name)
        if name.endswith("_g"):
            buf[o:o + n] = 1.0
        elif name.startswith("b") or name.endswith("_b"):
            buf[o:o + n] = 0.0
        else:
            buf[o:o + n] = (INIT_STD * gen.standard_normal(n)).astype(cdt)
    return buf.astype(dtype, copy=False)


@dataclass
class Batch:
    """src/zosim/model.py:232-267."""

    token_ids: np.ndarray
    targets: np.ndarray

    def __post_init__(self):
        self.token_ids = np.asarray(self.token_ids)
        self.targets = np.asarray(self.targets)
        if self.token_ids.shape != self.targets.shape:
            raise DimensionError(f"token_ids shape {self.token_ids.shape} != targets shape {self.targets.shape}")
        if self.token_ids.ndim != 2:
            raise DimensionError(f"batch must be 2-D (batch, seq), got {self.token_ids.ndim}-D")

    def validate(self, config: ModelConfig) -> "Batch":
        if self.token_ids.shape[1] > config.seq_len:
            raise DimensionError(f"sequence length {self.token_ids.shape[1]} exceeds model seq_len {config.seq_len}")
        for name, arr in (("token_ids", self.token_ids), ("targets", self.targets)):
            if arr.size and (arr.min() < 0 or arr.max() >= config.vocab_size):
                raise ConfigurationError(f"{name} out of range for vocab_size={config.vocab_size}")
        return self

    @property
    def size(self) -> int:
        return self.token_ids.shape[0]

    def shard(self, k: int, rank: int) -> "Batch":
        if self.size % k != 0:
            raise ConfigurationError(f"batch size {self.size} not divisible by {k} shards")
        step = self.size // k
        return Batch(self.token_ids[rank * step:(rank + 1) * step], self.targets[rank * step:(rank + 1) * step])


def make_batch(config: ModelConfig, batch_size: int, seed: int) -> Batch:
    """Synthetic next-token batch (model.py:270-274)."""
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), 0xDA7A])))
    ids = gen.integers(0, config.vocab_size, size=(batch_size, config.seq_len + 1))
    return Batch(ids[:, :-1], ids[:, 1:])
