"""Real-OPT compatibility: HF ``OPTForCausalLM``
weights <-> the B200 master.

The zosim architecture the reference trains differs from real OPT (ReLU FFN,
tied bias-free LM head, learned positions with offset 2); ``OPTConfig``
(model.py) describes the real one and the engine runs it with the same
kernels (ZO_EPI_BIAS_RELU_BF16, and the CE head GEMM reading the token
embedding's bf16 shadow as a K-major B operand).

Master layout for an OPTConfig (which keys the direction z):
  block 0          tok_emb [V, d], pos_emb [max_positions + 2, d]
  blocks 1..N      ln1_g, ln1_b, wq, bq, wk, bk, wv, bv, wo, bo, ln2_g, ln2_b,
                   w1, b1, w2, b2  (zosim order; weights (d_in, d_out), i.e.
                   nn.Linear's (out, in) transposed on load)
  block N+1        lnf_g, lnf_b
HF names (transformers' modeling_opt):
  model.decoder.embed_tokens / embed_positions / final_layer_norm,
  model.decoder.layers.{i}.self_attn.{q,k,v,out}_proj, self_attn_layer_norm,
  fc1, fc2, final_layer_norm; lm_head.weight is tied to embed_tokens.

Files: ``model.safetensors`` (optionally sharded with
``model.safetensors.index.json``) or ``pytorch_model.bin``, plus
``config.json``.  No network: point ``load_pretrained`` at a local directory.
"""

from __future__ import annotations

import json
import os

import numpy as np

from .errors import ConfigurationError, DimensionError
from .model import OPTConfig, model_layout

_PFX = "model.decoder."
_LAYER_MAP = [  # (our name, HF suffix, transpose)
    ("ln1_g", "self_attn_layer_norm.weight", False), ("ln1_b", "self_attn_layer_norm.bias", False),
    ("wq", "self_attn.q_proj.weight", True), ("bq", "self_attn.q_proj.bias", False),
    ("wk", "self_attn.k_proj.weight", True), ("bk", "self_attn.k_proj.bias", False),
    ("wv", "self_attn.v_proj.weight", True), ("bv", "self_attn.v_proj.bias", False),
    ("wo", "self_attn.out_proj.weight", True), ("bo", "self_attn.out_proj.bias", False),
    ("ln2_g", "final_layer_norm.weight", False), ("ln2_b", "final_layer_norm.bias", False),
    ("w1", "fc1.weight", True), ("b1", "fc1.bias", False),
    ("w2", "fc2.weight", True), ("b2", "fc2.bias", False),
]


def config_from_hf(hf: dict, seq_len: int | None = None) -> OPTConfig:
    """OPTConfig from a HF ``config.json`` dict; refuses the variants the
    engine does not run (post-LN 350m, projected embeddings, non-ReLU)."""
    d = hf["hidden_size"]
    checks = [
        (hf.get("do_layer_norm_before", True), "do_layer_norm_before=False (opt-350m) is not supported"),
        (hf.get("word_embed_proj_dim", d) == d, "word_embed_proj_dim != hidden_size is not supported"),
        (hf.get("ffn_dim", 4 * d) == 4 * d, "ffn_dim must be 4 * hidden_size"),
        (hf.get("activation_function", "relu") == "relu", "only the ReLU activation is supported"),
        (hf.get("enable_bias", True), "enable_bias=False is not supported"),
        (hf.get("layer_norm_elementwise_affine", True), "non-affine LayerNorm is not supported"),
        (not hf.get("_remove_final_layer_norm", False), "_remove_final_layer_norm is not supported"),
        (hf.get("tie_word_embeddings", True), "an untied LM head is not supported"),
    ]
    for ok, msg in checks:
        if not ok:
            raise ConfigurationError(msg)
    mp = hf.get("max_position_embeddings", 2048)
    return OPTConfig(vocab_size=hf["vocab_size"], d_model=d, n_heads=hf["num_attention_heads"],
                     n_blocks=hf["num_hidden_layers"], seq_len=seq_len or mp, dtype="f32",
                     max_positions=mp).validate()


def config_to_hf(cfg: OPTConfig) -> dict:
    return {"model_type": "opt", "architectures": ["OPTForCausalLM"], "vocab_size": cfg.vocab_size,
            "hidden_size": cfg.d_model, "num_attention_heads": cfg.n_heads, "num_hidden_layers": cfg.n_blocks,
            "ffn_dim": 4 * cfg.d_model, "max_position_embeddings": cfg.max_positions,
            "word_embed_proj_dim": cfg.d_model, "do_layer_norm_before": True, "activation_function": "relu",
            "enable_bias": True, "layer_norm_elementwise_affine": True, "tie_word_embeddings": True}


def _get(sd, name, shape):
    if name not in sd:
        raise ConfigurationError(f"checkpoint lacks {name}")
    a = np.asarray(sd[name], dtype=np.float32)
    if a.shape != tuple(shape):
        raise DimensionError(f"{name}: checkpoint shape {a.shape} != expected {tuple(shape)}")
    return a


def master_from_hf(sd, cfg: OPTConfig) -> np.ndarray:
    """Flat fp32 master (key order) from a HF state dict of numpy arrays
    (or anything np.asarray accepts, e.g. CPU torch tensors)."""
    if "lm_head.weight" in sd and "model.decoder.embed_tokens.weight" in sd:
        if not np.array_equal(np.asarray(sd["lm_head.weight"], dtype=np.float32),
                              np.asarray(sd["model.decoder.embed_tokens.weight"], dtype=np.float32)):
            raise ConfigurationError("lm_head.weight differs from embed_tokens.weight (untied head)")
    layouts = model_layout(cfg)
    out = np.empty(sum(b.elem_count for b in layouts), dtype=np.float32)

    def put(bl, name, arr):
        k = bl.key(name)
        out[k:k + arr.size] = arr.reshape(-1)

    emb, head = layouts[0], layouts[-1]
    put(emb, "tok_emb", _get(sd, _PFX + "embed_tokens.weight", emb.shapes["tok_emb"]))
    put(emb, "pos_emb", _get(sd, _PFX + "embed_positions.weight", emb.shapes["pos_emb"]))
    for i, bl in enumerate(layouts[1:-1]):
        for ours, hf, tr in _LAYER_MAP:
            shp = bl.shapes[ours]
            a = _get(sd, f"{_PFX}layers.{i}.{hf}", shp[::-1] if tr else shp)
            put(bl, ours, np.ascontiguousarray(a.T) if tr else a)
    put(head, "lnf_g", _get(sd, _PFX + "final_layer_norm.weight", (cfg.d_model,)))
    put(head, "lnf_b", _get(sd, _PFX + "final_layer_norm.bias", (cfg.d_model,)))
    return out


def hf_from_master(master: np.ndarray, cfg: OPTConfig) -> dict:
    """HF state dict (numpy fp32, lm_head tied) from a flat master."""
    layouts = model_layout(cfg)
    sd = {}

    def get(bl, name):
        k = bl.key(name)
        return master[k:k + bl.size(name)].reshape(bl.shapes[name])

    emb, head = layouts[0], layouts[-1]
    sd[_PFX + "embed_tokens.weight"] = get(emb, "tok_emb").copy()
    sd[_PFX + "embed_positions.weight"] = get(emb, "pos_emb").copy()
    sd[_PFX + "final_layer_norm.weight"] = get(head, "lnf_g").copy()
    sd[_PFX + "final_layer_norm.bias"] = get(head, "lnf_b").copy()
    for i, bl in enumerate(layouts[1:-1]):
        for ours, hf, tr in _LAYER_MAP:
            a = get(bl, ours)
            sd[f"{_PFX}layers.{i}.{hf}"] = np.ascontiguousarray(a.T) if tr else a.copy()
    sd["lm_head.weight"] = sd[_PFX + "embed_tokens.weight"]
    return sd


def read_hf_dir(path: str) -> tuple[dict, dict]:
    """(config.json dict, state dict of numpy fp32 arrays) from a local HF
    model directory."""
    with open(os.path.join(path, "config.json")) as f:
        hf = json.load(f)
    idx = os.path.join(path, "model.safetensors.index.json")
    single = os.path.join(path, "model.safetensors")
    sd = {}
    if os.path.exists(idx) or os.path.exists(single):
        from safetensors.numpy import load_file

        files = [single] if os.path.exists(single) else sorted(
            {os.path.join(path, f) for f in json.load(open(idx))["weight_map"].values()})
        for fn in files:
            for k, v in load_file(fn).items():
                sd[k] = v.astype(np.float32, copy=False)
    elif os.path.exists(os.path.join(path, "pytorch_model.bin")):
        import torch

        raw = torch.load(os.path.join(path, "pytorch_model.bin"), map_location="cpu", weights_only=True)
        sd = {k: v.float().numpy() for k, v in raw.items()}
    else:
        raise ConfigurationError(f"{path}: no model.safetensors(.index.json) or pytorch_model.bin")
    return hf, sd


def load_pretrained(path: str, seq_len: int | None = None, device=None, directions=None):
    """DeviceStore holding a local HF OPT checkpoint (fp32 master)."""
    import torch

    from .engine import MINUS, PLUS, DeviceStore

    hf, sd = read_hf_dir(path)
    cfg = config_from_hf(hf, seq_len)
    master = master_from_hf(sd, cfg)
    store = DeviceStore(cfg, init_seed=0, device=device, init="none", directions=directions or (PLUS, MINUS))
    store.theta.copy_(torch.from_numpy(master))
    return store


def save_pretrained(store, path: str) -> None:
    """Write the (flushed) master as a HF directory: config.json +
    model.safetensors (fp32, tied head saved once as embed_tokens)."""
    from safetensors.numpy import save_file

    if getattr(store, "unflushed", False):
        from .errors import ProtocolError

        raise ProtocolError("save_pretrained of a master with a deferred update: call flush() first")
    cfg = store.config
    if cfg.arch != "opt":
        raise ConfigurationError("save_pretrained needs an OPTConfig store")
    os.makedirs(path, exist_ok=True)
    sd = hf_from_master(store.theta.detach().cpu().numpy(), cfg)
    sd.pop("lm_head.weight")
    save_file(sd, os.path.join(path, "model.safetensors"), metadata={"format": "pt"})
    with open(os.path.join(path, "config.json"), "w") as f:
        json.dump(config_to_hf(cfg), f, indent=1)
