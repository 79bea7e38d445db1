"""Plain-torch fp32 restatement of HF transformers' OPTForCausalLM forward
(modeling_opt: OPTLearnedPositionalEmbedding offset 2, pre-LN decoder layers,
q scaled by head_dim**-0.5, causal softmax, ReLU FFN, final LayerNorm, tied
LM head).  Test infrastructure: pinned to transformers itself by
tests/test_opt_cpu.py, then used as the checker for the GPU OPT path."""

import math

import torch

P = "model.decoder."


def opt_forward_ref(sd: dict, n_heads: int, ids: torch.Tensor) -> torch.Tensor:
    """Logits [B, T, V] (fp32) for token ids [B, T] from a HF state dict."""
    f = {k: torch.as_tensor(v, dtype=torch.float32) for k, v in sd.items()}
    B, T = ids.shape
    emb = f[P + "embed_tokens.weight"]
    d = emb.shape[1]
    hd = d // n_heads
    x = emb[ids] + f[P + "embed_positions.weight"][torch.arange(T) + 2][None]
    n_layers = 1 + max(int(k.split(".")[3]) for k in f if k.startswith(P + "layers."))
    mask = torch.full((T, T), float("-inf")).triu(1)
    for i in range(n_layers):
        p = f"{P}layers.{i}."
        lin = lambda h, n: h @ f[p + n + ".weight"].t() + f[p + n + ".bias"]  # noqa: E731
        h = torch.nn.functional.layer_norm(x, (d,), f[p + "self_attn_layer_norm.weight"],
                                           f[p + "self_attn_layer_norm.bias"], 1e-5)
        q = lin(h, "self_attn.q_proj") * (hd ** -0.5)
        k = lin(h, "self_attn.k_proj")
        v = lin(h, "self_attn.v_proj")
        sh = lambda t: t.view(B, T, n_heads, hd).transpose(1, 2)  # noqa: E731
        s = sh(q) @ sh(k).transpose(-1, -2) + mask
        a = torch.softmax(s, dim=-1) @ sh(v)
        x = x + lin(a.transpose(1, 2).reshape(B, T, d), "self_attn.out_proj")
        h = torch.nn.functional.layer_norm(x, (d,), f[p + "final_layer_norm.weight"],
                                           f[p + "final_layer_norm.bias"], 1e-5)
        x = x + lin(torch.relu(lin(h, "fc1")), "fc2")
    x = torch.nn.functional.layer_norm(x, (d,), f[P + "final_layer_norm.weight"], f[P + "final_layer_norm.bias"],
                                       1e-5)
    return x @ emb.t()


def ce_f64(logits: torch.Tensor, targets: torch.Tensor) -> float:
    """Mean CE over all positions in f64 (the engine's loss, model.py:357-372)."""
    l64 = logits.double().reshape(-1, logits.shape[-1])
    return float(torch.nn.functional.cross_entropy(l64, targets.reshape(-1).long()))


def random_opt_state(vocab, d, heads, layers, max_pos, seed=0, std=0.02):
    """HF-named random OPT weights (LN gains around 1) for parity tests."""
    g = torch.Generator().manual_seed(seed)
    r = lambda *s: torch.randn(*s, generator=g) * std  # noqa: E731
    sd = {P + "embed_tokens.weight": r(vocab, d), P + "embed_positions.weight": r(max_pos + 2, d),
          P + "final_layer_norm.weight": 1 + r(d) * 5, P + "final_layer_norm.bias": r(d)}
    for i in range(layers):
        p = f"{P}layers.{i}."
        for n, (o, ii) in {"self_attn.q_proj": (d, d), "self_attn.k_proj": (d, d), "self_attn.v_proj": (d, d),
                           "self_attn.out_proj": (d, d), "fc1": (4 * d, d), "fc2": (d, 4 * d)}.items():
            sd[p + n + ".weight"] = r(o, ii) * (1.0 if n != "fc2" else 0.5)
            sd[p + n + ".bias"] = r(o)
        for n in ("self_attn_layer_norm", "final_layer_norm"):
            sd[p + n + ".weight"] = 1 + r(d) * 5
            sd[p + n + ".bias"] = r(d)
    sd["lm_head.weight"] = sd[P + "embed_tokens.weight"]
    _ = math
    return {k: v.numpy() for k, v in sd.items()}
