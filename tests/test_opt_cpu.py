"""Real-OPT compatibility, host side: the HF <-> master
mapping, the file reader, config checks, and the plain-torch OPT checker
pinned to transformers' own OPTForCausalLM."""

import json

import numpy as np
import pytest
import torch

from paper_2507_03211_b200 import opt
from paper_2507_03211_b200.errors import ConfigurationError, DimensionError
from paper_2507_03211_b200.model import ModelConfig, OPTConfig, model_layout, real_opt_config
from tests.opt_ref import ce_f64, opt_forward_ref, random_opt_state

transformers = pytest.importorskip("transformers")

TINY = dict(vocab_size=96, hidden_size=64, num_attention_heads=4, num_hidden_layers=2, ffn_dim=256,
            max_position_embeddings=32, word_embed_proj_dim=64)


def _hf_model(seed=0):
    torch.manual_seed(seed)
    c = transformers.OPTConfig(**TINY, attn_implementation="eager")
    m = transformers.OPTForCausalLM(c).eval()
    with torch.no_grad():    # non-trivial LN / bias values
        for n, p in m.named_parameters():
            if "layer_norm" in n or n.endswith("bias"):
                p.add_(0.05 * torch.randn_like(p))
    return c, m


def test_reference_forward_matches_transformers():
    c, m = _hf_model()
    ids = torch.randint(0, 96, (2, 20), generator=torch.Generator().manual_seed(1))
    with torch.no_grad():
        want = m(input_ids=ids).logits
    sd = {k: v.numpy() for k, v in m.state_dict().items()}
    got = opt_forward_ref(sd, 4, ids)
    torch.testing.assert_close(got, want, rtol=1e-5, atol=1e-5)
    # HF's own shifted-label loss == ce_f64 over the shifted positions
    with torch.no_grad():
        hf_loss = m(input_ids=ids, labels=ids).loss.item()
    assert abs(ce_f64(want[:, :-1], ids[:, 1:]) - hf_loss) < 1e-5


def test_master_roundtrip_and_layout():
    c, m = _hf_model()
    sd = {k: v.numpy() for k, v in m.state_dict().items()}
    cfg = opt.config_from_hf(c.to_dict(), seq_len=16)
    assert isinstance(cfg, OPTConfig) and cfg.max_positions == 32
    assert cfg.param_count() == sum(p.numel() for p in m.parameters())
    master = opt.master_from_hf(sd, cfg)
    assert master.size == cfg.param_count()
    back = opt.hf_from_master(master, cfg)
    assert set(back) == set(sd)
    for k in sd:
        assert np.array_equal(back[k], sd[k]), k
    # weights are stored (d_in, d_out): wq block == q_proj.weight.T
    bl = model_layout(cfg)[1]
    k = bl.key("wq")
    assert np.array_equal(master[k:k + 64 * 64].reshape(64, 64),
                          sd["model.decoder.layers.0.self_attn.q_proj.weight"].T)


def test_read_hf_dir_safetensors_and_bin(tmp_path):
    c, m = _hf_model()
    m.save_pretrained(tmp_path / "st", safe_serialization=True)
    hf, sd = opt.read_hf_dir(str(tmp_path / "st"))
    cfg = opt.config_from_hf(hf, 16)
    want = opt.master_from_hf({k: v.numpy() for k, v in m.state_dict().items()}, cfg)
    assert np.array_equal(opt.master_from_hf(sd, cfg), want)
    (tmp_path / "bin").mkdir()
    torch.save(m.state_dict(), tmp_path / "bin" / "pytorch_model.bin")
    (tmp_path / "bin" / "config.json").write_text(json.dumps(c.to_dict()))
    _, sd2 = opt.read_hf_dir(str(tmp_path / "bin"))
    assert np.array_equal(opt.master_from_hf(sd2, cfg), want)


@pytest.mark.parametrize("bad,msg", [({"do_layer_norm_before": False}, "350m"),
                                     ({"word_embed_proj_dim": 32}, "word_embed_proj_dim"),
                                     ({"activation_function": "gelu"}, "ReLU"),
                                     ({"ffn_dim": 100}, "ffn_dim")])
def test_config_refusals(bad, msg):
    hf = dict(TINY, **bad)
    with pytest.raises(ConfigurationError, match=msg):
        opt.config_from_hf(hf)


def test_mapping_errors():
    cfg = OPTConfig(96, 64, 4, 2, 16, "f32", max_positions=32).validate()
    sd = random_opt_state(96, 64, 4, 2, 32)
    sd2 = dict(sd)
    sd2["lm_head.weight"] = sd["lm_head.weight"] + 1
    with pytest.raises(ConfigurationError, match="untied"):
        opt.master_from_hf(sd2, cfg)
    sd3 = dict(sd)
    del sd3["model.decoder.layers.1.fc2.bias"]
    with pytest.raises(ConfigurationError, match="lacks"):
        opt.master_from_hf(sd3, cfg)
    sd4 = dict(sd)
    sd4["model.decoder.layers.0.fc1.weight"] = sd["model.decoder.layers.0.fc1.weight"][:, :32]
    with pytest.raises(DimensionError):
        opt.master_from_hf(sd4, cfg)
    with pytest.raises(ConfigurationError, match="max_positions"):
        OPTConfig(96, 64, 4, 2, 64, "f32", max_positions=32).validate()


def test_config_dict_dispatch_and_real_sizes():
    c = real_opt_config("opt-1.3b", 512)
    assert ModelConfig.from_dict(c.to_dict()) == c
    assert c.param_count() == 1_315_758_080          # facebook/opt-1.3b parameter count
    assert real_opt_config("opt-125m", 2048).param_count() == 125_239_296
