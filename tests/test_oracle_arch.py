"""Pin the oracle's decoder *structure* (norm placement, RoPE convention, attention scaling,
SiLU gating, residuals, untied head) against an independent library implementation:
HuggingFace transformers' LlamaForCausalLM ("Llama2 model series"), run in
float64 with the oracle in its unrounded mode.  HF computes RMSNorm variance and the RoPE
tables in float32, so agreement is to ~1e-5 relative, far below any structural error."""
import numpy as np
import pytest
import torch

import hsgen
from oracle.decoder import Group, Weights
from oracle.numerics import exact


def hf_model(cfg, W: Weights):
    from transformers import LlamaConfig, LlamaForCausalLM
    c = LlamaConfig(hidden_size=cfg["hidden"], intermediate_size=cfg["ffn"],
                    num_attention_heads=cfg["n_heads"], num_key_value_heads=cfg["n_heads"],
                    num_hidden_layers=cfg["n_layers"], vocab_size=cfg["vocab"], rms_norm_eps=cfg["rms_eps"],
                    rope_theta=cfg["rope_theta"], max_position_embeddings=4096, tie_word_embeddings=False,
                    attention_bias=False, mlp_bias=False, hidden_act="silu", head_dim=cfg["head_dim"])
    c._attn_implementation = "eager"
    m = LlamaForCausalLM(c).double().eval()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(t(W.embed_rows(np.arange(cfg["vocab"]))))
        for l, L in enumerate(m.model.layers):
            w = W.layer(l)
            L.input_layernorm.weight.copy_(t(w["attn_norm"]))
            L.post_attention_layernorm.weight.copy_(t(w["ffn_norm"]))
            L.self_attn.q_proj.weight.copy_(t(w["wq"]))
            L.self_attn.k_proj.weight.copy_(t(w["wk"]))
            L.self_attn.v_proj.weight.copy_(t(w["wv"]))
            L.self_attn.o_proj.weight.copy_(t(w["wo"]))
            L.mlp.gate_proj.weight.copy_(t(w["wg"]))
            L.mlp.up_proj.weight.copy_(t(w["wu"]))
            L.mlp.down_proj.weight.copy_(t(w["wd"]))
        m.model.norm.weight.copy_(t(W.final_norm()))
        m.lm_head.weight.copy_(t(W.lm_head()))
    return m


@pytest.mark.parametrize("name,cfg", [
    ("mini", dict(n_layers=2, hidden=64, n_heads=2, n_kv_heads=2, head_dim=32, ffn=192, vocab=128,
                  max_seq=256, rms_eps=1e-5, rope_theta=10000.0)),
    ("tiny", hsgen.CONFIGS["tiny"]),
])
def test_oracle_matches_hf_llama_fp64(name, cfg):
    W = Weights(cfg, seed=7)
    m = hf_model(cfg, W)
    prompt = hsgen.tokens(99, 20, cfg["vocab"])
    g = Group(cfg, W, pp=2, num_blocks=16, rnd=exact)
    toks, logits = g.prefill([0], [prompt])
    seq = list(prompt)
    with torch.no_grad():
        ref = m(torch.tensor([seq])).logits[0, -1].numpy()
    assert np.allclose(logits[0], ref, rtol=1e-4, atol=1e-4 * np.abs(ref).max())
    # three cached decode steps vs full recompute in HF
    for step in range(3):
        seq.append(toks[0])
        toks, logits = g.decode([0], toks)
        with torch.no_grad():
            ref = m(torch.tensor([seq])).logits[0, -1].numpy()
        assert np.allclose(logits[0], ref, rtol=1e-4, atol=1e-4 * np.abs(ref).max()), step
