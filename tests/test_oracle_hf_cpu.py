"""Pins the transformer oracle (oracle/transformer.py) to an independent
implementation: HuggingFace `transformers` LlamaForCausalLM / Qwen2ForCausalLM
(5.5.0, installed in this image), fp32, loaded with the SAME counter-based
weights (oracle.transformer.build_weights, the engine's init_weights).

The reference itself has no model (its LLM operator is a hash,
/root/reference/proj/src/evaluator.cpp:37-58), so this is what pins the math
half of the oracle: RMSNorm, RoPE (rotate-half, theta from the model card),
GQA causal attention, SwiGLU, QKV bias (Qwen2), untied LM head. The oracle's
incremental greedy decode (contiguous KV cache) must reproduce HF's full
causal forward over prompt||generated at every generated position, within
1e-5 of max |logit| (the north-star fp32 tolerance), and pick the same tokens.
"""
from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

from oracle.transformer import Decoder, build_weights, top2_margin
from paper_2603_16104_b200.engine import LLAMA3_8B, QWEN25_32B, TINY, reduced

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

FP32_TOL = 1e-5


def hf_model(m, w, **override):
    """HF model of config m whose parameters are views of the oracle's weights."""
    common = dict(vocab_size=m.vocab, hidden_size=m.d_model, intermediate_size=m.ffn_dim,
                  num_hidden_layers=m.n_layers, num_attention_heads=m.n_heads, num_key_value_heads=m.n_kv_heads,
                  head_dim=m.head_dim, rope_theta=m.rope_theta, rms_norm_eps=m.rms_eps, tie_word_embeddings=False,
                  max_position_embeddings=4096, torch_dtype=torch.float32)
    common.update(override)
    if m.qkv_bias:
        cfg = transformers.Qwen2Config(**common, use_sliding_window=False)
        cls = transformers.Qwen2ForCausalLM
    else:
        cfg = transformers.LlamaConfig(**common, attention_bias=False, mlp_bias=False)
        cls = transformers.LlamaForCausalLM
    cfg._attn_implementation = "eager"
    with torch.device("meta"):
        model = cls(cfg)
    H, Hkv, hd, F, d = m.n_heads, m.n_kv_heads, m.head_dim, m.ffn_dim, m.d_model
    t = torch.from_numpy
    sd = {"model.embed_tokens.weight": t(w.embed), "model.norm.weight": torch.ones(d), "lm_head.weight": t(w.lm_head)}
    for l, lw in enumerate(w.layers):
        p = f"model.layers.{l}."
        q, k, v = H * hd, H * hd + Hkv * hd, (H + 2 * Hkv) * hd
        sd[p + "self_attn.q_proj.weight"] = t(lw["wqkv"][:q])
        sd[p + "self_attn.k_proj.weight"] = t(lw["wqkv"][q:k])
        sd[p + "self_attn.v_proj.weight"] = t(lw["wqkv"][k:v])
        if m.qkv_bias:
            sd[p + "self_attn.q_proj.bias"] = t(lw["bqkv"][:q])
            sd[p + "self_attn.k_proj.bias"] = t(lw["bqkv"][q:k])
            sd[p + "self_attn.v_proj.bias"] = t(lw["bqkv"][k:v])
        sd[p + "self_attn.o_proj.weight"] = t(lw["wo"])
        sd[p + "mlp.gate_proj.weight"] = t(lw["wgu"][:F])
        sd[p + "mlp.up_proj.weight"] = t(lw["wgu"][F:])
        sd[p + "mlp.down_proj.weight"] = t(lw["wd"])
        sd[p + "input_layernorm.weight"] = torch.ones(d)
        sd[p + "post_attention_layernorm.weight"] = torch.ones(d)
    missing, unexpected = model.load_state_dict(sd, strict=False, assign=True)
    assert not unexpected, unexpected
    assert all("rotary" in k for k in missing), missing
    model.model.rotary_emb = type(model.model.rotary_emb)(cfg)  # materialise inv_freq off the meta device
    return model.eval()


def check_against_hf(m, prompt_len, n_new, seed, **hf_override):
    m = replace(m, fp32=True)
    w = build_weights(m)
    dec = Decoder(m, w, max_pos=prompt_len + n_new + 8)
    rng = np.random.default_rng(seed)
    prompt = rng.integers(0, m.vocab, size=prompt_len).tolist()
    toks, logits = dec.generate(prompt, n_new)
    model = hf_model(m, w, **hf_override)
    seq = torch.tensor([prompt + toks[:-1]], dtype=torch.long)
    with torch.no_grad():
        hf = model(input_ids=seq).logits[0].numpy()
    worst = 0.0
    for k in range(n_new):
        ref = hf[prompt_len - 1 + k]
        err = float(np.abs(logits[k] - ref).max() / np.abs(ref).max())
        worst = max(worst, err)
        assert err < FP32_TOL, (m.name, k, err)
        # same greedy choice unless HF's own top two are within the tolerance
        if int(np.argmax(ref)) != toks[k]:
            assert top2_margin(ref) < 2 * FP32_TOL * np.abs(ref).max()
    return worst


def test_oracle_matches_hf_llama_tiny():
    check_against_hf(TINY, 60, 6, 0)


def test_oracle_matches_hf_llama3_8b_width_full_vocab():
    """Llama-3-8B widths (d 4096, 32/8 heads, FFN 14336, vocab 128256, theta 5e5), 2 layers."""
    check_against_hf(reduced(LLAMA3_8B, 2), 40, 4, 1)


def test_oracle_matches_hf_qwen25_32b_width():
    """Qwen2.5-32B widths (d 5120, 40/8 heads, FFN 27648, QKV bias, theta 1e6, eps 1e-6), 1 layer."""
    check_against_hf(reduced(QWEN25_32B, 1, vocab=32768), 40, 4, 2)


def test_hf_check_detects_a_rope_mismatch():
    """Negative control: the comparison is sensitive (HF with another RoPE theta fails it)."""
    with pytest.raises(AssertionError):
        check_against_hf(TINY, 60, 3, 0, rope_theta=20000.0)
