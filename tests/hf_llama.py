"""Independent third-party forward for pinning the oracle: Hugging Face
`transformers` LlamaForCausalLM (transformers 5.5, eager attention), run in
fp64 on CPU with the SAME bf16 weights and the same post-RoPE prefix KV.

Test infrastructure only.  The point is that RoPE pairing (rotate-half over
(i, i + d/2)), GQA head mapping (query head h reads kv head h // n_rep),
RMSNorm placement, the SiLU(gate) * up order and the position offsets come
from an implementation this repo did not write; `oracle/vc_oracle.c` and the
CUDA engine are then compared against it (tests/test_oracle_hf.py,
tests/test_model_parity.py)."""
from __future__ import annotations

import numpy as np


def _f64(bits) -> "np.ndarray":
    return (np.asarray(bits, np.uint32) << 16).view(np.float32).astype(np.float64)


def build(shape, w):
    """LlamaForCausalLM (fp64) carrying the logical bf16 weights `w`
    (layouts of oracle/vc_oracle.h)."""
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    cfg = LlamaConfig(vocab_size=shape.vocab, hidden_size=shape.hidden, intermediate_size=shape.ffn,
                      num_hidden_layers=shape.layers, num_attention_heads=shape.n_q,
                      num_key_value_heads=shape.n_kv, head_dim=shape.d_head,
                      rope_theta=float(shape.rope_theta), rms_norm_eps=float(shape.rms_eps),
                      tie_word_embeddings=False, attention_bias=False, mlp_bias=False,
                      max_position_embeddings=1 << 20)
    cfg._attn_implementation = "eager"
    with torch.device("meta"):
        m = LlamaForCausalLM(cfg)
    m = m.to_empty(device="cpu").to(torch.float64)
    nq, nkv, d = shape.n_q, shape.n_kv, shape.d_head
    t = lambda a: torch.from_numpy(_f64(a))  # noqa: E731
    sd = {"model.embed_tokens.weight": t(w["embed"]), "model.norm.weight": t(w["final_norm"]),
          "lm_head.weight": t(w["lm_head"])}
    for l in range(shape.layers):
        p = f"model.layers.{l}."
        qkv = np.asarray(w["wqkv"][l]).reshape((nq + 2 * nkv) * d, shape.hidden)
        sd[p + "self_attn.q_proj.weight"] = t(qkv[: nq * d])
        sd[p + "self_attn.k_proj.weight"] = t(qkv[nq * d:(nq + nkv) * d])
        sd[p + "self_attn.v_proj.weight"] = t(qkv[(nq + nkv) * d:])
        sd[p + "self_attn.o_proj.weight"] = t(w["wo"][l])
        sd[p + "mlp.gate_proj.weight"] = t(w["wgate"][l])
        sd[p + "mlp.up_proj.weight"] = t(w["wup"][l])
        sd[p + "mlp.down_proj.weight"] = t(w["wdown"][l])
        sd[p + "input_layernorm.weight"] = t(w["attn_norm"][l])
        sd[p + "post_attention_layernorm.weight"] = t(w["mlp_norm"][l])
    missing, unexpected = m.load_state_dict(sd, strict=False)
    missing = [k for k in missing if "rotary_emb" not in k]
    assert not missing and not unexpected, (missing, unexpected)
    # the rotary buffers were created on the meta device: recompute them
    rot = m.model.rotary_emb
    inv = 1.0 / (float(shape.rope_theta) ** (torch.arange(0, d, 2, dtype=torch.float64) / d))
    rot.inv_freq = inv
    if hasattr(rot, "original_inv_freq"):
        rot.original_inv_freq = inv
    m.eval()
    return m


def forward(model, shape, k_bits, v_bits, tokens):
    """Logits [n][vocab] (fp64) of `tokens` at positions T..T+n-1 after a
    prefix whose post-RoPE K/V are k_bits / v_bits ([layers][n_kv][T][d] bf16)."""
    import torch
    from transformers import DynamicCache

    T = k_bits.shape[2]
    cache = DynamicCache(ddp_cache_data=[(torch.from_numpy(_f64(k_bits[l]))[None],
                                          torch.from_numpy(_f64(v_bits[l]))[None])
                                         for l in range(shape.layers)], config=model.config)
    ids = torch.tensor([list(tokens)], dtype=torch.long)
    pos = torch.arange(T, T + len(tokens), dtype=torch.long)[None]
    with torch.no_grad():
        out = model(input_ids=ids, position_ids=pos, past_key_values=cache, use_cache=True)
    return out.logits[0].numpy()
