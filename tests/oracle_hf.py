"""Independent Llama implementation (HuggingFace transformers) loaded with the
oracle's weights, float64 CPU (RoPE angles in float64 too). Used only as a pin
for oracle/model.py (target forward) and oracle/engine.py (the S0 draft chain)."""
import numpy as np
import torch
from transformers import LlamaConfig, LlamaForCausalLM


def hf_model(model):
    c = model.cfg
    hc = LlamaConfig(vocab_size=c.vocab, hidden_size=c.hidden, intermediate_size=c.ffn,
                     num_hidden_layers=model.n_layers, num_attention_heads=c.q_heads,
                     num_key_value_heads=c.kv_heads, head_dim=c.head_dim, rms_norm_eps=c.rms_eps,
                     rope_theta=c.rope_theta, tie_word_embeddings=False,
                     max_position_embeddings=4096, attn_implementation="sdpa")
    hf = LlamaForCausalLM(hc).to(torch.float64).eval()
    sd = {"model.embed_tokens.weight": model.embed, "lm_head.weight": model.head,
          "model.norm.weight": np.ones(c.hidden)}
    for l, lw in enumerate(model.layers):
        p = f"model.layers.{l}."
        sd[p + "self_attn.q_proj.weight"] = lw.wq
        sd[p + "self_attn.k_proj.weight"] = lw.wk
        sd[p + "self_attn.v_proj.weight"] = lw.wv
        sd[p + "self_attn.o_proj.weight"] = lw.wo
        sd[p + "mlp.gate_proj.weight"] = lw.wg
        sd[p + "mlp.up_proj.weight"] = lw.wu
        sd[p + "mlp.down_proj.weight"] = lw.wd
        sd[p + "input_layernorm.weight"] = np.ones(c.hidden)
        sd[p + "post_attention_layernorm.weight"] = np.ones(c.hidden)
    hf.load_state_dict({k: torch.from_numpy(np.asarray(v, dtype=np.float64)) for k, v in sd.items()})
    f64_rotary(hf.model, c.rope_theta, c.head_dim)
    f64_norms(hf)
    return hf


def hf_logits_and_hidden(hf, tokens):
    with torch.no_grad():
        out = hf(torch.tensor([list(tokens)]), output_hidden_states=True)
    return out.logits[0].numpy(), out.hidden_states[-1][0].numpy()


def f64_rotary(hf_inner, theta, hd):
    """Replace HF's rotary embedding forward (which evaluates the angles in
    float32) by the same default Llama RoPE -- inv_freq_i = theta^(-2i/hd),
    emb = [freqs, freqs] (rotate_half layout) -- evaluated in float64, so the
    HF pins agree with the float64 oracle to rounding (~1e-12), not ~1e-7."""
    inv = 1.0 / (float(theta) ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))

    def fwd(x, position_ids):
        freqs = position_ids[..., None].to(torch.float64) * inv
        emb = torch.cat((freqs, freqs), dim=-1)
        return emb.cos().to(x.dtype), emb.sin().to(x.dtype)

    hf_inner.rotary_emb.forward = fwd


def f64_norms(hf):
    """HF's LlamaRMSNorm upcasts to float32 only (`hidden_states.to(torch.float32)`);
    keep its formula w * x * rsqrt(mean(x^2) + eps) but in the model's float64."""
    from transformers.models.llama.modeling_llama import LlamaRMSNorm
    for mod in hf.modules():
        if isinstance(mod, LlamaRMSNorm):
            mod.forward = (lambda h, mod=mod: mod.weight * (h * torch.rsqrt(h.pow(2).mean(-1, keepdim=True)
                                                                             + mod.variance_epsilon)))


def hf_draft_layer(model):
    """The draft head's transformer layer TL as a one-layer
    HuggingFace LlamaModel (independent Llama decoder-layer implementation)
    loaded with the oracle's draft weights, float64, float64 RoPE."""
    from transformers import LlamaModel
    c = model.cfg
    hc = LlamaConfig(vocab_size=c.vocab, hidden_size=c.hidden, intermediate_size=c.ffn,
                     num_hidden_layers=1, num_attention_heads=c.q_heads,
                     num_key_value_heads=c.kv_heads, head_dim=c.head_dim, rms_norm_eps=c.rms_eps,
                     rope_theta=c.rope_theta, max_position_embeddings=4096, attn_implementation="sdpa")
    hf = LlamaModel(hc).to(torch.float64).eval()
    d = model.draft
    sd = {"embed_tokens.weight": model.embed, "norm.weight": np.ones(c.hidden),
          "layers.0.self_attn.q_proj.weight": d.wq, "layers.0.self_attn.k_proj.weight": d.wk,
          "layers.0.self_attn.v_proj.weight": d.wv, "layers.0.self_attn.o_proj.weight": d.wo,
          "layers.0.mlp.gate_proj.weight": d.wg, "layers.0.mlp.up_proj.weight": d.wu,
          "layers.0.mlp.down_proj.weight": d.wd,
          "layers.0.input_layernorm.weight": np.ones(c.hidden),
          "layers.0.post_attention_layernorm.weight": np.ones(c.hidden)}
    hf.load_state_dict({k: torch.from_numpy(np.asarray(v, dtype=np.float64)) for k, v in sd.items()})
    f64_rotary(hf, c.rope_theta, c.head_dim)
    f64_norms(hf)
    return hf


def _last_layer_output(inner, run):
    """Run `run()` and return the output of inner.layers[-1] (the pre-final-norm
    hidden states), captured with a forward hook."""
    got = {}

    def hook(_mod, _inp, out):
        got["h"] = out[0] if isinstance(out, tuple) else out

    h = inner.layers[-1].register_forward_hook(hook)
    try:
        with torch.no_grad():
            run()
    finally:
        h.remove()
    return got["h"][0].numpy()


def hf_layer_outputs(hf_draft, inputs_embeds, positions):
    """Pre-norm outputs of the one-layer model over a causal sequence of input
    vectors at explicit RoPE positions."""
    x = torch.from_numpy(np.asarray(inputs_embeds, dtype=np.float64))[None]
    pos = torch.tensor([list(positions)], dtype=torch.long)
    return _last_layer_output(hf_draft, lambda: hf_draft(inputs_embeds=x, position_ids=pos))


def hf_prenorm_hidden(hf, tokens):
    """Target pre-final-norm hidden states H (the paper's h) of a
    token sequence at positions 0..len-1."""
    ids = torch.tensor([list(tokens)])
    return _last_layer_output(hf.model, lambda: hf(ids))
