"""Independent Llama implementation (HuggingFace transformers) loaded with the
oracle's weights, float64 CPU. Used only as a pin for oracle/model.py."""
import numpy as np
import torch
from transformers import LlamaConfig, LlamaForCausalLM


def hf_model(model):
    c = model.cfg
    hc = LlamaConfig(vocab_size=c.vocab, hidden_size=c.hidden, intermediate_size=c.ffn,
                     num_hidden_layers=model.n_layers, num_attention_heads=c.q_heads,
                     num_key_value_heads=c.kv_heads, head_dim=c.head_dim, rms_norm_eps=c.rms_eps,
                     rope_theta=c.rope_theta, tie_word_embeddings=False,
                     max_position_embeddings=4096, attn_implementation="eager")
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
    return hf


def hf_logits_and_hidden(hf, tokens):
    with torch.no_grad():
        out = hf(torch.tensor([list(tokens)]), output_hidden_states=True)
    return out.logits[0].numpy(), out.hidden_states[-1][0].numpy()
