"""Generates tests/golden/llama_hf.json: Hugging Face transformers
LlamaForCausalLM (fp32, CPU) logits on the repo's deterministic weights.

This pins the CPU numeric oracle (oracle/llama_ref.c, round_act = 0 mode) to
an independent, widely used Llama implementation: same weights (the
generator of csrc/gpu/model.cuh, read element by element through
ora_weight), same prompt tokens, HF's own RMSNorm / RoPE / GQA / SwiGLU code.
The reference artifact has no model arithmetic of its own, so
this is the logits oracle's anchor. Run once in the dev container (needs
transformers); the JSON is committed and the test does not import HF.

    python tests/golden/make_llama_golden.py
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import llama_oracle as ora  # noqa: E402
from paper_2507_00507_b200.gpu import SHAPES  # noqa: E402

T_EMB, T_WQ, T_WK, T_WV, T_WO, T_WGATE, T_WUP, T_WDOWN, T_LM, T_GATTN, T_GMLP, T_GFINAL = range(12)
SEED = 7
PROMPT_LEN = 40


def tensor(seed, t, layer, rows, cols=None):
    n = rows * (cols or 1)
    w = ora.lib().ora_weight
    v = np.fromiter((w(seed, t, layer, i) for i in range(n)), dtype=np.float32, count=n)
    return torch.from_numpy(v.reshape(rows, cols) if cols else v)


def build_hf(shape, seed):
    from transformers import LlamaConfig, LlamaForCausalLM

    cfg = LlamaConfig(vocab_size=shape.vocab, hidden_size=shape.d_model, intermediate_size=shape.d_ff,
                      num_hidden_layers=shape.n_layers, num_attention_heads=shape.n_heads,
                      num_key_value_heads=shape.n_kv_heads, head_dim=shape.d_head,
                      max_position_embeddings=shape.max_seq_len, rms_norm_eps=shape.rms_eps,
                      rope_theta=shape.rope_theta, tie_word_embeddings=bool(shape.tied), attention_bias=False,
                      mlp_bias=False, torch_dtype=torch.float32)
    m = LlamaForCausalLM(cfg).eval()
    d, qd, kd, ff = shape.d_model, shape.n_heads * shape.d_head, shape.n_kv_heads * shape.d_head, shape.d_ff
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(tensor(seed, T_EMB, 0, shape.vocab, d))
        for l, layer in enumerate(m.model.layers):
            layer.self_attn.q_proj.weight.copy_(tensor(seed, T_WQ, l, qd, d))
            layer.self_attn.k_proj.weight.copy_(tensor(seed, T_WK, l, kd, d))
            layer.self_attn.v_proj.weight.copy_(tensor(seed, T_WV, l, kd, d))
            layer.self_attn.o_proj.weight.copy_(tensor(seed, T_WO, l, d, qd))
            layer.mlp.gate_proj.weight.copy_(tensor(seed, T_WGATE, l, ff, d))
            layer.mlp.up_proj.weight.copy_(tensor(seed, T_WUP, l, ff, d))
            layer.mlp.down_proj.weight.copy_(tensor(seed, T_WDOWN, l, d, ff))
            layer.input_layernorm.weight.copy_(tensor(seed, T_GATTN, l, d))
            layer.post_attention_layernorm.weight.copy_(tensor(seed, T_GMLP, l, d))
        m.model.norm.weight.copy_(tensor(seed, T_GFINAL, 0, d))
        if not shape.tied:
            m.lm_head.weight.copy_(tensor(seed, T_LM, 0, shape.vocab, d))
    return m


def main():
    out = {"generator": "transformers.LlamaForCausalLM fp32 CPU", "seed": SEED, "cases": []}
    import transformers

    out["transformers"] = transformers.__version__
    for name in ["tiny", "tiny128"]:
        shape = SHAPES[name]
        m = build_hf(shape, SEED)
        toks = [ora.prompt_token(SEED, 3, p, shape.vocab) for p in range(PROMPT_LEN)]
        with torch.no_grad():
            logits = m(torch.tensor([toks])).logits[0].float().numpy()
        keep = [0, 1, PROMPT_LEN // 2, PROMPT_LEN - 1]
        out["cases"].append({
            "shape": name,
            "prompt": toks,
            "argmax": [int(i) for i in logits.argmax(-1)],
            "positions": keep,
            "logits": [[round(float(x), 6) for x in logits[p]] for p in keep],
            "max_abs_logit": float(np.abs(logits).max()),
        })
        print(name, "argmax head", out["cases"][-1]["argmax"][:8])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "llama_hf.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
