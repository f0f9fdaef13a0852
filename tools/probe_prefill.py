"""Prefill step time (CUDA events, whole step incl. embed/norm/GEMMs/attention/lm_head)
and achieved TF/s for each model at L tokens, median of N prefills. MESH_PF_ATTN=mma
selects the mma.sync attention for an A/B. usage: python tools/probe_prefill.py 1b,7b 1024"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu  # noqa: E402


def run(name, L, n=8):
    s = SHAPES[name]
    with MeshGpu(0, kv_pool_bytes=40 << 30) as g:
        g.create_instance(1, s, seed=1)
        g.kv_resize(1, 0, (n + 2) * (L + 64) * s.kv_bytes_per_token)
        ms = []
        for r in range(n):
            g.step(1, prefill=r, prefill_len=L)
            ms.append(g.stats()["last_kernel_ms"])
    pf = sorted(ms)[len(ms) // 2]
    flops = 2 * L * s.p_body + 2 * s.vocab * s.d_model + 2 * s.n_layers * s.n_heads * s.d_head * L * (L + 1)
    attn = 2 * s.n_layers * s.n_heads * s.d_head * L * (L + 1)
    return dict(model=name, L=L, ms=round(pf, 4), TFLOPs=round(flops / pf / 1e9, 1), attn_share_flops=round(attn / flops, 3),
                attn=os.environ.get("MESH_PF_ATTN", "tc"))


if __name__ == "__main__":
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    for m in (sys.argv[1] if len(sys.argv) > 1 else "1b,3b,7b,13b").split(","):
        print(json.dumps(run(m, L)), flush=True)
