"""Quick device-time probe of the decode/prefill kernels (not the bench)."""
import sys, time, json
sys.path.insert(0, '.')
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu

def run(name, B=8, ctx=1024, iters=20, pf_len=512):
    s = SHAPES[name]
    out = {}
    with MeshGpu(0, kv_pool_bytes=40 << 30) as g:
        g.create_instance(1, s, seed=1)
        g.kv_resize(1, 0, (B + 2) * (ctx + 64) * s.kv_bytes_per_token)
        t0 = time.time()
        pfs = []
        for r in range(B):
            g.step(1, prefill=r, prefill_len=ctx)
            pfs.append(g.stats()['last_step_ms'])
        pf = sorted(pfs)[len(pfs) // 2]  # median of the B prefills
        rids = list(range(B))
        ms = g.bench_decode(1, rids, iters)
        W = s.weight_bytes_streamed
        kv = B * ctx * s.kv_bytes_per_token + B * s.kv_bytes_per_token
        bytes_ = W + kv + B * s.d_model * 2
        out = dict(model=name, B=B, ctx=ctx, decode_ms=ms, decode_GBps=bytes_ / ms / 1e6,
                   frac=bytes_ / ms / 1e6 / 6539.2, prefill_ms_ctx=pf)
        # prefill flops for L=ctx
        L = ctx
        flops = 2 * L * s.p_body + 2 * s.vocab * s.d_model + 2 * s.n_layers * s.n_heads * s.d_head * L * (L + 1)
        out['prefill_TFLOPs'] = flops / pf / 1e9
    print(json.dumps(out))

import os
ITERS=int(os.environ.get('PROBE_ITERS','20'))
for name in sys.argv[1:] or ['1b']:
    run(name, iters=ITERS)
