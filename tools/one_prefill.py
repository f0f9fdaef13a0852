"""One prefill of `model` at L tokens (for ncu launch lists): python tools/one_prefill.py 7b 4000 [layers]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu  # noqa: E402

name, L = sys.argv[1], int(sys.argv[2])
s = SHAPES[name]
if len(sys.argv) > 3:
    s = s.replace(n_layers=int(sys.argv[3]))
with MeshGpu(0, kv_pool_bytes=40 << 30) as g:
    g.create_instance(1, s, seed=1)
    g.kv_resize(1, 0, 2 * (L + 64) * s.kv_bytes_per_token)
    g.step(1, prefill=0, prefill_len=L)
    g.step(1, prefill=1, prefill_len=L)
