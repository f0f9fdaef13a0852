import sys, os, json, time
sys.path.insert(0, ".")
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu
name, L, nl = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
kw = {}
for kv in sys.argv[4:]:
    k, v = kv.split("="); kw[k] = int(v)
s = SHAPES[name].replace(n_layers=nl, **kw)
with MeshGpu(0, kv_pool_bytes=8 << 30) as g:
    g.create_instance(1, s, seed=1)
    g.kv_resize(1, 0, 4 * (L + 64) * s.kv_bytes_per_token)
    t = time.time()
    g.step(1, prefill=0, prefill_len=L)
    print(name, L, nl, kw, "ok", round(time.time() - t, 3), flush=True)
