"""Host-side cost of issuing prefill / decode steps through the C ABI versus
their device time (not the bench)."""
import sys, time, json
sys.path.insert(0, '.')
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu

name = sys.argv[1] if len(sys.argv) > 1 else '1b'
L = int(sys.argv[2]) if len(sys.argv) > 2 else 400
s = SHAPES[name]
with MeshGpu(0, kv_pool_bytes=20 << 30) as g:
    g.create_instance(1, s, seed=1)
    g.kv_resize(1, 0, 40 * (L + 64) * s.kv_bytes_per_token)
    g.step(1, prefill=0, prefill_len=L)
    n = 30
    dev = 0.0
    t0 = time.perf_counter()
    for r in range(1, n + 1):
        g.step(1, prefill=r, prefill_len=L)
        dev += g.stats()['last_step_ms']
    wall = (time.perf_counter() - t0) * 1e3 / n
    print(json.dumps(dict(model=name, L=L, prefill_wall_ms=wall, prefill_dev_ms=dev / n)))
