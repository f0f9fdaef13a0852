"""Per-barrier CTA arrival spread from MESH_GPU_TRACE=<f> (<f>.arrive): which phases have stragglers."""
import sys
import numpy as np
rows = [list(map(int, l.split())) for l in open(sys.argv[1]) if l.strip()]
a = np.array([r for r in rows if any(r)], dtype=np.float64)
a = a[:, :]
# barriers per layer: QKV -> attention has none (per-KV-head-group counters), so the
# first barrier of a layer closes QKV + attention
names = ["embed"] + [f"L{l}.{p}" for l in range(200) for p in ["qkv+attn", "o", "gu", "down"]]
prev_release = a[0].max()
tot = {}
for i in range(1, a.shape[0]):
    arr = a[i]
    ph = names[i].split(".")[-1]
    dur_max = (arr.max() - prev_release) / 1e3
    dur_med = (np.median(arr) - prev_release) / 1e3
    tot.setdefault(ph, [0, 0, 0])
    tot[ph][0] += dur_max; tot[ph][1] += dur_med; tot[ph][2] += 1
    prev_release = arr.max()
print("phase   n   sum(max) us  sum(median) us  avg max  avg med   (max = slowest CTA)")
for ph, (mx, md, n) in tot.items():
    print(f"{ph:6s} {n:3d} {mx:10.1f} {md:12.1f} {mx/n:8.2f} {md/n:8.2f}")
print("span us", (a[-1].max() - a[0].min()) / 1e3)
