"""Summarise a MESH_GPU_TRACE dump of the decode kernel (CTA 0 phase timeline)."""
import collections, sys
NAMES = {1: "phase-begin", 2: "operands", 3: "stages-done", 4: "epilogue", 5: "barrier", 6: "attn-begin", 7: "attn-end"}
for path in sys.argv[1:]:
    rows = [(a, b % 100) for a, b in (tuple(map(int, l.split())) for l in open(path) if l.strip())]
    t0 = rows[0][0]
    agg = collections.defaultdict(float); cnt = collections.Counter()
    for (ta, ga), (tb, gb) in zip(rows, rows[1:]):
        agg[(ga, gb)] += (tb - ta) / 1000; cnt[(ga, gb)] += 1
    print(path, "CTA0 span us", (rows[-1][0] - t0) / 1000)
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
        print(f"   {NAMES[k[0]]:>12} -> {NAMES[k[1]]:<12} total {v:8.1f} us  n={cnt[k]:4d}  avg {v / cnt[k]:6.2f}")
