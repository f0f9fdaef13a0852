"""CTA 0 timeline of a MESH_GPU_TRACE dump (decode kernel): time between consecutive tags,
aggregated (consumer tags only)."""
import collections
import sys

NAMES = {1: "phase-begin", 2: "operands", 3: "stages-done", 4: "epilogue", 5: "barrier", 6: "attn-begin",
         7: "attn-end", 12: "attn-first-stage", 13: "attn-loop-end", 14: "attn-flushed", 15: "attn-csync",
         16: "cmb-begin", 17: "cmb-pre", 18: "cmb-arrive"}
for path in sys.argv[1:]:
    rows = [tuple(map(int, ln.split())) for ln in open(path) if ln.strip()]
    cons = [(a, b) for a, b in rows if b < 100]
    t0 = cons[0][0]
    agg = collections.defaultdict(float)
    cnt = collections.Counter()
    for (ta, ga), (tb, gb) in zip(cons, cons[1:]):
        agg[(ga, gb)] += (tb - ta) / 1000
        cnt[(ga, gb)] += 1
    print(path, "CTA0 span us", (cons[-1][0] - t0) / 1000)
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:16]:
        a, b = NAMES.get(k[0], str(k[0])), NAMES.get(k[1], str(k[1]))
        print(f"   {a:>16} -> {b:<16} total {v:8.1f} us  n={cnt[k]:4d}  avg {v / cnt[k]:6.2f}")
