"""Print CTA 0's consumer (tags 1-7) and producer (tags 108-111) timelines for the first layers."""
import sys
rows = sorted(tuple(map(int, l.split())) for l in open(sys.argv[1]) if l.strip())
t0 = rows[0][0]
names = {1: "c:phase", 2: "c:operands", 3: "c:stages", 4: "c:epi", 5: "c:barrier", 6: "c:attn+", 7: "c:attn-",
         12: "c:attn 1st stage done", 13: "c:attn loop end", 14: "c:attn flushed", 15: "c:attn csync",
         16: "c:cta-combine+", 17: "c:cta-combine-", 18: "c:arrive(+final)", 108: "p:qkv+", 109: "p:attn+", 110: "p:O+", 111: "p:O-"}
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
for t, g in rows[:n]:
    print(f"{(t - t0) / 1000:9.2f} us  {names.get(g, g)}")
