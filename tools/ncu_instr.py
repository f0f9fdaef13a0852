"""Sum ncu 'Instructions Executed' (warp-level) and stall samples per CUDA source line range."""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
si = hdr.index('Warp Stall Sampling (All Samples)'); ii = hdr.index('Instructions Executed')
addr0 = int(data[0][0], 16)
line_of = {}; cur = None
for l in open(sys.argv[2]):
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m and cur: line_of[int(m.group(1), 16)] = cur
lo, hi = int(sys.argv[3]), int(sys.argv[4])
ins = collections.Counter(); smp = collections.Counter()
for r in data:
    if not r[0].startswith('0x'): continue
    f, ln = line_of.get(int(r[0], 16) - addr0, ('?', 0))
    if f == 'decode.cu' and lo <= ln <= hi:
        ins[ln] += int(r[ii] or 0); smp[ln] += int(r[si] or 0)
src = open('paper_2507_00507_b200/csrc/gpu/decode.cu').read().split('\n')
tot = sum(ins.values())
print('instructions in range', tot, 'samples', sum(smp.values()))
for ln, n in sorted(ins.items(), key=lambda x: -x[1])[:30]:
    print(f'{n:10d} {smp[ln]:7d}  {ln}: {src[ln-1].strip()[:90]}')
