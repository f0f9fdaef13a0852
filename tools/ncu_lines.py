"""Attribute ncu SASS-level warp-stall samples to CUDA source lines.
usage: ncu_lines.py <ncu source-page sass csv> <nvdisasm -g -c output> [file-substring]"""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
si = hdr.index('Warp Stall Sampling (All Samples)')
addr0 = int(data[0][0], 16)
samples = {int(r[0], 16) - addr0: int(r[si] or 0) for r in data if r[0].startswith('0x')}
line_of = {}
cur = None
for l in open(sys.argv[2]):
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
agg = collections.Counter()
for off, s in samples.items():
    agg[line_of.get(off, ('?', 0))] += s
tot = sum(samples.values())
src = {}
want = sys.argv[3] if len(sys.argv) > 3 else ''
print('total samples', tot)
for (f, ln), s in agg.most_common(40):
    if want and want not in f: continue
    try:
        text = open('paper_2507_00507_b200/csrc/gpu/' + f).read().split('\n')[ln - 1].strip()[:90]
    except Exception:
        text = ''
    print(f'{s:7d} {100*s/tot:5.1f}%  {f}:{ln}  {text}')
