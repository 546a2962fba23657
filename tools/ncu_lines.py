"""Dev: attribute ncu stall samples (source page, SASS) to CUDA source lines
via nvdisasm --print-line-info of the same cubin.
usage: ncu_lines.py <sass.csv> <all.sass> <function-prefix> [top]"""
import csv, re, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
S, addr, src = ix['Warp Stall Sampling (All Samples)'], ix['Address'], ix['Source']
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
base = min(int(r[addr], 16) for r in data)
lines = open(sys.argv[2]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('.text.' + sys.argv[3])][0]
cur, off2line, off2txt = None, {}, {}
for l in lines[start + 1:]:
    if l.startswith('.text.') or l.strip().startswith('.section'):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        off2line[int(m.group(1), 16)] = cur
        off2txt[int(m.group(1), 16)] = m.group(2).strip()
mism = sum(1 for r in data if off2txt.get(int(r[addr], 16) - base, '').split()[:1] != r[src].split()[:1])
tot = sum(float(r[S] or 0) for r in data)
agg = defaultdict(float)
rs = defaultdict(lambda: defaultdict(float))
for r in data:
    k = off2line.get(int(r[addr], 16) - base)
    agg[k] += float(r[S] or 0)
    for q in reasons:
        rs[k][q] += float(r[ix[q]] or 0)
print(f"samples {tot:.0f}, sass mismatches {mism}")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    top = sorted(rs[k].items(), key=lambda x: -x[1])[:3]
    print(f"{v / tot * 100:5.2f}%  {k}  " + ", ".join(f"{q[6:]}={w / max(v, 1) * 100:.0f}%" for q, w in top))
