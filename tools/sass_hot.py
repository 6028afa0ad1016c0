"""Summarise an ncu --page source --print-source sass CSV: samples by opcode and the hottest instructions."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}; data = rows[2:]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sc = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = sum(int(r[idx['# Samples']]) for r in data)
print("kernel", rows[0][1][:100], "samples", tot)
agg = Counter()
for r in data:
    for h in sc: agg[h] += int(r[idx[h]])
print("stalls:", [(h, v) for h, v in agg.most_common(8)])
c = Counter()
for r in data:
    s = r[idx['Source']].strip().split()
    if not s: continue
    op = s[1] if s[0].startswith('@') else s[0]
    c[op.split('.')[0]] += int(r[idx['# Samples']])
print("by opcode:", c.most_common(14))
top = sorted(range(len(data)), key=lambda i: -int(data[i][idx['# Samples']]))[:ntop]
for i in sorted(top):
    r = data[i]
    st = sorted(((int(r[idx[h]]), h[6:]) for h in sc), reverse=True)[:2]
    print(i, r[idx['Address']][-5:], r[idx['Source']].strip()[:60].ljust(60), r[idx['# Samples']].rjust(5), st)
