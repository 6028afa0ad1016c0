"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count / total / share
of the LAST `--calls` fraction (default: second half = the second of two identical calls)."""
import csv, re, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if 'Kernel Name' in r:
        hdr = r; start = i + 1; break
idx = {h: i for i, h in enumerate(hdr)}
ks = [(r[idx['Kernel Name']], float(r[idx['Metric Value']])) for r in rows[start:]
      if r[idx['Metric Name']] == 'gpu__time_duration.sum' and not re.search(r'\bat(_cuda_detail)?::', r[idx['Kernel Name']])]
ks = ks[len(ks) // 2:] if '--all' not in sys.argv else ks
agg = OrderedDict()
for n, t in ks:
    n = n.split('(')[0].replace('sorsvd_dev::', '')
    c, s = agg.get(n, (0, 0.0)); agg[n] = (c + 1, s + t)
tot = sum(s for _, s in agg.values())
print("# kernel | launches | total us | share")
for n, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n} | {c} | {s/1000:.1f} | {s/tot:.3f}")
print(f"TOTAL | {sum(c for c, _ in agg.values())} | {tot/1000:.1f} | 1.0")
