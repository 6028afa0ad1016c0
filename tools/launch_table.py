"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per kernel
name, launches and total time (ms), our kernels only (torch's excluded)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        out.append((r[ki], v))
    return out


if __name__ == "__main__":
    seq = [(n, v) for n, v in load(sys.argv[1]) if "at::" not in n and "cutlass" not in n and "cublas" not in n.lower()
           and "elementwise" not in n and "distribution" not in n]
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for n, v in seq:
        key = n.split("(")[0].replace("void ", "").replace("sorsvd_dev::", "")
        tot[key] = tot.get(key, 0.0) + v
        cnt[key] += 1
    all_ms = sum(tot.values())
    print(f"{'ms':>10} {'share':>6} {'n':>5}  kernel   (total {all_ms:.3f} ms, {len(seq)} launches)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:10.3f} {v / all_ms:6.1%} {cnt[k]:5d}  {k}")
