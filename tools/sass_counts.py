"""SASS mnemonic counts per kernel: cuobjdump -sass <lib> | python tools/sass_counts.py > profiles/..."""
import collections, re, sys
cur = None
counts = collections.OrderedDict()
want = re.compile(r'\b(UTMALDG|UBLKCP|UTCIMMA|UTCHMMA|UTCBAR|LDTM|STTM|DMMA|LDGSTS|SYNCS|UTCCP|F2I|DFMA|DMUL)\b')
for line in sys.stdin:
    m = re.search(r'Function : (\S+)', line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur:
        for w in want.findall(line):
            counts[cur][w] += 1
print("# SASS mnemonic counts per kernel (cuobjdump -sass libsorsvd_b200.so, sm_100a): the A-streaming pass kernels and helpers")
for k, v in counts.items():
    if any(t in k for t in ('ozaki', 'skinny_pair', 'gemm_f64_kernel', 'tc_gemm', 'gen_lowrank', 'gaussian_fill')) and v:
        print(k[:120], dict(v))
