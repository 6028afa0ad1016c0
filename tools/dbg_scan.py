import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
m = 6000
for n in (600, 800, 1000, 1023, 1024, 1025, 1100, 1500):
    row = []
    for k in (32, 48, 64, 100):
        A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + 5)
        base = O.sor_svd_power(A, k, O.SketchConfig(k, 0, 13))
        f = P.sor_svd_power(A, k, P.SketchConfig(k, 0, 13), fp64_mode="dmma")
        row.append("%d:%.0e" % (k, O.sigma_rel_err(f.sigma, base.sigma).max()))
    print(n, row, flush=True)
