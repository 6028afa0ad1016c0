"""Repro: full_svd after a NaN input on the barrier cluster ring (k > 128)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
for k in [int(x) for x in (sys.argv[1:] or ["200"])]:
    mm = O.gaussian_matrix(k, k, 7)
    mm[:, 3] = 1.0
    ref = np.linalg.svd(mm, compute_uv=False)
    _, s, _, sw = P.full_svd(torch.from_numpy(mm).cuda())
    e0 = np.abs(s.cpu().numpy() - ref).max() / ref[0]
    bad = mm.copy(); bad[:, 3] = np.nan
    _, sb, _, swb = P.full_svd(torch.from_numpy(bad).cuda())
    _, s2, _, sw2 = P.full_svd(torch.from_numpy(mm).cuda())
    e2 = np.abs(s2.cpu().numpy() - ref).max() / ref[0]
    ctx = P.Context(0)
    _, s3, _, _ = P.full_svd(torch.from_numpy(mm).cuda(), ctx=ctx)
    e3 = np.abs(s3.cpu().numpy() - ref).max() / ref[0]
    print(f"k={k} clean err {e0:.2e} sweeps {sw}; nan sweeps {swb} sig0 {sb[0].item()}; after-nan err {e2:.2e} sweeps {sw2}; fresh ctx err {e3:.2e}", flush=True)
