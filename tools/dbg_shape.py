import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
for (m, n, k, q) in [(6000, 1100, 64, 1), (6000, 1100, 64, 0), (6000, 500, 64, 1), (3000, 1100, 64, 0)]:
    A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + 5)
    cfg = O.SketchConfig(k, q, 13)
    base = O.sor_svd_power(A, k, cfg)
    ref = O.Ref.sor_svd_power(A, k, cfg)
    d = P.sor_svd_power(A, k, P.SketchConfig(k, q, 13), fp64_mode="dmma")
    e = O.sigma_rel_err(d.sigma, base.sigma)
    er = O.sigma_rel_err(ref.sigma, base.sigma)
    print(m, n, k, q, "gpu-vs-port max %.1e at %d" % (e.max(), e.argmax()), "ref-vs-port max %.1e" % er.max(),
          "sig", base.sigma[[0, 39, 40, 63]], d.sigma[[0, 39, 40, 63]], flush=True)
    # thin_qr pieces
    om = O.gaussian_matrix(n, k, 13)
    t1 = A @ om
    q1g, r1g = P.thin_qr(torch.from_numpy(t1).cuda())
    q1o, r1o = O.thin_qr(t1)
    print("   qr T1 diff %.1e" % np.abs(q1g.cpu().numpy() - q1o).max(), "cond", np.linalg.cond(t1))
    t2 = A.T @ t1
    q2g, r2g = P.thin_qr(torch.from_numpy(t2).cuda())
    q2o, r2o = O.thin_qr(t2)
    print("   qr T2 diff %.1e" % np.abs(q2g.cpu().numpy() - q2o).max(), "cond", np.linalg.cond(t2))
