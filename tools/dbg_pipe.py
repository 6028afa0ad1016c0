import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
m, n, k, q = 6000, 1100, 64, 0
A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + 5)
cfg = O.SketchConfig(k, q, 13)
base = O.sor_svd_power(A, k, cfg)
ex = base.extras
Ad = torch.from_numpy(A).cuda()
om = torch.from_numpy(O.gaussian_matrix(n, k, 13)).cuda()
t1 = P.matmul(Ad, om)
t2 = P.matmul(Ad, t1, transpose_a=True)
q1, _ = P.thin_qr(t1)
q2, _ = P.thin_qr(t2)
y = P.matmul(Ad, q2)
mm = P.matmul(q1, y, transpose_a=True)
u, s, v, sw = P.full_svd(mm)
print("manual pipeline sigma err %.1e" % O.sigma_rel_err(s.cpu().numpy(), base.sigma).max())
print("q1 diff %.1e  q2 diff %.1e  M diff %.1e" % (np.abs(q1.cpu().numpy() - ex["q1"]).max(),
      np.abs(q2.cpu().numpy() - ex["q2"]).max(), np.abs(mm.cpu().numpy() - ex["m"]).max()))
so = np.linalg.svd(ex["m"], compute_uv=False)
print("svd(M_oracle) vs base %.1e; our svd of oracle M: %.1e" % (O.sigma_rel_err(so, base.sigma).max(),
      O.sigma_rel_err(P.full_svd(torch.from_numpy(ex["m"]).cuda())[1].cpu().numpy(), base.sigma).max()))
for tag, kw in (("graph", {}), ("nograph", {"use_graph": False}), ("stage", {"stage_times": True})):
    f = P.sor_svd_power(Ad, k, P.SketchConfig(k, q, 13), fp64_mode="dmma", **kw)
    print(tag, "%.1e" % O.sigma_rel_err(f.sigma.cpu().numpy(), base.sigma).max())
