"""Localise the k = 512 FP64 parity gap: QR vs core SVD vs passes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402
from oracle import sorsvd_oracle as O  # noqa: E402

A = O.gen_lowrank_decay(4096, 3000, 512, lambda j: 1.0 / j, 1e-6, 5)
cfg = O.SketchConfig(512, 1, 41)
base = O.sor_svd_power(A, 512, cfg)
mm, q1r, q2r = base.extras["m"], base.extras["q1"], base.extras["q2"]
# perturbed-input floor (1 trial)
Ap = A * (1 + 1e-16 * np.random.default_rng(1).standard_normal(A.shape))
pert = O.sor_svd_power(Ap, 512, cfg)
fl = O.sigma_rel_err(pert.sigma, base.sigma)
# 1) core SVD alone on the oracle's M
u, s, v, sw = P.full_svd(torch.from_numpy(mm).cuda())
e_svd = O.sigma_rel_err(s.cpu().numpy(), base.sigma)
# 2) QR alone: our Q1, Q2 from the oracle's T1, T2, then M in numpy
om = O.gaussian_matrix(3000, 512, 41)
t1 = A @ om
t2 = A.T @ t1
t1 = A @ t2
t2 = A.T @ t1
q1, _ = P.thin_qr(torch.from_numpy(t1).cuda())
q2, _ = P.thin_qr(torch.from_numpy(t2).cuda())
q1, q2 = q1.cpu().numpy(), q2.cpu().numpy()
m2 = q1.T @ A @ q2
e_qr = O.sigma_rel_err(np.linalg.svd(m2, compute_uv=False), base.sigma)
print("orth q1", np.abs(q1.T @ q1 - np.eye(512)).max(), "q2", np.abs(q2.T @ q2 - np.eye(512)).max())
# Householder (numpy) Q of the same T for comparison
q1h, _ = np.linalg.qr(t1)
q2h, _ = np.linalg.qr(t2)
m3 = q1h.T @ A @ q2h
e_np = O.sigma_rel_err(np.linalg.svd(m3, compute_uv=False), base.sigma)
# 3) full GPU pipeline
f = P.sor_svd_power(A, 512, P.SketchConfig(512, 1, 41))
e_all = O.sigma_rel_err(f.sigma, base.sigma)
for name, e in [("floor", fl), ("svd", e_svd), ("qr", e_qr), ("np_householder", e_np), ("gpu_all", e_all)]:
    print(name, " ".join(f"{e[a:b].max():.2e}" for a, b in [(0, 64), (64, 128), (128, 256), (256, 384), (384, 512)]))
