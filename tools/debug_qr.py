import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
for (m, k) in [(1500, 256), (512, 256), (300, 256), (5000, 100), (4000, 100), (2000, 256), (20000, 64), (50, 10), (2, 1), (33, 32)]:
    t = O.gaussian_matrix(m, k, m * 7 + k)
    q_ref, r_ref = O.thin_qr(t)
    q, r = P.thin_qr(torch.from_numpy(t).cuda())
    q = q.cpu().numpy(); r = r.cpu().numpy()
    ecol = np.abs(q @ r - t).max(axis=0)
    eq = np.abs(q - q_ref).max(axis=0)
    er = np.abs(r - r_ref).max(axis=1)
    bad = np.where(ecol > 1e-10)[0]
    print(m, k, "recon max", ecol.max(), "bad cols", bad[:10], "q-qref max", eq.max(), "worst q col", eq.argmax(), "r rows bad", np.where(er > 1e-9)[0][:10], "orth", np.abs(q.T @ q - np.eye(k)).max())
