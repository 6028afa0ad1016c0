import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
A = O.gen_c2(2)
om = O.gaussian_matrix(4000, 100, 21)
T1 = A @ om; T2 = A.T @ T1; T1 = A @ T2; T2 = A.T @ T1
for name, T in (("T1", T1), ("T2", T2)):
    q, r = P.thin_qr(torch.from_numpy(T).cuda())
    q = q.cpu().numpy(); r = r.cpu().numpy()
    qn, rn = O.thin_qr(T)
    print(name, "gpu orth", np.abs(q.T@q - np.eye(100)).max(), "recon", np.linalg.norm(q@r - T)/np.linalg.norm(T),
          "| np orth", np.abs(qn.T@qn - np.eye(100)).max(), "recon", np.linalg.norm(qn@rn - T)/np.linalg.norm(T))
    # subspace agreement for leading columns
    for j in (10, 30, 50, 70, 100):
        s = np.linalg.svd(q[:, :j].T @ qn[:, :j], compute_uv=False)
        print("   lead", j, "min cos", s.min())
At = torch.from_numpy(A).cuda()
def fro(u, s, v): return float(torch.linalg.norm(At - (torch.from_numpy(u).cuda()*torch.from_numpy(s).cuda())@torch.from_numpy(v).cuda().T))
for trial in range(3):
    f = P.sor_svd_power(A, 100, P.SketchConfig(100, 1, 21))
    print("gpu fro", fro(f.u, f.sigma, f.v))
b = O.sor_svd_power(A, 100, O.SketchConfig(100, 1, 21))
print("oracle fro", fro(b.u, b.sigma, b.v))
# hybrid: oracle Q1/Q2 + gpu small svd
q1, _ = O.thin_qr(T1); q2, _ = O.thin_qr(T2)
M = q1.T @ A @ q2
u, s, v, sw = P.full_svd(torch.from_numpy(M).cuda())
u, s, v = u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy()
print("oracle QR + gpu jacobi fro", fro(q1@u, s, q2@v), "sweeps", sw)
uo, so, vo = O.full_svd(M)
print("oracle QR + oracle svd fro", fro(q1@uo, so, q2@vo))
# gpu QR + oracle SVD
g1, _ = P.thin_qr(torch.from_numpy(T1).cuda()); g2, _ = P.thin_qr(torch.from_numpy(T2).cuda())
g1 = g1.cpu().numpy(); g2 = g2.cpu().numpy()
Mg = g1.T @ A @ g2
uo, so, vo = O.full_svd(Mg)
print("gpu QR + oracle svd fro", fro(g1@uo, so, g2@vo))
