import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
A = O.gen_c2(2)
om = O.gaussian_matrix(4000, 100, 21)
At = torch.from_numpy(A).cuda()
def fro(u, s, v): return float(torch.linalg.norm(At - (torch.from_numpy(u).cuda()*torch.from_numpy(s).cuda())@torch.from_numpy(v).cuda().T))
def finish(q1, q2, M):
    u, s, v = O.full_svd(M); return fro(q1@u, s, q2@v)
mm = lambda a, b, t=False: P.matmul(torch.from_numpy(np.ascontiguousarray(a)).cuda(), torch.from_numpy(np.ascontiguousarray(b)).cuda(), transpose_a=t).cpu().numpy()
# numpy chain
T1 = A @ om; T2 = A.T @ T1; T1 = A @ T2; T2 = A.T @ T1
# gpu chain
G1 = mm(A, om); G2 = mm(A, G1, True); G1 = mm(A, G2); G2 = mm(A, G1, True)
print("rel diff T1", np.linalg.norm(G1-T1)/np.linalg.norm(T1), "T2", np.linalg.norm(G2-T2)/np.linalg.norm(T2))
q1, _ = O.thin_qr(T1); q2, _ = O.thin_qr(T2)
print("(0) all numpy", finish(q1, q2, (q1.T @ A) @ q2))
print("(c) numpy, M = Q1^T (A Q2)", finish(q1, q2, q1.T @ (A @ q2)))
g1, _ = O.thin_qr(G1); g2, _ = O.thin_qr(G2)
print("(a) gpu sketches + numpy rest", finish(g1, g2, (g1.T @ A) @ g2))
Y = mm(A, q2); M = mm(q1, Y, True)
print("(b) numpy sketches/QR, gpu projection", finish(q1, q2, M))
f = P.sor_svd_power(A, 100, P.SketchConfig(100, 1, 21))
print("full gpu", fro(f.u, f.sigma, f.v))
