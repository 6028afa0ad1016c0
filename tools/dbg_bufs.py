import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
lib = P._capi.lib()
m, n, k = 6000, 1100, 64
A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + 5)
base = O.sor_svd_power(A, k, O.SketchConfig(k, 0, 13))
ctx = P.Context(0)
Ad = torch.from_numpy(A).cuda()
f = P.sor_svd_power(Ad, k, P.SketchConfig(k, 0, 13), fp64_mode="dmma", ctx=ctx, use_graph=False)
print("sigma err %.1e" % O.sigma_rel_err(f.sigma.cpu().numpy(), base.sigma).max())
def get(name, rows, cols):
    t = torch.empty(rows * cols, dtype=torch.float64, device="cuda")
    P._check(lib.sorsvd_debug_buffer(ctx.handle, name.encode(), t.data_ptr(), rows * cols), ctx.handle)
    return t.view(rows, cols).cpu().numpy()
om = O.gaussian_matrix(n, k, 13)
t1 = A @ om
t2 = A.T @ t1
T1, T2, Q1, Q2, Mk = get("T1", m, k), get("T2", n, k), get("Q1", m, k), get("Q2", n, k), get("Mk", k, k)
q1, _ = O.thin_qr(t1); q2, _ = O.thin_qr(t2)
print("T1 %.1e T2 %.1e Q1 %.1e Q2 %.1e M %.1e" % (np.abs(T1 - t1).max() / np.abs(t1).max(), np.abs(T2 - t2).max() / np.abs(t2).max(),
      np.abs(Q1 - q1).max(), np.abs(Q2 - q2).max(), np.abs(Mk - base.extras["m"]).max()))
print("Q1 orth %.1e Q2 orth %.1e" % (np.abs(Q1.T @ Q1 - np.eye(k)).max(), np.abs(Q2.T @ Q2 - np.eye(k)).max()))
OM = get("omega_in", n, k)
print("omega_in vs oracle: %.1e; cols wrong:" % np.abs(OM - om).max(), np.nonzero(np.abs(OM - om).max(0) > 0)[0][:10],
      "rows wrong:", np.nonzero(np.abs(OM - om).max(1) > 0)[0][:10])
print("lib gaussian vs oracle: %.1e" % np.abs(P.gaussian_matrix(n, k, 13) - om).max())
print("Q1 vs q1 per column:", np.round(np.log10(np.abs(Q1 - q1).max(0) + 1e-300), 1)[-6:])
print("Q2 vs q2 per column max:", np.round(np.log10(np.abs(Q2 - q2).max(0) + 1e-300), 1)[:64])
