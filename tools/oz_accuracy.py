"""Error of one pass T = A X of each FP64 engine against an 80-bit (numpy longdouble) product, in units of
max|a_row| max|x_col| and of |a_row|.|x_col| (the componentwise bound FP64 dot products obey)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1804_00462_b200 as P
lib = P._capi.lib()
print("digit products per FMA:", lib.sorsvd_ozaki_products())
ctx = P.Context(0); ctx.set_stream(torch.cuda.current_stream(0).cuda_stream)
rng = np.random.default_rng(3)
for name, m, n, ell, gen in [("gauss", 1024, 20000, 64, lambda s: rng.standard_normal(s)),
                             ("lowrank+noise", 1024, 20000, 64, None),
                             ("wide range", 1024, 4096, 32, lambda s: rng.standard_normal(s) * 10.0 ** rng.uniform(-6, 0, s))]:
    if gen is None:
        A = (rng.standard_normal((m, 30)) * 10.0 ** (-np.arange(30) / 8.0)) @ rng.standard_normal((30, n)) / 100 + 1e-3 * rng.standard_normal((m, n))
    else:
        A = gen((m, n))
    X = rng.standard_normal((n, ell))
    ref = np.zeros((m, ell), dtype=np.longdouble)
    Al, Xl = A.astype(np.longdouble), X.astype(np.longdouble)
    for j0 in range(0, n, 2048):
        ref += Al[:, j0:j0 + 2048] @ Xl[j0:j0 + 2048]
    absdot = np.abs(A) @ np.abs(X)
    scale = np.abs(A).max(1)[:, None] * np.abs(X).max(0)[None, :]
    Np = (ell + 7) // 8 * 8 if ell <= 128 else (ell + 127) // 128 * 128
    Ad = torch.from_numpy(A).cuda(); Xd = torch.zeros(n, Np, dtype=torch.float64, device="cuda"); Xd[:, :ell] = torch.from_numpy(X).cuda()
    out = {}
    T = torch.zeros(m, Np, dtype=torch.float64, device="cuda")
    ms, msc, lp = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
    P._check(lib.sorsvd_pass_ozaki_device(ctx.handle, 0, m, n, n, ell, 0, Ad.data_ptr(), Xd.data_ptr(), T.data_ptr(), 1, ctypes.byref(ms), ctypes.byref(msc)), ctx.handle)
    torch.cuda.synchronize(); out["ozaki int8"] = T[:, :ell].cpu().numpy()
    T.zero_()
    P._check(lib.sorsvd_pass_device(ctx.handle, 0, m, n, n, ell, Ad.data_ptr(), Xd.data_ptr(), T.data_ptr(), 1, ctypes.byref(ms), ctypes.byref(lp)), ctx.handle)
    torch.cuda.synchronize(); out["dmma"] = T[:, :ell].cpu().numpy()
    out["torch fp64 (cuBLAS)"] = (Ad @ Xd[:, :ell]).cpu().numpy()
    out["numpy fp64 (OpenBLAS)"] = A @ X
    for k, v in out.items():
        e = np.abs(v.astype(np.longdouble) - ref).astype(np.float64)
        print(f"{name:14s} {k:22s} max err / (max|a| max|x|) = {np.max(e / scale):.2e}   max err / (|a|.|x|) = {np.max(e / absdot):.2e}   rms err / (|a|.|x|) = {np.sqrt(np.mean((e / absdot) ** 2)):.2e}", flush=True)
