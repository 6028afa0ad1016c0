import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
lib = P._capi.lib()
ctx = P.Context(0)
ctx.set_stream(torch.cuda.current_stream(0).cuda_stream)
for (m, n, ell, ta) in [(6000, 1100, 64, 1), (6000, 500, 64, 1), (6000, 1100, 64, 0), (20000, 300, 10, 1), (4000, 4000, 100, 1),
                        (4000, 4000, 100, 0), (25344, 300, 10, 1), (1000, 1000, 20, 1)]:
    g = torch.Generator(device="cuda"); g.manual_seed(m + n)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    Np = (ell + 7) // 8 * 8 if ell <= 128 else (ell + 127) // 128 * 128
    X = torch.zeros(m if ta else n, Np, device="cuda", dtype=torch.float64)
    X[:, :ell] = torch.randn(X.shape[0], ell, generator=g, device="cuda", dtype=torch.float64)
    T = torch.full((n if ta else m, Np), float("nan"), device="cuda", dtype=torch.float64)
    ms = ctypes.c_double(); l = ctypes.c_int32()
    P._check(lib.sorsvd_pass_device(ctx.handle, ta, m, n, n, ell, A.data_ptr(), X.data_ptr(), T.data_ptr(), 1,
                                    ctypes.byref(ms), ctypes.byref(l)), ctx.handle)
    torch.cuda.synchronize()
    ref = (A.T if ta else A) @ X
    err = ((T - ref).abs().max() / ref.abs().max()).item()
    bad = ((T - ref).abs().amax(1) > 1e-10 * ref.abs().max()).nonzero().flatten()
    print(m, n, ell, ta, "launches", l.value, "%.1e" % err, "bad rows", bad[:6].tolist(), len(bad), flush=True)
