"""FP64 pass throughput vs problem size (ell fixed): separates fixed per-launch
overhead from the DMMA main-loop rate.."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_00462_b200 as P
ell = int(os.environ.get("ELL", "100"))
Np = (ell + 7) // 8 * 8 if ell <= 128 else (ell + 127) // 128 * 128
ctx = P.default_context(0)
lib = P._capi.lib()
for m, n in [(2000, 2000), (4000, 4000), (4000, 8000), (8000, 4000), (8000, 8000), (16000, 16000)]:
    A = torch.randn(m, n, dtype=torch.float64, device="cuda")
    for ta in (0, 1):
        X = torch.randn(m if ta else n, Np, device="cuda", dtype=torch.float64)
        T = torch.empty(n if ta else m, Np, device="cuda", dtype=torch.float64)
        ms = ctypes.c_double(); l = ctypes.c_int32()
        P._check(lib.sorsvd_pass_device(ctx.handle, ta, m, n, n, ell, A.data_ptr(), X.data_ptr(), T.data_ptr(), 20,
                                        ctypes.byref(ms), ctypes.byref(l)), ctx.handle)
        tf = 2.0 * m * n * ell / (ms.value * 1e-3) / 1e12
        print(f"m={m} n={n} ta={ta} ell={ell}: {ms.value*1e3:.1f} us  {tf:.2f} TF  launches {l.value}")
    del A
