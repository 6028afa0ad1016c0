"""One Ozaki pass on the C3 matrix shape (random A), for ncu captures / timing."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_00462_b200 as P
m, n, ell = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (200000, 20000, 256))]
ta = int(sys.argv[4]) if len(sys.argv) > 4 else 0
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
dbg = int(sys.argv[6]) if len(sys.argv) > 6 else 0
dev = torch.device("cuda", 0)
A = torch.randn(m, n, device=dev, dtype=torch.float64)
Np = (ell + 7) // 8 * 8 if ell <= 128 else (ell + 127) // 128 * 128
X = torch.randn(m if ta else n, Np, device=dev, dtype=torch.float64)
T = torch.empty(n if ta else m, Np, device=dev, dtype=torch.float64)
ctx = P.Context(0)
ms, msc = ctypes.c_double(), ctypes.c_double()
for _ in range(2):  # the first call allocates the workspaces (its "scales" time includes that)
    P._check(P._capi.lib().sorsvd_pass_ozaki_device(ctx.handle, ta, m, n, n, ell, dbg << 8, A.data_ptr(), X.data_ptr(),
                                                    T.data_ptr(), reps, ctypes.byref(ms), ctypes.byref(msc)), ctx.handle)
    torch.cuda.synchronize()
print(f"ozaki m={m} n={n} ell={ell} ta={ta} dbg={dbg}: pass {ms.value:.3f} ms, scales {msc.value:.3f} ms")
