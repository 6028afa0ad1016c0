"""Repeat Ozaki passes on fixed inputs: bitwise stability across repeats and error vs torch FP64."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_00462_b200 as P
lib = P._capi.lib()
ctx = P.Context(0)
ctx.set_stream(torch.cuda.current_stream(0).cuda_stream)
dev = torch.device("cuda", 0)
for (m, n, ell, ta, dbg) in [(300, 20000, 10, 1, 0), (20000, 2000, 256, 1, 0), (20000, 2000, 256, 0, 0),
                             (4000, 3000, 64, 1, 0), (300, 20000, 10, 1, 4 | 0)]:
    g = torch.Generator(device=dev); g.manual_seed(m + n)
    A = torch.randn(m, n, generator=g, device=dev, dtype=torch.float64)
    Np = (ell + 7) // 8 * 8 if ell <= 128 else (ell + 127) // 128 * 128
    K = m if ta else n
    X = torch.zeros(K, Np, device=dev, dtype=torch.float64)
    X[:, :ell] = torch.randn(K, ell, generator=g, device=dev, dtype=torch.float64)
    ref = (A.T if ta else A) @ X
    outs = []
    for rep in range(4):
        T = torch.full(((n if ta else m), Np), float("nan"), device=dev, dtype=torch.float64)
        ms, msc = ctypes.c_double(), ctypes.c_double()
        P._check(lib.sorsvd_pass_ozaki_device(ctx.handle, ta, m, n, n, ell, dbg << 8, A.data_ptr(), X.data_ptr(),
                                              T.data_ptr(), 1, ctypes.byref(ms), ctypes.byref(msc)), ctx.handle)
        torch.cuda.synchronize()
        outs.append(T)
    errs = [((o - ref).abs().max() / ref.abs().max()).item() for o in outs]
    same = [torch.equal(outs[0], o) for o in outs[1:]]
    badtiles = sorted(set((((outs[0] - ref).abs() > 1e-9 * ref.abs().max()).nonzero()[:, 0] // 128).tolist()))
    print(dict(m=m, n=n, ell=ell, ta=ta, dbg=dbg, errs=["%.1e" % e for e in errs], same=same, badtiles=badtiles[:10]),
          flush=True)
