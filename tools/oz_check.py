"""Dev check of the Ozaki (int8 tensor-core) pass against torch FP64 matmul, and its timing."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
C = P._capi
lib = C.lib()
ctx = P.Context(0)
ctx.set_stream(torch.cuda.current_stream(0).cuda_stream)  # order with torch's allocations / generators


def npad(ell):
    return (ell + 7) // 8 * 8 if ell <= 128 else (ell + 127) // 128 * 128


def one(m, n, ell, ta, dtype=torch.float64, reps=1, gen=None):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev); g.manual_seed(m + n + ell + ta)
    A = gen(m, n) if gen else torch.randn(m, n, generator=g, device=dev, dtype=torch.float64)
    A = A.to(dtype)
    Np = npad(ell)
    K = m if ta else n
    X = torch.zeros(K, Np, device=dev, dtype=torch.float64)
    X[:, :ell] = torch.randn(K, ell, generator=g, device=dev, dtype=torch.float64)
    T = torch.full(((n if ta else m), Np), float("nan"), device=dev, dtype=torch.float64)
    ms, msc = ctypes.c_double(), ctypes.c_double()
    P._check(lib.sorsvd_pass_ozaki_device(ctx.handle, ta, m, n, n, ell, 1 if dtype == torch.float32 else 0,
                                          A.data_ptr(), X.data_ptr(), T.data_ptr(), reps, ctypes.byref(ms),
                                          ctypes.byref(msc)), ctx.handle)
    torch.cuda.synchronize()
    A64 = A.double()
    ref = (A64.T if ta else A64) @ X
    err = (T - ref).abs()
    scale = (A64.abs().amax(dim=0 if ta else 1, keepdim=True).T if False else None)
    denom = ref.abs().max().item()
    rel = err.max().item() / max(denom, 1e-300)
    # per-entry error relative to sqrt(K) max|a| max|x| (the bound's shape)
    amax = A64.abs().amax(dim=0 if ta else 1)  # per left row
    xmax = X.abs().amax(dim=0)
    bnd = (amax[:, None] * xmax[None, :]) * np.sqrt(K)
    normed = (err[:, :ell] / bnd[:, :ell].clamp_min(1e-300)).max().item()
    nan = torch.isnan(T[:, :ell]).any().item()
    bad = (err[:, :ell] > 1e-6 * denom)
    nbad = int(bad.sum().item())
    info = {}
    if nbad:
        idx = bad.nonzero()
        brows = sorted(set(idx[:, 0].tolist()))[:6]
        rm = [float(A64[r].abs().max()) if not ta else float(A64[:, r].abs().max()) for r in brows]
        am = [int(A64[r].abs().argmax()) if not ta else int(A64[:, r].abs().argmax()) for r in brows]
        info = dict(nbad=nbad, brows=brows, rowmax=rm, argmax=am, frexp=[np.frexp(x) for x in rm])
    return dict(**info, m=m, n=n, ell=ell, ta=ta, dtype=str(dtype), max_rel=rel, normed=normed, nan=nan,
                ms=ms.value, ms_scales=msc.value)


def scales(m, n, seed):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev); g.manual_seed(seed)
    A = torch.randn(m, n, generator=g, device=dev, dtype=torch.float64)
    re = torch.zeros(m, dtype=torch.int32, device=dev); ce = torch.zeros(n, dtype=torch.int32, device=dev)
    P._check(lib.sorsvd_ozaki_scales_device(ctx.handle, m, n, n, 0, A.data_ptr(), re.data_ptr(), ce.data_ptr()),
             ctx.handle)
    rm = A.abs().amax(1).cpu().numpy(); cm = A.abs().amax(0).cpu().numpy()
    er = np.frexp(rm)[1]; ec = np.frexp(cm)[1]
    br = np.nonzero(re.cpu().numpy() != er)[0]; bc = np.nonzero(ce.cpu().numpy() != ec)[0]
    print(dict(m=m, n=n, bad_rows=br[:5].tolist(), nbr=len(br), bad_cols=bc[:5].tolist(), nbc=len(bc),
               got=re.cpu().numpy()[br[:3]].tolist(), want=er[br[:3]].tolist(), rowmax=rm[br[:3]].tolist()), flush=True)


for args in [(1000, 700, 20, 0), (1000, 700, 20, 1), (4001, 999, 100, 0), (3999, 1001, 100, 1),
             (513, 2049, 256, 0), (513, 2049, 256, 1), (300, 20000, 10, 1), (20000, 300, 10, 0),
             (130, 33, 8, 0), (33, 130, 8, 1), (20000, 2000, 256, 0), (20000, 2000, 256, 1),
             (20000, 2001, 64, 0), (20000, 2001, 64, 1), (40000, 1000, 128, 1)]:
    print(one(*args), flush=True)
for args in [(4000, 3000, 64, 0), (4000, 3000, 64, 1), (4000, 3001, 64, 0), (3001, 4000, 200, 1)]:
    print(one(*args, dtype=torch.float32), flush=True)
for ta in (0, 1):
    print(one(200000, 20000, 256, ta, reps=3), flush=True)
