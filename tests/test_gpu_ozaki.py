"""The Ozaki-scheme FP64 passes (exact int8 slice products on the tcgen05
tensor cores; ozaki_planes_i8.cuh: A cut into digit planes once per call,
ozaki_i8.cuh: A converted inside every pass) against FP64 references: the pass kernel itself
against an FP64 GEMM of the same operands, and whole sor_svd_power calls in
fp64_mode="ozaki" against the CPU oracle under the same parity protocol as
the DMMA path (tests/test_gpu_parity.py)."""
import ctypes

import numpy as np
import pytest

from oracle import sorsvd_oracle as O

pytestmark = pytest.mark.gpu

# error bound of one pass, per output entry, in units of sqrt(K) max|a_row| max|x_col|:
# the 2^-55 fixed-point grid and the dropped digit levels give ~1e-15 (measured <= 3e-15);
# FP64 dgemm's own sum rounding is of the same order
PASS_TOL = 2e-14


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_00462_b200 as P
    return P


def _npad(ell):
    return (ell + 7) // 8 * 8 if ell <= 128 else (ell + 127) // 128 * 128


def _pass(P, A, X, ta, m, n, ell, lda=None, dtype=0, reps=1, planes=True):
    import torch
    ctx = P.Context(0)
    ctx.set_option(P.Context.OPT_OZAKI_PLANES, int(planes))
    ctx.set_stream(torch.cuda.current_stream(0).cuda_stream)
    Np = _npad(ell)
    T = torch.full(((n if ta else m), Np), float("nan"), device="cuda", dtype=torch.float64)
    ms, msc = ctypes.c_double(), ctypes.c_double()
    P._check(P._capi.lib().sorsvd_pass_ozaki_device(ctx.handle, ta, m, n, lda or n, ell, dtype, A.data_ptr(),
                                                     X.data_ptr(), T.data_ptr(), reps, ctypes.byref(ms),
                                                     ctypes.byref(msc)), ctx.handle)
    torch.cuda.synchronize()
    return T


def _operands(m, n, ell, ta, seed, lda=None, f32=False):
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    lda = lda or n
    buf = torch.randn(m, lda, generator=g, device="cuda", dtype=torch.float64)
    buf *= torch.exp(2.0 * torch.randn(m, 1, generator=g, device="cuda", dtype=torch.float64))  # graded rows
    if f32:
        buf = buf.float()
    A = buf[:, :n]
    Np = _npad(ell)
    K = m if ta else n
    X = torch.zeros(K, Np, device="cuda", dtype=torch.float64)
    X[:, :ell] = torch.randn(K, ell, generator=g, device="cuda", dtype=torch.float64)
    return buf, A, X


@pytest.mark.parametrize("m,n,ell,ta,lda,f32", [
    (1000, 700, 20, 0, None, False), (1000, 700, 20, 1, None, False),
    (4001, 999, 100, 0, None, False), (3999, 1001, 100, 1, None, False),   # odd lda: no TMA
    (513, 2049, 256, 0, None, False), (513, 2049, 256, 1, None, False),
    (300, 20000, 10, 1, None, False), (20000, 300, 10, 0, None, False),
    (130, 33, 8, 0, None, False), (33, 130, 8, 1, None, False),
    (20000, 2000, 256, 0, None, False), (20000, 2000, 256, 1, None, False),
    (700, 500, 64, 0, 513, False), (700, 500, 64, 1, 513, False),         # padded lda
    (4000, 3000, 64, 0, None, True), (4000, 3000, 64, 1, None, True),     # FP32 storage
    (4000, 3001, 64, 0, None, True), (3001, 4000, 200, 1, None, True),
    (40000, 1000, 512, 1, None, False), (1000, 40000, 136, 0, None, False),  # several TMEM drains
    (70000, 600, 64, 1, None, False),                                        # planes engine: split-K
])
@pytest.mark.parametrize("planes", [True, False])
def test_ozaki_pass_vs_fp64(P, m, n, ell, ta, lda, f32, planes):
    import torch
    buf, A, X = _operands(m, n, ell, ta, m + 7 * n + ell, lda, f32)
    T = _pass(P, buf, X, ta, m, n, ell, lda=lda or n, dtype=1 if f32 else 0, planes=planes)
    A64 = A.double()
    ref = (A64.T if ta else A64) @ X
    K = m if ta else n
    # the per-call planes are scaled by rows for both orientations: the TN error is relative to
    # the largest row maximum met in the column, not to the column's own maximum
    amax = A64.abs().amax(dim=0 if ta else 1)
    if ta and planes:
        amax = torch.maximum(amax, (A64.abs().amax(dim=1)[:, None] * (A64 != 0)).amax(dim=0))
    xmax = X.abs().amax(dim=0).clamp_min(1e-300)
    err = (T - ref).abs()[:, :ell] / (amax[:, None] * xmax[None, :ell] * np.sqrt(K)).clamp_min(1e-300)
    assert not torch.isnan(T[:, :ell]).any()
    assert err.max().item() <= PASS_TOL, err.max().item()
    if T.shape[1] > ell:
        assert torch.all(T[:, ell:] == 0)


@pytest.mark.parametrize("planes", [True, False])
def test_ozaki_pass_deterministic(P, planes):
    import torch
    buf, A, X = _operands(20000, 2000, 256, 1, 5)
    outs = [_pass(P, buf, X, 1, 20000, 2000, 256, planes=planes) for _ in range(3)]
    assert all(torch.equal(outs[0], o) for o in outs[1:])


def test_ozaki_planes_tn_nonfinite(P):
    """TN from row-scaled planes: a non-finite entry of A reaches every output (as NaN), like the
    reference's A^T T1 with T1's row already non-finite."""
    import torch
    buf, A, X = _operands(600, 400, 32, 1, 9)
    A[5, 17] = float("inf")
    T = _pass(P, buf, X, 1, 600, 400, 32, planes=True)
    assert torch.isnan(T[:, :32]).all()


@pytest.mark.parametrize("planes", [True, False])
def test_ozaki_pass_nonfinite_and_zero_rows(P, planes):
    import torch
    buf, A, X = _operands(600, 400, 32, 0, 9)
    A[5, 17] = float("nan")
    A[9, :] = 0.0
    X[3, 7] = float("inf")
    T = _pass(P, buf, X, 0, 600, 400, 32, planes=planes)
    assert torch.isnan(T[5, :32]).all()        # the row with a NaN
    assert torch.isnan(T[:, 7]).all()          # the column of X with an Inf
    ok = [j for j in range(32) if j != 7]
    assert torch.all(T[9, ok] == 0)            # an all-zero row
    ref = A @ X
    rows = [i for i in range(600) if i != 5]
    d = (T[rows][:, ok] - ref[rows][:, ok]).abs().max().item()
    assert d <= 1e-12 * ref[rows][:, ok].abs().max().item()


# ---------------------------------------------------------- whole decompositions --
def _check_parity(got, base, ds=None, dl=0.0, tol_s=1e-10, tol_lr=1e-9):
    s = np.asarray(got.sigma.cpu() if hasattr(got.sigma, "cpu") else got.sigma)
    u = np.asarray(got.u.cpu() if hasattr(got.u, "cpu") else got.u)
    v = np.asarray(got.v.cpu() if hasattr(got.v, "cpu") else got.v)
    es = O.sigma_rel_err(s, base.sigma)
    lim = np.maximum(tol_s, 10 * np.maximum.accumulate(ds)) if ds is not None else tol_s
    assert np.all(es <= lim), (es.max(), es)
    lr = O.lowrank_rel_diff(u, s, v, base.u, base.sigma, base.v)
    assert lr <= max(tol_lr, 10 * dl), lr


@pytest.mark.parametrize("planes", [True, False])
def test_ozaki_golden_cases(P, golden, planes):
    g, meta = golden
    ctx = P.Context(0)
    ctx.set_option(P.Context.OPT_OZAKI_PLANES, int(planes))
    for name in meta["cases"]:
        md = meta["meta"][name]
        A = g[name + "_A"]
        f = P.sor_svd_power(A, md["k"], P.SketchConfig(md["ell"], md["q"], md["seed"]), fp64_mode="ozaki", ctx=ctx)
        assert f.stats["pass_kind"] == 1 and f.stats["oz_planes"] == int(planes)
        _, ds, dl = O.perturbation_floor(A, md["k"], O.SketchConfig(md["ell"], md["q"], md["seed"]))
        base = type("B", (), {"sigma": g[name + "_s"], "u": g[name + "_u"], "v": g[name + "_v"]})
        _check_parity(f, base, ds, dl)


@pytest.mark.parametrize("m,n,k,ell,q,sp", [(400, 300, 10, 10, 0, False), (300, 400, 10, 14, 2, False),
                                            (2001, 1500, 50, 60, 1, False), (2001, 1500, 50, 60, 1, True),
                                            (64, 1000, 8, 8, 1, False)])
def test_ozaki_shapes_vs_oracle(P, m, n, k, ell, q, sp):
    A = O.gen_lowrank_decay(m, n, min(m, n) - 1 if min(m, n) < 40 else 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + n)
    cfg = O.SketchConfig(ell, q, 17, single_pass=sp)
    base, ds, dl = O.perturbation_floor(A, k, cfg)
    f = P.sor_svd_power(A, k, P.SketchConfig(ell, q, 17, single_pass=sp), fp64_mode="ozaki")
    _check_parity(f, base, ds, dl)


def test_ozaki_config3_scaled_k256_and_f32(P):
    import torch
    A = O.gen_lowrank_decay(20000, 2000, 256, lambda j: 10.0 ** (-j / 64.0), 1e-3, 3)
    cfg = O.SketchConfig(256, 1, 31)
    base, ds, dl = O.perturbation_floor(A, 256, cfg, trials=1)
    f = P.sor_svd_power(A, 256, P.SketchConfig(256, 1, 31), fp64_mode="ozaki")
    _check_parity(f, base, ds, dl)
    a32 = A.astype(np.float32)
    base32 = O.sor_svd_power(a32.astype(np.float64), 256, cfg)
    f32 = P.sor_svd_power(torch.from_numpy(a32).cuda(), 256, P.SketchConfig(256, 1, 31), fp64_mode="ozaki")
    _check_parity(f32, base32, ds, dl)


def test_ozaki_k512(P):
    A = O.gen_lowrank_decay(4096, 3000, 512, lambda j: 1.0 / j, 1e-6, 5)
    cfg = O.SketchConfig(512, 1, 41)
    base, ds, dl = O.perturbation_floor(A, 512, cfg, trials=1, qr_variants=2)
    f = P.sor_svd_power(A, 512, P.SketchConfig(512, 1, 41), fp64_mode="ozaki")
    env = np.maximum.accumulate(ds)
    es = O.sigma_rel_err(f.sigma, base.sigma)
    assert np.all(es <= np.maximum(1e-10, 10 * env)), es.max()


def test_auto_mode_selection(P):
    import torch
    small = O.gen_lowrank_decay(400, 300, 20, lambda j: 1.0 / j, 1e-6, 2)
    assert P.sor_svd_power(small, 10, P.SketchConfig(10, 1, 1)).stats["pass_kind"] == 0    # auto -> DMMA
    assert P.sor_svd_power(small, 10, P.SketchConfig(10, 1, 1), fp64_mode="ozaki").stats["pass_kind"] == 1
    big = torch.randn(20000, 20000, dtype=torch.float64, device="cuda")                  # m n ell = 2^36.2
    f = P.sor_svd_power(big, 200, P.SketchConfig(200, 0, 1))
    assert f.stats["pass_kind"] == 1
    assert P.sor_svd_power(big, 200, P.SketchConfig(200, 0, 1), fp64_mode="dmma").stats["pass_kind"] == 0
    g = P.sor_svd_power(big, 200, P.SketchConfig(200, 0, 1), fp64_mode="dmma")
    np.testing.assert_allclose(f.sigma.cpu().numpy(), g.sigma.cpu().numpy(), rtol=1e-12)


@pytest.mark.parametrize("f32", [False, True])
def test_host_call_pipelined_upload(P, f32):
    """Host-buffer calls of the planes engine upload A in row chunks and convert / sweep each chunk as it lands.
    With only the first pass T1 = A Omega under the upload (OPT_UPLOAD_TN = 0; rows are independent) the result
    equals the device-resident call bit for bit, for several chunk sizes (one chunk, ragged last chunk, many
    chunks). With the first A^T T1 pass chunked too (default; its K ranges are added in chunk order) the call is
    repeatable bit for bit and agrees with the device call to rounding."""
    import torch
    A = O.gen_lowrank_decay(30000, 600, 40, lambda j: 2.0 ** (-j / 5), 1e-3, 17)
    if f32:
        A = A.astype(np.float32)
    cfg = P.SketchConfig(40, 1, 5)
    dev = P.sor_svd_power(torch.from_numpy(A).cuda(), 32, cfg, fp64_mode="ozaki")
    assert dev.stats["oz_planes"] == 1
    ds, du, dv = dev.sigma.cpu().numpy(), dev.u.cpu().numpy(), dev.v.cpu().numpy()
    for mb in (1536, 24, 2):
        ctx = P.Context(0)
        ctx.set_option(P.Context.OPT_UPLOAD_CHUNK_MB, mb)
        ctx.set_option(P.Context.OPT_UPLOAD_TN, 0)
        host = P.sor_svd_power(A, 32, cfg, fp64_mode="ozaki", ctx=ctx)
        assert host.stats["oz_planes"] == 1
        assert np.array_equal(np.asarray(host.sigma), ds)
        assert np.array_equal(np.asarray(host.u), du)
        assert np.array_equal(np.asarray(host.v), dv)
        host2 = P.sor_svd_power(A, 32, cfg, fp64_mode="ozaki", ctx=ctx)   # a second call on the same context
        assert np.array_equal(np.asarray(host2.u), np.asarray(host.u))
        ctx.set_option(P.Context.OPT_UPLOAD_TN, 1)
        h1 = P.sor_svd_power(A, 32, cfg, fp64_mode="ozaki", ctx=ctx)
        h2 = P.sor_svd_power(A, 32, cfg, fp64_mode="ozaki", ctx=ctx)
        assert np.array_equal(np.asarray(h1.u), np.asarray(h2.u)) and np.array_equal(np.asarray(h1.sigma), np.asarray(h2.sigma))
        assert O.sigma_rel_err(np.asarray(h1.sigma), ds).max() <= 1e-12
        assert O.lowrank_rel_diff(np.asarray(h1.u), np.asarray(h1.sigma), np.asarray(h1.v), du, ds, dv) <= 1e-11
    # q = 0 (no A^T pass before the QR) and single_pass keep the first-pass-only pipeline
    ctx = P.Context(0)
    ctx.set_option(P.Context.OPT_UPLOAD_CHUNK_MB, 8)
    for c0 in (P.SketchConfig(40, 0, 5), P.SketchConfig(40, 1, 5, single_pass=True)):
        d0 = P.sor_svd_power(torch.from_numpy(A).cuda(), 32, c0, fp64_mode="ozaki")
        h0 = P.sor_svd_power(A, 32, c0, fp64_mode="ozaki", ctx=ctx)
        assert np.array_equal(np.asarray(h0.sigma), d0.sigma.cpu().numpy())


@pytest.mark.parametrize("m,n,ell,ta", [(3000, 2000, 256, 0), (2000, 3000, 256, 1), (1500, 900, 136, 0), (70000, 600, 128, 1),
                                        (700, 500, 512, 0)])
def test_ozaki_planes_multicast_same_bits(P, m, n, ell, ta):
    """SORSVD_OPT_OZAKI_MULTICAST: the column-chunk CTAs of a row tile as one cluster sharing the A planes by TMA
    multicast (clusters of 2, 3, 4 and 8 CTAs, split-K) give the bits of the one-CTA-per-tile pass."""
    import torch
    buf, A, X = _operands(m, n, ell, ta, m + n + ell)
    outs = []
    for mc in (0, 1):
        ctx = P.Context(0)
        ctx.set_option(P.Context.OPT_OZAKI_MULTICAST, mc)
        ctx.set_stream(torch.cuda.current_stream(0).cuda_stream)
        Np = _npad(ell)
        T = torch.full(((n if ta else m), Np), float("nan"), device="cuda", dtype=torch.float64)
        ms, msc = ctypes.c_double(), ctypes.c_double()
        P._check(P._capi.lib().sorsvd_pass_ozaki_device(ctx.handle, ta, m, n, n, ell, 0, buf.data_ptr(), X.data_ptr(),
                                                         T.data_ptr(), 1, ctypes.byref(ms), ctypes.byref(msc)), ctx.handle)
        torch.cuda.synchronize()
        outs.append(T)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("m,n,ell,ta,f32", [(4000, 3000, 256, 0, False), (4000, 3000, 256, 1, False), (3001, 999, 64, 1, False),
                                            (5000, 2000, 136, 0, True), (5000, 2000, 136, 1, True), (40000, 600, 512, 1, False)])
def test_ozaki_partial_planes(P, m, n, ell, ta, f32):
    """Planes for the leading rows only (what fits in HBM: config 5 on one GPU), the in-pass converter for
    the rest: NN writes the two row ranges, TN sums the two K ranges. OPT_OZAKI_PLANES > 1 caps the rows."""
    import torch
    buf, A, X = _operands(m, n, ell, ta, m + 3 * n + ell, None, f32)
    T = _pass(P, buf, X, ta, m, n, ell, dtype=1 if f32 else 0, planes=1280)
    A64 = A.double()
    ref = (A64.T if ta else A64) @ X
    K = m if ta else n
    amax = A64.abs().amax() if ta else A64.abs().amax(dim=1)[:, None]
    xmax = X.abs().amax(dim=0).clamp_min(1e-300)
    err = (T - ref).abs()[:, :ell] / (amax * xmax[None, :ell] * np.sqrt(K)).clamp_min(1e-300)
    assert not torch.isnan(T[:, :ell]).any()
    assert err.max().item() <= PASS_TOL, err.max().item()
    again = _pass(P, buf, X, ta, m, n, ell, dtype=1 if f32 else 0, planes=1280)
    assert torch.equal(T, again)


def test_ozaki_partial_planes_whole_call(P):
    import torch
    A = O.gen_lowrank_decay(6000, 1500, 40, lambda j: 2.0 ** (-j / 4), 1e-3, 23)
    cfg = O.SketchConfig(48, 2, 9)
    base, ds, dl = O.perturbation_floor(A, 40, cfg)
    ctx = P.Context(0)
    ctx.set_option(P.Context.OPT_OZAKI_PLANES, 2560)
    f = P.sor_svd_power(torch.from_numpy(A).cuda(), 40, P.SketchConfig(48, 2, 9), fp64_mode="ozaki", ctx=ctx)
    assert f.stats["pass_kind"] == 1 and f.stats["oz_planes"] == 2
    _check_parity(f, base, ds, dl)
    h = P.sor_svd_power(A, 40, P.SketchConfig(48, 2, 9), fp64_mode="ozaki", ctx=ctx)   # host call: no pipelined upload
    assert np.array_equal(np.asarray(h.sigma), f.sigma.cpu().numpy())


def test_chunked_first_pass_keeps_split_k_bits(P):
    """The first pass T1 = A Omega run by row chunks (conversion under the pass, SORSVD_OPT_OZAKI_OVERLAP; host
    calls: under the upload) keeps the K partition of the one-launch pass: a long K (n = 4096) and a short last
    chunk, for which the split-K heuristic alone would pick another partition, give the same bits with the
    overlap on and off and through the host-buffer call."""
    import torch
    m, n, ell = 40000, 4096, 64
    A = P.gen_lowrank_device(m, n, 2.0 ** (-np.arange(1, 31) / 4.0), 1e-3, 91, x_scale=m ** -0.5, y_scale=n ** -0.5)
    cfg = P.SketchConfig(ell, 1, 3)
    outs = []
    for ov in (1, 0):
        ctx = P.Context(0)
        ctx.set_option(P.Context.OPT_OZAKI_OVERLAP, ov)
        f = P.sor_svd_power(A, 48, cfg, fp64_mode="ozaki", ctx=ctx)
        assert f.stats["oz_planes"] == 1
        outs.append((f.sigma.cpu().numpy(), f.u.cpu().numpy(), f.v.cpu().numpy()))
        ctx.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    ctx = P.Context(0)
    ctx.set_option(P.Context.OPT_UPLOAD_CHUNK_MB, 300)   # 9156-row chunks: 4 full + one ragged
    ctx.set_option(P.Context.OPT_UPLOAD_TN, 0)
    h = P.sor_svd_power(A.cpu().numpy(), 48, cfg, fp64_mode="ozaki", ctx=ctx)
    assert np.array_equal(np.asarray(h.sigma), outs[0][0]) and np.array_equal(np.asarray(h.u), outs[0][1])
    ctx.close()
