"""GPU parity for the baselines of sketch.hpp: r_svd (:124-136) and tsr_svd
(:139-149), through the C ABI, against the compiled-reference golden vectors
and the numpy restatement on the same seeded inputs. Tolerances as for
sor_svd_power: sigma rel <= 1e-10 and low-rank rel <= 1e-9, raised to 10x
the perturbation floor of the algorithm itself where its sketch tail is
rounding noise (oracle.baseline_floor)."""
import numpy as np
import pytest

from oracle import sorsvd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_00462_b200 as P
    return P


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def _check(f, base_s, base_u, base_v, ds, dl, tol_s=1e-10, tol_lr=1e-9):
    s = _np(f.sigma)
    es = O.sigma_rel_err(s, base_s)
    lim = np.maximum(tol_s, 10 * np.maximum.accumulate(ds))
    assert np.all(es <= lim), (es.max(), int(np.argmax(es / lim)))
    lr = O.lowrank_rel_diff(_np(f.u), s, _np(f.v), base_u, base_s, base_v)
    assert lr <= max(tol_lr, 10 * dl), lr
    u, v = _np(f.u), _np(f.v)
    k = s.size
    assert np.abs(u.T @ u - np.eye(k)).max() < 1e-12 and np.abs(v.T @ v - np.eye(k)).max() < 1e-12
    assert np.all(np.diff(s) <= 0)
    return es.max(), lr


def _run(P, kind, A, ell, q, seed, **kw):
    return P.r_svd(A, ell, q, seed, **kw) if kind == "rsvd" else P.tsr_svd(A, ell, seed, **kw)


@pytest.mark.parametrize("kind", ["rsvd", "tsr"])
def test_baseline_golden_host_api(P, golden, kind):
    g, meta = golden
    for name in [n for n in meta["bl_cases"] if meta["meta"][n]["kind"] == kind]:
        md = meta["meta"][name]
        A = g[name + "_A"]
        f = _run(P, kind, A, md["ell"], md["q"], md["seed"])
        assert f.passes == md["passes"] and int(f.method) == md["method"]
        _, ds, dl = O.baseline_floor(kind, A, md["ell"], md["q"], md["seed"])
        _check(f, g[name + "_s"], g[name + "_u"], g[name + "_v"], ds, dl)


@pytest.mark.parametrize("kind,m,n,ell,q", [("rsvd", 400, 300, 12, 0), ("rsvd", 300, 500, 20, 1),
                                            ("rsvd", 2000, 1500, 60, 1), ("rsvd", 1000, 64, 8, 2),
                                            ("tsr", 400, 300, 12, 0), ("tsr", 300, 500, 20, 0),
                                            ("tsr", 2000, 1500, 60, 0), ("tsr", 64, 1000, 8, 0)])
def test_baseline_device_vs_oracle(P, kind, m, n, ell, q):
    import torch
    A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + n + ell)
    base, ds, dl = O.baseline_floor(kind, A, ell, q, 29)
    f = _run(P, kind, torch.from_numpy(A).cuda(), ell, q, 29)
    assert f.u.shape == (m, ell) and f.v.shape == (n, ell) and f.sigma.shape == (ell,)
    _check(f, base.sigma, base.u, base.v, ds, dl)
    # graph replay and un-graphed issue give the same bits
    f2 = _run(P, kind, torch.from_numpy(A).cuda(), ell, q, 29, use_graph=False)
    assert torch.equal(f.sigma, f2.sigma) and torch.equal(f.u, f2.u) and torch.equal(f.v, f2.v)


def test_rsvd_full_svd_sign_convention(P):
    # full_svd(B) canonicalises B's left factor (dense.hpp:80-95): U_B = Qy^T U has a positive
    # largest-magnitude entry in every column; on a well-separated spectrum the raw factors match
    A = O.gen_lowrank_decay(500, 400, 12, lambda j: 2.0 ** (-j), 1e-9, 3)
    f = P.r_svd(A, 12, 1, 5)
    r = O.r_svd(A, 12, 1, 5)
    np.testing.assert_allclose(f.sigma, r.sigma, rtol=1e-11)
    np.testing.assert_allclose(f.u[:, :8], r.u[:, :8], atol=1e-9)
    np.testing.assert_allclose(f.v[:, :8], r.v[:, :8], atol=1e-9)


def test_tsr_explicit_test_matrices_equal_seeded(P):
    A = O.gaussian_matrix(150, 110, 8)
    f1 = P.tsr_svd(A, 10, 77)
    f2 = P.tsr_svd(A, 10, 5, psi1=O.gaussian_matrix(110, 10, 77), psi2=O.gaussian_matrix(150, 10, 77 ^ 1))
    np.testing.assert_array_equal(f1.sigma, f2.sigma)
    np.testing.assert_array_equal(f1.u, f2.u)
    om = O.gaussian_matrix(110, 10, 61)
    r1 = P.r_svd(A, 10, 1, 61)
    r2 = P.r_svd(A, 10, 1, 3, omega=om)
    np.testing.assert_array_equal(r1.sigma, r2.sigma)


def test_baseline_fp32_storage_vs_oracle(P):
    # FP32-stored A, FP64 arithmetic: the FP64 oracle on the rounded matrix
    A = O.gen_lowrank_decay(900, 700, 30, lambda j: 2.0 ** (-j / 3), 1e-4, 12).astype(np.float32)
    A64 = A.astype(np.float64)
    for kind, q in (("rsvd", 1), ("tsr", 0)):
        base, ds, dl = O.baseline_floor(kind, A64, 24, q, 41)
        f = _run(P, kind, A, 24, q, 41)
        _check(f, base.sigma, base.u, base.v, ds, dl)


def test_truncate_and_errors(P):
    A = O.gaussian_matrix(60, 40, 2)
    f = P.r_svd(A, 8, 0, 1)
    t = P.truncate(f, 3)
    assert t.u.shape == (60, 3) and t.v.shape == (40, 3)
    np.testing.assert_array_equal(t.sigma, f.sigma[:3])
    with pytest.raises(P.ParameterError):
        P.truncate(f, 9)
    with pytest.raises(P.ParameterError):  # ell < min(m, n) (sketch.hpp:67)
        P.r_svd(A, 40, 0, 1)
    with pytest.raises(P.ParameterError):
        P.tsr_svd(A, 0, 1)
    with pytest.raises(P.ParameterError):
        P.r_svd(A, 5, -1, 1)
    with pytest.raises(P.ParameterError):
        P.tsr_svd(A, 5, 1, psi1=O.gaussian_matrix(40, 5, 1))


def test_approx_error_frobenius_vs_reference(P, golden):
    # approx_error(a, x, frobenius) (sketch.hpp:168-172), one fused pass over A on the device,
    # against the compiled reference evaluated on the same factors
    import torch
    g, meta = golden
    for name in meta["cases"][:3] + ["c1"]:
        if name == "c1":
            A, u, s, v = O.gen_c1(1), g["c1_u"], g["c1_s"], g["c1_v"]
        else:
            A, u, s, v = g[name + "_A"], g[name + "_u"], g[name + "_s"], g[name + "_v"]
        x = O.LowRankApprox(u, s, v, 0, 0, len(s), 0, 0)
        ref = O.Ref.approx_error(A, u, s, v, 0) if O.os.path.exists(O.REF_LIB_PATH) else O.approx_error(A, x)
        got = P.approx_error(A, x)
        assert abs(got - ref) <= 1e-10 * ref, (name, got, ref)
        got_dev = P.approx_error(torch.from_numpy(A).cuda(), x)
        assert got_dev == got
    # FP32-stored A: the FP64 oracle on the rounded matrix
    A = O.gen_lowrank_decay(700, 500, 30, lambda j: 2.0 ** (-j / 3), 1e-3, 4).astype(np.float32)
    f = P.sor_svd_power(A, 20, P.SketchConfig(24, 1, 2))
    ref = O.approx_error(A.astype(np.float64), O.LowRankApprox(f.u, f.sigma, f.v, 0, 0, 20, 0, 0))
    assert abs(P.approx_error(A, f) - ref) <= 1e-10 * ref
    # the spectral norm of the difference (device Gram / Rayleigh-Ritz estimate) vs dgesdd
    ref2 = np.linalg.norm(A.astype(np.float64) - (f.u * f.sigma) @ f.v.T, 2)
    assert abs(P.approx_error(A, f, "spectral") - ref2) <= 1e-9 * ref2
    with pytest.raises(P.ParameterError):
        P.approx_error(A, f, "nuclear")
    with pytest.raises(P.ShapeError):
        P.approx_error(A[:100], f)
