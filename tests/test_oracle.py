"""CPU: pin the oracle restatements (oracle/c, oracle/sorsvd_oracle.py)
against the golden vectors produced by the compiled reference, and against
the compiled reference itself when oracle/_ref is present."""
import numpy as np
import pytest

from oracle import sorsvd_oracle as O


def test_gaussian_matrix_bit_exact(golden):
    g, _ = golden
    assert np.array_equal(O.gaussian_matrix(7, 5, 123), g["gauss_7x5_s123"])
    assert np.array_equal(O.gaussian_matrix(3, 3, 0), g["gauss_3x3_s0"])
    assert np.array_equal(O.gaussian_matrix(1, 9, 2**64 - 1), g["gauss_1x9_smax"])


def test_sub_seed(golden):
    g, _ = golden
    got = [O.sub_seed(s, t) for s in (0, 1, 42, 2**63) for t in (0, 1, 2, 3)]
    assert np.array_equal(np.array(got, dtype=np.uint64), g["sub_seeds"])


def test_gaussian_moments():
    # determinism and moments of the draw
    x = O.gaussian_matrix(500, 400, 99)
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1) < 0.01
    assert np.array_equal(x, O.gaussian_matrix(500, 400, 99))


def test_flop_estimate(golden):
    g, _ = golden
    assert O.flop_estimate(1000, 1000, 38, 20, 0, 0) == 239813744
    args = [(1000, 1000, 38, 20, 0), (4000, 4000, 100, 100, 1), (200000, 20000, 256, 256, 1), (25344, 300, 10, 10, 1)]
    got = [[O.flop_estimate(*a, v) for v in range(4)] for a in args]
    assert np.array_equal(np.array(got, dtype=np.int64), g["flops"])
    with pytest.raises(O.ParameterError):
        O.flop_estimate(0, 1, 1, 1, 0, 0)


def test_dense_kats(golden):
    g, _ = golden
    np.testing.assert_allclose(g["matmul_kat"], [[17.0], [39.0]])
    q, r = O.thin_qr(np.array([[3.0], [4.0]]))
    np.testing.assert_allclose(q, g["qr34_q"], atol=1e-15)
    np.testing.assert_allclose(r, g["qr34_r"], atol=1e-15)
    np.testing.assert_allclose(g["qr34_q"].ravel(), [0.6, 0.8], atol=1e-15)
    u, s, v = O.full_svd(np.diag([3.0, 2.0, 1.0]))
    np.testing.assert_allclose(s, g["svd321_s"], atol=1e-15)
    np.testing.assert_allclose(u, g["svd321_u"], atol=1e-15)
    q, r = O.thin_qr(g["qr50x10_a"])
    np.testing.assert_allclose(q, g["qr50x10_q"], atol=1e-13)
    np.testing.assert_allclose(r, g["qr50x10_r"], atol=1e-12)
    u, s, v = O.full_svd(g["svd20_m"])
    np.testing.assert_allclose(s, g["svd20_s"], rtol=1e-13)
    np.testing.assert_allclose(u, g["svd20_u"], atol=1e-12)
    np.testing.assert_allclose(v, g["svd20_v"], atol=1e-12)


def test_sor_svd_power_port_matches_reference_golden(golden):
    g, meta = golden
    for name in meta["cases"]:
        md = meta["meta"][name]
        f = O.sor_svd_power(g[name + "_A"], md["k"], O.SketchConfig(md["ell"], md["q"], md["seed"]))
        assert f.passes == md["passes"] and f.method == md["method"]
        # tolerance = max(tight, 10 x the reference's own perturbation floor)
        _, ds, dl = O.perturbation_floor(g[name + "_A"], md["k"], O.SketchConfig(md["ell"], md["q"], md["seed"]))
        tol_s = np.maximum(1e-11, 10 * ds)
        assert np.all(O.sigma_rel_err(f.sigma, g[name + "_s"]) <= tol_s), name
        assert O.lowrank_rel_diff(f.u, f.sigma, f.v, g[name + "_u"], g[name + "_s"], g[name + "_v"]) <= max(1e-10, 10 * dl), name


def test_single_pass_port_matches_reference_golden(golden):
    # m_approx + pseudo_inverse (sketch.hpp:54-58, dense.hpp:138-157), 2q+2 passes
    g, meta = golden
    assert len(meta["sp_cases"]) == 3
    for name in meta["sp_cases"]:
        md = meta["meta"][name]
        cfg = O.SketchConfig(md["ell"], md["q"], md["seed"], single_pass=True)
        f = O.sor_svd_power(g[name + "_A"], md["k"], cfg)
        assert f.passes == md["passes"] == 2 * md["q"] + 2
        _, ds, dl = O.perturbation_floor(g[name + "_A"], md["k"], cfg)
        assert np.all(O.sigma_rel_err(f.sigma, g[name + "_s"]) <= np.maximum(1e-11, 10 * ds)), name
        assert O.lowrank_rel_diff(f.u, f.sigma, f.v, g[name + "_u"], g[name + "_s"], g[name + "_v"]) <= max(1e-10, 10 * dl), name


@pytest.mark.parametrize("kind", ["rsvd", "tsr"])
def test_baselines_port_match_reference_golden(golden, kind):
    # r_svd (sketch.hpp:124-136) and tsr_svd (sketch.hpp:139-149) restated in numpy vs the compiled reference
    g, meta = golden
    names = [n for n in meta["bl_cases"] if meta["meta"][n]["kind"] == kind]
    assert len(names) == 3
    for name in names:
        md = meta["meta"][name]
        A = g[name + "_A"]
        f = O.r_svd(A, md["ell"], md["q"], md["seed"]) if kind == "rsvd" else O.tsr_svd(A, md["ell"], md["seed"])
        assert f.passes == md["passes"] == (2 * md["q"] + 2 if kind == "rsvd" else 1)
        assert f.method == md["method"] == (O.RSVD if kind == "rsvd" else O.TSR)
        _, ds, dl = O.baseline_floor(kind, A, md["ell"], md["q"], md["seed"], include_reference=False)
        assert np.all(O.sigma_rel_err(f.sigma, g[name + "_s"]) <= np.maximum(1e-11, 10 * ds)), name
        assert O.lowrank_rel_diff(f.u, f.sigma, f.v, g[name + "_u"], g[name + "_s"], g[name + "_v"]) <= max(1e-10, 10 * dl), name


def test_approx_error_port_vs_reference(ref_available):
    # sketch.hpp:168-172 on a sor_svd_power result: restatement vs the compiled reference
    if not ref_available:
        pytest.skip("oracle/_ref not built")
    a = O.gen_lowrank_decay(120, 90, 20, lambda j: 2.0 ** (-j / 2), 1e-4, 8)
    f = O.sor_svd_power(a, 10, O.SketchConfig(12, 1, 3))
    for kind, code in (("frobenius", 0), ("spectral", 1)):
        r = O.Ref.approx_error(a, f.u, f.sigma, f.v, code)
        assert abs(O.approx_error(a, f, kind) - r) <= 1e-12 * r


def test_truncate_rules():
    a = O.gaussian_matrix(30, 20, 3)
    f = O.r_svd(a, 6, 0, 1)
    t = O.truncate(f, 4)
    assert t.u.shape == (30, 4) and t.v.shape == (20, 4) and np.array_equal(t.sigma, f.sigma[:4])
    for k in (0, 7):
        with pytest.raises(O.ParameterError):
            O.truncate(f, k)


def test_rank1_exact(golden):
    # rank-1 100x80, k=1, ell=4 -> error <= 1e-10
    g, _ = golden
    f = O.sor_svd_power(g["rank1_A"], 1, O.SketchConfig(4, 0, 93))
    err = np.linalg.norm(g["rank1_A"] - (f.u * f.sigma) @ f.v.T) / np.linalg.norm(g["rank1_A"])
    assert err < 1e-10
    assert O.sigma_rel_err(f.sigma, g["rank1_s"]).max() < 1e-13


def test_c1_port_vs_reference(golden):
    g, meta = golden
    A = O.gen_c1(1)
    np.testing.assert_allclose([A.sum(), (A * A).sum(), A[123, 456]], g["c1_A_checksum"], rtol=1e-13)
    f = O.sor_svd_power(A, 20, O.SketchConfig(20, 0, 7))
    assert O.sigma_rel_err(f.sigma, g["c1_s"]).max() < 1e-12
    assert O.lowrank_rel_diff(f.u, f.sigma, f.v, g["c1_u"], g["c1_s"], g["c1_v"]) < 1e-11


def test_q0_power_equals_basic():
    # the q = 0 power path equals sor_svd
    a = O.gaussian_matrix(50, 30, 5)
    f1 = O.sor_svd_power(a, 4, O.SketchConfig(6, 0, 3))
    f2 = O.sor_svd(a, 4, O.SketchConfig(6, 0, 3))
    assert np.array_equal(f1.sigma, f2.sigma)
    with pytest.raises(O.ParameterError):
        O.sor_svd(a, 4, O.SketchConfig(6, 1, 3))


def test_validate_sketch_rules():
    # sketch.hpp:62-69
    for args in [(1, 5, 1, 1, 0), (5, 5, 0, 1, 0), (5, 5, 3, 2, 0), (5, 5, 2, 5, 0), (5, 5, 1, 2, -1)]:
        with pytest.raises(O.ParameterError):
            O.validate_sketch(*args)
    O.validate_sketch(5, 5, 2, 4, 0)


def test_rpca_restatement_golden(golden):
    g, meta = golden
    md = meta["meta"]["rpca100"]
    cfg = O.RpcaConfig(lam=md["lam"], mu0=md["mu0"], ell=md["ell"], q=md["q"], seed=md["seed"], max_iter=100)
    r = O.rpca_alm(g["rpca100_X"], cfg)
    assert r.iterations == md["iterations"] and r.rank_l == md["rank"] and r.nnz_s == md["nnz"]
    assert r.converged
    np.testing.assert_allclose(r.l, g["rpca100_L"], atol=1e-8 * np.abs(g["rpca100_L"]).max())
    np.testing.assert_allclose(r.s, g["rpca100_S"], atol=1e-8 * 50)


def test_soft_threshold():
    # SPEC.md rpca soft_threshold examples
    np.testing.assert_allclose(O.soft_threshold(1.2, 0.5), 0.7)
    np.testing.assert_allclose(O.soft_threshold(-1.2, 0.5), -0.7)
    assert O.soft_threshold(0.3, 0.5) == 0.0


def test_port_vs_compiled_reference_live(ref_available):
    if not ref_available:
        pytest.skip("oracle/_ref not built")
    Ref = O.Ref
    Ref.set_threads(1)
    a = O.gen_lowrank_decay(300, 200, 20, lambda j: 10.0 ** (-j / 8), 1e-6, 9)
    for q in (0, 1, 2):
        cfg = O.SketchConfig(12, q, 100 + q)
        f = O.sor_svd_power(a, 10, cfg)
        r = Ref.sor_svd_power(a, 10, cfg)
        assert O.sigma_rel_err(f.sigma, r.sigma).max() < 1e-10
        assert O.lowrank_rel_diff(f.u, f.sigma, f.v, r.u, r.sigma, r.v) < 1e-9
    # C4-shaped generator uses Floyd sampling with exact count
    D, L0, S0 = O.gen_c4(4, m=500, n=60)
    assert np.count_nonzero(S0) == round(0.1 * 500 * 60)
    assert np.abs(S0).max() <= 50


@pytest.mark.parametrize("frac,lo,hi,nnz", [(0.05, 14, 20, 12500), (0.1, 16, 23, 25000)])
def test_rpca_paper_table_pins(ref_available, frac, lo, hi, nnz):
    # SPEC.md:393-394 / acceptance criteria 1-2 (Table IV / V, n = 500, r = 25):
    # rank(L) = 25, ||S||_0 = s, rel_error < 1e-7, iterations within [lo, hi] (paper: 17 / 20),
    # on matrixgen's RPCA instance (matrixgen.hpp:99-124) with l = 2r, q = 1
    if not ref_available:
        pytest.skip("oracle/_ref not built")
    n = 500
    x, _, s0 = O.Ref.gen_rpca_instance(n, 25, int(frac * n * n), 1)
    assert np.count_nonzero(s0) == nnz
    cfg = O.RpcaConfig(lam=1 / np.sqrt(n), mu0=1.25 / O.norm_spectral(x), ell=50, q=1, seed=1, max_iter=500)
    for r in (O.rpca_alm(x, cfg), O.Ref.rpca_alm(x, cfg)):
        assert r.converged and r.rel_error < 1e-7
        assert r.rank_l == 25 and r.nnz_s == nnz
        assert lo <= r.iterations <= hi, r.iterations
