"""The spec's RPCA surface beside rpca_alm: estimate_rank_bound,
rpca_default_config's ell rule and the per-iteration telemetry, against the numpy oracle
restatement (oracle/sorsvd_oracle.py; the reference ships no RPCA code)."""
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


def test_estimate_rank_bound_spec_examples(P):
    import torch
    u = O.gaussian_matrix(300, 1, 1)
    v = O.gaussian_matrix(120, 1, 2)
    assert P.estimate_rank_bound(u @ v.T) == 1                       # rank 1 -> 1
    assert P.estimate_rank_bound(np.eye(64)) == 64                   # I_n -> n
    assert P.estimate_rank_bound(torch.eye(3, dtype=torch.float64, device="cuda")) == 3
    for shape, seed in [((200, 50), 3), ((50, 200), 4), ((512, 512), 5), ((7, 1), 6)]:
        x = O.gaussian_matrix(*shape, seed)
        assert P.estimate_rank_bound(x) == O.estimate_rank_bound(x)
    lowrank = O.gaussian_matrix(400, 5, 7) @ O.gaussian_matrix(5, 300, 8)
    assert P.estimate_rank_bound(lowrank) <= 5
    with pytest.raises(P.ParameterError):
        P.estimate_rank_bound(np.zeros((10, 8)))
    with pytest.raises(P.UnsupportedError):
        P.estimate_rank_bound(torch.zeros(600, 600, dtype=torch.float64, device="cuda") + 1.0)


def test_rpca_default_config(P):
    x = O.gaussian_matrix(500, 5, 11) @ O.gaussian_matrix(5, 500, 12)
    cfg = P.rpca_default_config(x)
    assert cfg.lam == pytest.approx(1.0 / np.sqrt(500))
    assert cfg.tol == 1e-7 and cfg.rho == 1.6 and cfg.max_iter == 500 and cfg.q == 1
    r = P.estimate_rank_bound(x)
    assert cfg.ell == min(2 * r, 499) and cfg.ell <= 10             # exactly rank-5 X -> at most 2r = 10
    assert P.rpca_default_config(25344, 300).ell == 10               # caller-chosen sketch size form


@pytest.mark.parametrize("m,n,r,frac", [(120, 90, 4, 0.05), (300, 200, 6, 0.1)])
def test_rpca_telemetry_vs_oracle(P, m, n, r, frac):
    rng = np.random.default_rng(m + n)
    l0 = O.gaussian_matrix(m, r, 21) @ O.gaussian_matrix(r, n, 22)
    s0 = np.zeros(m * n)
    idx = rng.choice(m * n, int(frac * m * n), replace=False)
    s0[idx] = rng.uniform(-50, 50, idx.size)
    d = l0 + s0.reshape(m, n)
    mu0 = 1.25 / np.linalg.norm(d, 2)
    cfg = dict(lam=1.0 / np.sqrt(max(m, n)), mu0=mu0, ell=2 * r, q=1, seed=5, max_iter=60)
    ref = O.rpca_alm(d, O.RpcaConfig(**cfg))
    got = P.rpca_alm(d, P.RpcaConfig(mu_bar_factor=1e7, rho=1.6, tol=1e-7, **cfg))
    assert got.iterations == ref.iterations and got.converged == ref.converged
    t, rt = got.telemetry, ref.telemetry
    assert t.shape == rt.shape == (ref.iterations, 5)
    assert np.array_equal(t[:, 0], np.arange(1, ref.iterations + 1))
    np.testing.assert_allclose(t[:, 1], rt[:, 1], rtol=1e-15)        # mu_k: the data-independent schedule
    np.testing.assert_allclose(t[:, 2], rt[:, 2], rtol=1e-6, atol=1e-15)  # ||D - L - S||_F / ||D||_F per iteration
    assert np.array_equal(t[:, 3], rt[:, 3])                         # rank_l per iteration
    assert np.array_equal(t[:, 4], rt[:, 4])                         # nnz_s per iteration
    assert t[-1, 3] == got.rank_l and t[-1, 4] == got.nnz_s and t[-1, 2] == pytest.approx(got.rel_error, rel=1e-12)
    csv = got.telemetry_csv().splitlines()
    assert csv[0] == "iter,mu,rel_error,rank_l,nnz_s" and len(csv) == ref.iterations + 1
    # a device-resident call fills the same rows
    import torch
    got_d = P.rpca_alm(torch.from_numpy(d).cuda(), P.RpcaConfig(mu_bar_factor=1e7, rho=1.6, tol=1e-7, **cfg))
    assert np.array_equal(got_d.telemetry, t)


def test_rpca_zero_matrix_telemetry(P):
    got = P.rpca_alm(np.zeros((40, 30)), P.RpcaConfig(lam=0.1, mu0=1.0, ell=4, q=1, seed=1, max_iter=10,
                                                      mu_bar_factor=1e7, rho=1.6, tol=1e-7))
    assert got.iterations == 1 and got.converged and got.telemetry.shape == (1, 5)
