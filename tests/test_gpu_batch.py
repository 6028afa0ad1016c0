"""GPU: batched trials (the Monte-Carlo loop of bounds.hpp:262-379: trial t
calls sor_svd_power with seed + t). Every pass over A serves all trials in
one launch; each trial must match the oracle (and the single call) on the
same A and the same host-drawn Omega_t, to the usual parity tolerances."""
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


def _check(f, base, ds, dl):
    s = _np(f.sigma)
    es = O.sigma_rel_err(s, base.sigma)
    lim = np.maximum(1e-10, 10 * np.maximum.accumulate(ds))
    assert np.all(es <= lim), (es.max(), int(np.argmax(es / lim)))
    lr = O.lowrank_rel_diff(_np(f.u), s, _np(f.v), base.u, base.sigma, base.v)
    assert lr <= max(1e-9, 10 * dl), lr


@pytest.mark.parametrize("m,n,k,ell,q,trials", [(400, 300, 10, 12, 1, 3), (300, 500, 8, 8, 0, 5),
                                                (2000, 1500, 50, 60, 1, 4), (1000, 64, 8, 8, 2, 9)])
def test_batch_trials_vs_oracle(P, m, n, k, ell, q, trials):
    import torch
    A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + n + trials)
    out = P.sor_svd_power_batch(torch.from_numpy(A).cuda(), k, P.SketchConfig(ell, q, 100), trials)
    assert len(out) == trials
    for t, f in enumerate(out):
        assert f.seed == 100 + t and f.passes == 2 * q + 3 and f.u.shape == (m, k) and f.v.shape == (n, k)
        base, ds, dl = O.perturbation_floor(A, k, O.SketchConfig(ell, q, 100 + t))
        _check(f, base, ds, dl)


def test_batch_matches_single_calls_and_host_api(P):
    import torch
    A = O.gen_lowrank_decay(700, 500, 30, lambda j: 2.0 ** (-j / 3), 1e-6, 3)
    seeds = [7, 99, 12345]
    dev = P.sor_svd_power_batch(torch.from_numpy(A).cuda(), 16, P.SketchConfig(20, 1, 0), 3, seeds=seeds)
    host = P.sor_svd_power_batch(A, 16, P.SketchConfig(20, 1, 0), 3, seeds=seeds)
    for t, s in enumerate(seeds):
        one = P.sor_svd_power(A, 16, P.SketchConfig(20, 1, s))
        np.testing.assert_array_equal(_np(dev[t].sigma), host[t].sigma)
        np.testing.assert_allclose(host[t].sigma, one.sigma, rtol=1e-11)
        assert O.lowrank_rel_diff(host[t].u, host[t].sigma, host[t].v, one.u, one.sigma, one.v) < 1e-10
    # explicit test matrices equal the seeded draws
    om = np.stack([O.gaussian_matrix(500, 20, s) for s in seeds])
    given = P.sor_svd_power_batch(A, 16, P.SketchConfig(20, 1, 0), 3, omegas=om)
    for t in range(3):
        np.testing.assert_array_equal(given[t].sigma, host[t].sigma)


def test_batch_fp32_storage(P):
    A = O.gen_lowrank_decay(900, 700, 30, lambda j: 2.0 ** (-j / 3), 1e-4, 12).astype(np.float32)
    out = P.sor_svd_power_batch(A, 20, P.SketchConfig(24, 1, 5), 2)
    for t, f in enumerate(out):
        base, ds, dl = O.perturbation_floor(A.astype(np.float64), 20, O.SketchConfig(24, 1, 5 + t))
        _check(f, base, ds, dl)


def test_batch_errors(P):
    A = O.gaussian_matrix(60, 40, 2)
    with pytest.raises(P.ParameterError):
        P.sor_svd_power_batch(A, 5, P.SketchConfig(8, 0, 1), 0)
    with pytest.raises(P.ParameterError):  # validate_sketch (sketch.hpp:62-69) applies per call
        P.sor_svd_power_batch(A, 5, P.SketchConfig(40, 0, 1), 2)
    with pytest.raises(P.ShapeError):
        P.sor_svd_power_batch(A, 5, P.SketchConfig(8, 0, 1), 2, seeds=[1, 2, 3])
