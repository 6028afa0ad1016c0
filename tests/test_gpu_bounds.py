"""The bound harness on the device (paper_1804_00462_b200/bounds.py: batched
sor_svd_power trials, device approx_error in both norms, device omega_split)
against the compiled reference's pieces (golden_bounds.npz; the experiment is
the oracle's restatement of bounds.hpp:265-379 around them, since the
reference's own omega_split reads a moved-from matrix -- oracle/ref_capi.cpp)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_00462_b200 as P
    from paper_1804_00462_b200 import bounds as B
    g = dict(np.load(os.path.join(GOLD, "golden_bounds.npz")))
    meta = json.load(open(os.path.join(GOLD, "golden_bounds_meta.json")))
    return P, B, g, meta


def test_spectral_norm_vs_lapack(env):
    import torch
    P, B, g, _ = env
    for shape in [(120, 80), (80, 120), (9, 12), (700, 12), (1500, 1100)]:
        a = torch.randn(*shape, dtype=torch.float64, device="cuda")
        ref = float(torch.linalg.matrix_norm(a, 2))
        assert P.norm(a, "spectral") == pytest.approx(ref, rel=1e-10)
        assert P.norm(a, "frobenius") == pytest.approx(float(a.norm()), rel=1e-13)


def test_approx_error_spectral_vs_reference(env):
    import torch
    P, B, g, _ = env
    a = torch.from_numpy(g["exp_A"]).cuda()
    x = P.sor_svd_power(a, 6, P.SketchConfig(12, 1, 4100))
    tv = g["expdet_trial_vals"][0]
    assert P.approx_error(a, x, "frobenius") == pytest.approx(tv[0], rel=1e-9)
    assert P.approx_error(a, x, "spectral") == pytest.approx(tv[1], rel=1e-9)


def test_omega_split_vs_reference(env):
    import torch
    P, B, g, meta = env
    sp = meta["split"]
    v = torch.from_numpy(g["exp_V"]).cuda()
    om = torch.from_numpy(P.gaussian_matrix(sp["n"], sp["ell"], sp["omega_seed"])).cuda()
    s = B.omega_split(v, om, B.BoundParams(sp["k"], sp["ell"], sp["p"], sp["q"]))
    n2, n1p, frr = g["split_norms"]
    assert s.full_row_rank == bool(frr)
    assert s.norm_omega2 == pytest.approx(n2, rel=1e-11)
    assert s.norm_omega1_pinv == pytest.approx(n1p, rel=1e-10)
    assert tuple(s.omega1.shape) == (sp["ell"] - sp["p"], sp["ell"]) and s.omega2.shape[0] == sp["n"] - sp["ell"] + sp["p"]


@pytest.mark.parametrize("name", ["expdet", "expavg"])
@pytest.mark.parametrize("own_svd", [True, False])
def test_bound_experiment_vs_reference(env, name, own_svd):
    import torch
    P, B, g, meta = env
    e = meta["experiment"]
    c = e[name]
    a = torch.from_numpy(g["exp_A"]).cuda()
    ref_svd = None if own_svd else (g["exp_sigma"], g["exp_V"])
    rep = B.bound_tightness_experiment(a, e["k"], B.BoundParams(e["k"], e["ell"], e["p"], c["q"]), c["trials"], c["seed"],
                                       kind=c["kind"], ref_svd=ref_svd, batch=4)
    tv, tf = g[f"{name}_trial_vals"], g[f"{name}_trial_flags"]
    got = np.array([[r.err_f, r.err_2, r.bound_f, r.bound_2] for r in rep.records])
    np.testing.assert_allclose(got[:, :2], tv[:, :2], rtol=1e-9)      # realized errors (north-star low-rank tolerance)
    np.testing.assert_allclose(got[:, 2:], tv[:, 2:], rtol=1e-8)      # bounds: Phi = (||O2|| ||O1^+||)^2
    assert [[r.satisfied_f, r.satisfied_2, r.full_row_rank] for r in rep.records] == tf.tolist()
    sc = g[f"{name}_scal"]
    assert rep.lowrank_bound_frobenius == pytest.approx(sc[0], rel=1e-8)
    assert rep.lowrank_bound_spectral == pytest.approx(sc[1], rel=1e-8)
    assert rep.realized_error_frobenius == pytest.approx(sc[2], rel=1e-9)
    assert rep.realized_error_spectral == pytest.approx(sc[3], rel=1e-9)
    np.testing.assert_allclose(rep.sv_lower_bounds, g[f"{name}_sv_lower_bounds"], rtol=1e-8)
    np.testing.assert_allclose(rep.realized_sigmas, g[f"{name}_realized_sigmas"], rtol=1e-10)
    assert rep.bound_satisfied == [bool(x) for x in g[f"{name}_bound_satisfied"]]
    assert all(rep.bound_satisfied)
    # every seed's record sits at its trial index, and the CSV has one row per trial + header + summary
    assert [r.seed for r in rep.records] == [c["seed"] + t for t in range(c["trials"])]
    assert B.bound_report_csv(rep).count("\n") == c["trials"] + 2


def test_interlacing_and_bounds_hold_polydecay(env):
    """SPEC.md:574 in small: Theorem 5's bound >= realized error, Theorem 3's lower bounds <= sigma_hat_j <= sigma_j."""
    import torch
    P, B, g, _ = env
    n = 200
    u, _ = torch.linalg.qr(torch.randn(300, n, dtype=torch.float64, device="cuda"))
    v, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda"))
    sg = 1.0 / torch.arange(1, n + 1, dtype=torch.float64, device="cuda")
    a = (u * sg) @ v.T
    for q in (0, 2):
        rep = B.bound_tightness_experiment(a, 10, B.BoundParams(10, 24, 6, q), 10, 900 + q, ref_svd=(sg.cpu().numpy(), v))
        assert rep.bound_satisfied[10] and rep.bound_satisfied[11], rep.bound_satisfied     # Theorem 5, both norms
        for r in rep.records:                                                               # interlacing
            assert all(sh <= 1.0 / (j + 1) + 1e-9 for j, sh in enumerate(r.sigma_hat))
        if q > 0:
            # Theorem 3's lower bounds; on this slowly decaying spectrum the q = 0 form (exponent 4,
            # bounds.hpp:103) is above the realized sigma_hat_1 for the reference as well
            assert all(rep.bound_satisfied), rep.bound_satisfied
            assert all(r.sv_satisfied for r in rep.records)
