"""f4: the device generators (gen_f64.cuh) against the host-exact draws: gaussian_matrix_device vs the
reference-exact host stream (a few ulp: device log / sincos), gen_lowrank_device vs the numpy restatement
(oracle.gen_lowrank_rows), gen_rpca_instance_device vs the compiled reference's gen_rpca_instance
(matrixgen.hpp:99-124: identical support and signs)."""
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


@pytest.mark.parametrize("rows,cols,seed", [(7, 5, 123), (1, 9, 2**64 - 1), (300, 257, 0), (1001, 3, 42)])
def test_gaussian_matrix_device_ulp_compatible(P, rows, cols, seed):
    g = P.gaussian_matrix_device(rows, cols, seed).cpu().numpy()
    h = O.gaussian_matrix(rows, cols, seed)
    # r = sqrt(-2 log u1) <= 8.6; cos / sin differ by a few ulp of 1: absolute 4e-15 covers r * 2 ulp
    np.testing.assert_allclose(g, h, rtol=0, atol=4e-15)
    assert np.mean(g == h) > 0.5          # most entries are bit-identical


@pytest.mark.parametrize("m,n,r,row0,mg,f32", [(300, 200, 8, 0, None, False), (130, 77, 5, 64, 400, False),
                                               (257, 129, 12, 3, 300, True)])
def test_gen_lowrank_device_vs_restatement(P, m, n, r, row0, mg, f32):
    import torch
    sg = 10.0 ** (-np.arange(1, r + 1) / 4.0)
    a = P.gen_lowrank_device(m, n, sg, 1e-3, 77, x_scale=1 / np.sqrt(mg or m), y_scale=1 / np.sqrt(n),
                             dtype=torch.float32 if f32 else torch.float64, row0=row0, m_global=mg or 0)
    ref = O.gen_lowrank_rows(m, n, sg, 1e-3, 77, 1 / np.sqrt(mg or m), 1 / np.sqrt(n), row0, mg)
    got = a.double().cpu().numpy()
    tol = 1e-7 * np.abs(ref).max() if f32 else 1e-15 * np.abs(ref).max() + 1e-3 * 4e-15
    assert np.abs(got - ref).max() <= tol
    # a row block of the global matrix is the same rows whichever rank generates them
    if row0:
        whole = P.gen_lowrank_device(row0 + m, n, sg, 1e-3, 77, x_scale=1 / np.sqrt(mg or m), y_scale=1 / np.sqrt(n),
                                     dtype=a.dtype, m_global=mg or 0)
        assert torch.equal(whole[row0:], a)


def test_gen_rpca_instance_device_vs_reference(P, ref_available):
    if not ref_available:
        pytest.skip("compiled reference not built")
    for n, r, s, seed in [(100, 5, 500, 77), (64, 3, 0, 1), (200, 10, 4000, 9)]:
        x, l, sp = P.gen_rpca_instance_device(n, r, s, seed)
        rx, rl, rs = O.Ref.gen_rpca_instance(n, r, s, seed)
        assert np.array_equal(sp.cpu().numpy(), rs)                       # support and +-50 values: identical
        np.testing.assert_allclose(l.cpu().numpy(), rl, rtol=0, atol=1e-13 * np.abs(rl).max())
        np.testing.assert_allclose(x.cpu().numpy(), rx, rtol=0, atol=1e-13 * np.abs(rx).max())
        assert int((sp != 0).sum()) == s
    with pytest.raises(P.ParameterError):
        P.gen_rpca_instance_device(10, 10, 5, 1)


def test_generated_c3_block_decomposes_like_the_oracle_one(P):
    """A C3-shaped block from the device generator through sor_svd_power vs the oracle on the same bytes."""
    import torch
    sg = 10.0 ** (-np.arange(1, 33) / 8.0)
    a = P.gen_lowrank_device(4000, 600, sg, 1e-3, 5, x_scale=1 / np.sqrt(4000), y_scale=1 / np.sqrt(600))
    f = P.sor_svd_power(a, 32, P.SketchConfig(32, 1, 3))
    ref = O.sor_svd_power(a.cpu().numpy(), 32, O.SketchConfig(32, 1, 3))
    assert O.sigma_rel_err(f.sigma.cpu().numpy(), ref.sigma).max() <= 1e-10
