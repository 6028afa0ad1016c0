"""GPU: the tcgen05 TF32 pass kernel (FP32 operands, FP32 accumulation in
TMEM) against an FP64 product of the same FP32 inputs. Tolerance: TF32
rounds each operand to 10 mantissa bits (unit roundoff 2^-11 = 4.9e-4), so
the relative Frobenius error of a length-K dot is ~2^-11 / sqrt(3) independent
of K; we require <= 2e-3 and also that the result is NOT bit-exact FP32
(i.e. it really ran on the tensor pipe)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_00462_b200 as P
    return P, torch


@pytest.mark.parametrize("M,K,N,ta", [(128, 32, 32, False), (1000, 700, 20, False), (4000, 4000, 100, False),
                                      (3000, 4000, 100, True), (257, 132, 256, False), (516, 2049, 256, True),
                                      (20000, 2000, 256, False), (2000, 20000, 256, True), (300, 9000, 512, True),
                                      (1024, 1024, 512, False), (131, 8, 8, False), (100, 5, 40, True)])
def test_tf32_gemm(env, M, K, N, ta):
    P, torch = env
    g = torch.Generator(device="cuda").manual_seed(M + 7 * K + N)
    a = torch.randn((K, M) if ta else (M, K), generator=g, device="cuda", dtype=torch.float32)
    b = torch.randn((K, N), generator=g, device="cuda", dtype=torch.float32)
    ref = (a.double().T if ta else a.double()) @ b.double()
    got = P.matmul(a, b, transpose_a=ta)
    torch.cuda.synchronize()
    rel = float(torch.linalg.norm(got.double() - ref) / torch.linalg.norm(ref))
    assert rel <= 2e-3, rel
    assert rel > 1e-9  # TF32, not an FP32 CUDA-core fallback


def test_tf32_gemm_requires_16B_rows(env):
    """cp.async.bulk.tensor needs 16-byte row pitch: lda % 4 == 0 (include/sorsvd_b200.h)."""
    P, torch = env
    a = torch.randn((257, 129), device="cuda", dtype=torch.float32)
    b = torch.randn((129, 32), device="cuda", dtype=torch.float32)
    with pytest.raises(P.ShapeError):
        P.matmul(a, b)


def test_sor_svd_fp32_vs_fp64_oracle(env):
    """Config-3 distributions at 1/10 x 1/10 scale, fp32 A, TF32 passes vs the
    FP64 oracle on the same (fp32-rounded) matrix. Stated tolerance for the
    TF32 path: sigma rel <= 3e-3 on the leading half of the
    spectrum, low-rank rel diff <= 3e-3 (measured 7.2e-4 / 8.7e-4)."""
    P, torch = env
    from oracle import sorsvd_oracle as O
    A = O.gen_lowrank_decay(20000, 2000, 256, lambda j: 10.0 ** (-j / 64.0), 1e-3, 3).astype(np.float32)
    Ad = A.astype(np.float64)
    base = O.sor_svd_power(Ad, 128, O.SketchConfig(128, 1, 31))
    f = P.sor_svd_power(torch.from_numpy(A).cuda(), 128, P.SketchConfig(128, 1, 31), fp32_mode="tf32")
    s = f.sigma.cpu().numpy()
    es = O.sigma_rel_err(s, base.sigma)
    assert es[:64].max() <= 3e-3, es[:64].max()
    lr = O.lowrank_rel_diff(f.u.cpu().numpy(), s, f.v.cpu().numpy(), base.u, base.sigma, base.v)
    assert lr <= 3e-3, lr
    print("fp32/TF32 sigma err (lead 64)", es[:64].max(), "all", es.max(), "low-rank", lr)


def test_sor_svd_fp32_storage_fp64_passes(env):
    """FP32-stored A with the default fp32_mode="fp64": the passes widen A to
    FP64 inside the DMMA GEMM, so the result matches the FP64 oracle on the
    same rounded matrix to FP64 parity (north-star tolerances, 10x floor)."""
    P, torch = env
    from oracle import sorsvd_oracle as O
    A = O.gen_lowrank_decay(20000, 2000, 256, lambda j: 10.0 ** (-j / 64.0), 1e-3, 3).astype(np.float32)
    Ad = A.astype(np.float64)
    cfg = O.SketchConfig(128, 1, 31)
    base, ds, dl = O.perturbation_floor(Ad, 128, cfg, trials=1)
    f = P.sor_svd_power(torch.from_numpy(A).cuda(), 128, P.SketchConfig(128, 1, 31))
    s = f.sigma.cpu().numpy()
    es = O.sigma_rel_err(s, base.sigma)
    assert np.all(es <= np.maximum(1e-10, 10 * np.maximum.accumulate(ds))), es.max()
    lr = O.lowrank_rel_diff(f.u.cpu().numpy(), s, f.v.cpu().numpy(), base.u, base.sigma, base.v)
    assert lr <= max(1e-9, 10 * dl), lr


def test_fp32_mode_rejects_unknown(env):
    P, torch = env
    a = torch.zeros((64, 48), device="cuda", dtype=torch.float32)
    with pytest.raises(P.ParameterError):
        P.sor_svd_power(a, 4, P.SketchConfig(8, 0, 1), fp32_mode="fp16")
