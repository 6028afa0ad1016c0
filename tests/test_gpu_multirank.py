"""GPU (single device): the row-sharded multi-GPU schedule, emulated in one
process — G contexts in one EmuGroup, one host thread each, every rank
holding a contiguous row block of A. Checks the sharded
result (U row blocks, replicated sigma and V) against the oracle on the full
matrix, and that every rank returns the same sigma and V."""
import threading

import numpy as np
import pytest

from oracle import sorsvd_oracle as O

pytestmark = pytest.mark.gpu


def _run_sharded(P, torch, A, k, cfg, world, dtype=None, fp64_mode="auto"):
    m = A.shape[0]
    g = P.EmuGroup(world)
    base, extra = divmod(m, world)
    bounds = []
    r0 = 0
    for r in range(world):
        cnt = base + (1 if r < extra else 0)
        bounds.append((r0, r0 + cnt))
        r0 += cnt
    ctxs = [P.Context(0, rank=r, emu_group=g) for r in range(world)]
    out = [None] * world
    err = [None] * world

    def work(r):
        try:
            a, b = bounds[r]
            blk = torch.from_numpy(np.ascontiguousarray(A[a:b])).cuda()
            if dtype is not None:
                blk = blk.to(dtype)
            out[r] = P.sor_svd_power(blk, k, cfg, ctx=ctxs[r], m_global=m, fp64_mode=fp64_mode)
            torch.cuda.synchronize()
        except Exception as e:  # surface in the main thread
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    for c in ctxs:
        c.close()
    g.close()
    u = np.vstack([o.u.cpu().numpy() for o in out])
    return out, u


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_00462_b200 as P
    return P, torch


@pytest.mark.parametrize("world,m,n,k,q", [(2, 3000, 800, 20, 1), (4, 6000, 500, 32, 0), (3, 2999, 700, 16, 2),
                                           (8, 8000, 400, 10, 1)])
def test_sharded_matches_oracle(env, world, m, n, k, q):
    P, torch = env
    A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + world)
    cfg = O.SketchConfig(k, q, 11)
    base, ds, dl = O.perturbation_floor(A, k, cfg)
    out, u = _run_sharded(P, torch, A, k, P.SketchConfig(k, q, 11), world)
    s0 = out[0].sigma.cpu().numpy()
    v0 = out[0].v.cpu().numpy()
    for o in out[1:]:  # replicated parts agree across ranks
        np.testing.assert_array_equal(o.sigma.cpu().numpy(), s0)
        np.testing.assert_array_equal(o.v.cpu().numpy(), v0)
    es = O.sigma_rel_err(s0, base.sigma)
    assert np.all(es <= np.maximum(1e-10, 10 * np.maximum.accumulate(ds))), es
    lr = O.lowrank_rel_diff(u, s0, v0, base.u, base.sigma, base.v)
    assert lr <= max(1e-9, 10 * dl), lr


@pytest.mark.parametrize("world,m,n,k,q", [(2, 3000, 800, 20, 1), (4, 6000, 1100, 64, 1), (3, 2999, 700, 16, 2)])
def test_sharded_ozaki_matches_oracle(env, world, m, n, k, q):
    # the int8 tensor-core passes over row blocks: per-rank scales, the T2 partials summed in
    # FP64 across ranks in column blocks on the comm stream (tn_pass_reduced)
    P, torch = env
    A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + world + 1)
    cfg = O.SketchConfig(k, q, 13)
    base, ds, dl = O.perturbation_floor(A, k, cfg)
    out, u = _run_sharded(P, torch, A, k, P.SketchConfig(k, q, 13), world, fp64_mode="ozaki")
    assert all(o.stats["pass_kind"] == 1 for o in out)
    s0 = out[0].sigma.cpu().numpy()
    for o in out[1:]:
        np.testing.assert_array_equal(o.sigma.cpu().numpy(), s0)
    es = O.sigma_rel_err(s0, base.sigma)
    assert np.all(es <= np.maximum(1e-10, 10 * np.maximum.accumulate(ds))), es
    lr = O.lowrank_rel_diff(u, s0, out[0].v.cpu().numpy(), base.u, base.sigma, base.v)
    assert lr <= max(1e-9, 10 * dl), lr


def test_sharded_c2_shape_householder_tree(env):
    """Ill-conditioned sketch (C2-like, q = 1): CholeskyQR2 is rejected, the
    cross-rank Householder TSQR tree (all-gather of R factors) runs."""
    P, torch = env
    A = O.gen_c2(2, n=1000)
    cfg = O.SketchConfig(40, 1, 5)
    base, ds, dl = O.perturbation_floor(A, 40, cfg)
    out, u = _run_sharded(P, torch, A, 40, P.SketchConfig(40, 1, 5), 4)
    s0 = out[0].sigma.cpu().numpy()
    env_ = np.maximum.accumulate(ds)
    jd = int(np.searchsorted(env_, 1e-10))
    es = O.sigma_rel_err(s0, base.sigma)
    assert jd >= 10 and np.all(es[:jd] <= np.maximum(1e-10, 10 * env_[:jd])), es[:jd]


def test_sharded_fp32(env):
    P, torch = env
    A = O.gen_lowrank_decay(8000, 1024, 64, lambda j: 10.0 ** (-j / 32.0), 1e-3, 9).astype(np.float32)
    cfg = O.SketchConfig(64, 1, 3)
    base = O.sor_svd_power(A.astype(np.float64), 64, cfg)
    out, u = _run_sharded(P, torch, A, 64, P.SketchConfig(64, 1, 3), 2, dtype=torch.float32)
    s0 = out[0].sigma.cpu().numpy()
    assert O.sigma_rel_err(s0, base.sigma)[:32].max() <= 3e-3


def _rpca_sharded(P, torch, D, cfg, world):
    m = D.shape[0]
    g = P.EmuGroup(world)
    base, extra = divmod(m, world)
    bounds, r0 = [], 0
    for r in range(world):
        cnt = base + (1 if r < extra else 0)
        bounds.append((r0, r0 + cnt))
        r0 += cnt
    ctxs = [P.Context(0, rank=r, emu_group=g) for r in range(world)]
    out, err = [None] * world, [None] * world

    def work(r):
        try:
            a, b = bounds[r]
            blk = torch.from_numpy(np.ascontiguousarray(D[a:b])).cuda()
            out[r] = P.rpca_alm(blk, cfg, ctx=ctxs[r], m_global=m)
            torch.cuda.synchronize()
        except Exception as e:
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    for c in ctxs:
        c.close()
    g.close()
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_rpca_sharded_matches_single(env, world):
    # Config 4 row-sharded: elementwise work local, the residual,
    # ||D||_F, the sigma_1 Gram and ||S||_0 summed over ranks
    P, torch = env
    D, L0, S0 = O.gen_c4(4, m=3000, n=150)
    cfg = P.RpcaConfig(lam=1 / np.sqrt(3000), mu0=0.0, ell=10, q=1, seed=9, max_iter=100)
    one = P.rpca_alm(torch.from_numpy(D).cuda(), cfg)
    out = _rpca_sharded(P, torch, D, cfg, world)
    for o in out:
        assert o.iterations == one.iterations and o.rank_l == one.rank_l and o.nnz_s == one.nnz_s
        assert abs(o.mu0 - one.mu0) <= 1e-12 * one.mu0
    l = np.vstack([o.l.cpu().numpy() for o in out])
    s = np.vstack([o.s.cpu().numpy() for o in out])
    l1, s1 = one.l.cpu().numpy(), one.s.cpu().numpy()
    assert np.linalg.norm(l - l1) <= 1e-9 * np.linalg.norm(l1)
    assert np.linalg.norm(s - s1) <= 1e-9 * np.linalg.norm(s1)


def test_sharded_k300_gram_qr(env):
    # k > 256 across ranks: the CholeskyQR Gram matrices are all-reduced
    P, torch = env
    A = O.gen_lowrank_decay(3000, 1200, 300, lambda j: 1.0 / j, 1e-6, 12)
    cfg = O.SketchConfig(300, 1, 5)
    base, ds, _ = O.perturbation_floor(A, 300, cfg, trials=1, qr_variants=2)
    out, u = _run_sharded(P, torch, A, 300, P.SketchConfig(300, 1, 5), 2)
    s = out[0].sigma.cpu().numpy()
    es = O.sigma_rel_err(s, base.sigma)
    assert np.all(es <= np.maximum(1e-10, 10 * np.maximum.accumulate(ds))), es.max()
    assert np.array_equal(s, out[1].sigma.cpu().numpy())


def test_sharded_replicated_outputs_deterministic(env):
    # sigma and V are replicated: bit-identical on every rank and on every repeat, with the
    # ranks' contexts created fresh each time (first-call allocations included) and all
    # eight ranks' streams running concurrently on the one device
    P, torch = env
    A = O.gen_lowrank_decay(8000, 400, 40, lambda j: 2.0 ** (-j / 4), 1e-3, 8008)
    ref = None
    for _ in range(6):
        out, _ = _run_sharded(P, torch, A, 10, P.SketchConfig(10, 1, 11), 8)
        for o in out:
            s, v = o.sigma.cpu().numpy(), o.v.cpu().numpy()
            if ref is None:
                ref = (s, v)
            np.testing.assert_array_equal(s, ref[0])
            np.testing.assert_array_equal(v, ref[1])


def test_concurrent_contexts_thin_qr_deterministic(env):
    # one context per host thread (the C ABI's threading contract): same input, same bits
    P, torch = env
    ctxs = [P.Context(0) for _ in range(8)]
    u, _ = np.linalg.qr(O.gaussian_matrix(1000, 10, 5))
    T = torch.from_numpy(u * np.logspace(0, -3, 10)).cuda()
    for _ in range(5):
        out = [None] * 8

        def work(r):
            out[r] = P.thin_qr(T.clone(), ctx=ctxs[r])[0]
            torch.cuda.synchronize()

        th = [threading.Thread(target=work, args=(r,)) for r in range(8)]
        [t.start() for t in th]
        [t.join() for t in th]
        for o in out[1:]:
            assert torch.equal(o, out[0])
    for c in ctxs:
        c.close()


def test_sharded_approx_error_matches_single(env):
    # approx_error over row-sharded A (each rank its row block of A and U): the sum of
    # squares is reduced over ranks and equals the single-rank value
    P, torch = env
    A = O.gen_lowrank_decay(3000, 500, 30, lambda j: 2.0 ** (-j / 4), 1e-3, 77)
    out, u = _run_sharded(P, torch, A, 16, P.SketchConfig(20, 1, 5), 3)
    s, v = out[0].sigma.cpu().numpy(), out[0].v.cpu().numpy()
    x = O.LowRankApprox(u, s, v, 0, 0, 16, 1, 5)
    ref = O.approx_error(A, x)
    g = P.EmuGroup(3)
    ctxs = [P.Context(0, rank=r, emu_group=g) for r in range(3)]
    blocks = np.array_split(np.arange(3000), 3)
    res = [None] * 3

    def work(r):
        a, b = blocks[r][0], blocks[r][-1] + 1
        xr = O.LowRankApprox(u[a:b], s, v, 0, 0, 16, 1, 5)
        res[r] = P.approx_error(torch.from_numpy(np.ascontiguousarray(A[a:b])).cuda(), xr, ctx=ctxs[r])

    th = [threading.Thread(target=work, args=(r,)) for r in range(3)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    for c in ctxs:
        c.close()
    g.close()
    assert res[0] == res[1] == res[2]
    assert abs(res[0] - ref) <= 1e-10 * ref


def _sharded_call(P, torch, A, world, fn):
    """fn(block, ctx, m_global) on every rank's contiguous row block of A, one host thread per rank."""
    m = A.shape[0]
    g = P.EmuGroup(world)
    base, extra = divmod(m, world)
    bounds, r0 = [], 0
    for r in range(world):
        cnt = base + (1 if r < extra else 0)
        bounds.append((r0, r0 + cnt))
        r0 += cnt
    ctxs = [P.Context(0, rank=r, emu_group=g) for r in range(world)]
    out, err = [None] * world, [None] * world

    def work(r):
        try:
            a, b = bounds[r]
            out[r] = fn(torch.from_numpy(np.ascontiguousarray(A[a:b])).cuda(), ctxs[r], m)
            torch.cuda.synchronize()
        except Exception as e:
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    for c in ctxs:
        c.close()
    g.close()
    return out


@pytest.mark.parametrize("world,m,n,ell,q", [(2, 3000, 500, 24, 1), (3, 2999, 700, 16, 0), (4, 4000, 300, 12, 2)])
def test_sharded_r_svd_matches_single_rank(env, world, m, n, ell, q):
    """r_svd (sketch.hpp:124-136) over row blocks: the sharded TSQR of Y, every A^T product summed over ranks."""
    P, torch = env
    A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + 3 * world)
    ref = O.r_svd(A, ell, q, 19)
    out = _sharded_call(P, torch, A, world, lambda blk, ctx, mg: P.r_svd(blk, ell, q, 19, ctx=ctx, m_global=mg))
    s0, v0 = out[0].sigma.cpu().numpy(), out[0].v.cpu().numpy()
    for o in out[1:]:
        np.testing.assert_array_equal(o.sigma.cpu().numpy(), s0)
        np.testing.assert_array_equal(o.v.cpu().numpy(), v0)
    u = np.vstack([o.u.cpu().numpy() for o in out])
    kk = min(ell, 10)
    assert O.sigma_rel_err(s0[:kk], ref.sigma[:kk]).max() <= 1e-10
    assert O.lowrank_rel_diff(u[:, :kk], s0[:kk], v0[:, :kk], ref.u[:, :kk], ref.sigma[:kk], ref.v[:, :kk]) <= 1e-8
    assert out[0].passes == ref.passes


@pytest.mark.parametrize("world,m,n,ell", [(2, 3000, 500, 24), (3, 2999, 700, 16)])
def test_sharded_tsr_svd_matches_oracle(env, world, m, n, ell):
    """tsr_svd (sketch.hpp:139-149) over row blocks: each rank draws ITS rows of Psi2 = gaussian_matrix(m, ell,
    seed ^ 1) (counter-based stream), Y2 and Q1^T Y1 are summed over ranks."""
    P, torch = env
    A = O.gen_lowrank_decay(m, n, 12, lambda j: 2.0 ** (-j), 1e-9, m + 5 * world)
    ref = O.tsr_svd(A, ell, 23)
    out = _sharded_call(P, torch, A, world, lambda blk, ctx, mg: P.tsr_svd(blk, ell, 23, ctx=ctx, m_global=mg))
    s0 = out[0].sigma.cpu().numpy()
    for o in out[1:]:
        np.testing.assert_array_equal(o.sigma.cpu().numpy(), s0)
    assert O.sigma_rel_err(s0[:8], ref.sigma[:8]).max() <= 1e-8
    single = P.tsr_svd(torch.from_numpy(A).cuda(), ell, 23)
    assert O.sigma_rel_err(s0[:8], single.sigma.cpu().numpy()[:8]).max() <= 1e-9


@pytest.mark.parametrize("world,m,n,k,q,trials", [(2, 3000, 400, 12, 1, 3), (4, 4001, 300, 8, 0, 5)])
def test_sharded_batched_trials_match_oracle(env, world, m, n, k, q, trials):
    """The bound harness's trial loop (bounds.hpp:288) over row blocks: each trial equals the oracle's call."""
    P, torch = env
    A = O.gen_lowrank_decay(m, n, 30, lambda j: 2.0 ** (-j / 3), 1e-4, m + 7 * world)
    cfg = P.SketchConfig(k, q, 300)
    out = _sharded_call(P, torch, A, world,
                        lambda blk, ctx, mg: P.sor_svd_power_batch(blk, k, cfg, trials, ctx=ctx, m_global=mg))
    for t in range(trials):
        ref = O.sor_svd_power(A, k, O.SketchConfig(k, q, 300 + t))
        s0 = out[0][t].sigma.cpu().numpy()
        for o in out[1:]:
            np.testing.assert_array_equal(o[t].sigma.cpu().numpy(), s0)
        u = np.vstack([o[t].u.cpu().numpy() for o in out])
        assert O.sigma_rel_err(s0, ref.sigma).max() <= 1e-10
        assert O.lowrank_rel_diff(u, s0, out[0][t].v.cpu().numpy(), ref.u, ref.sigma, ref.v) <= 1e-9


@pytest.mark.parametrize("world,m,n,k,ell,q", [(2, 3000, 600, 12, 16, 1), (3, 2999, 500, 8, 12, 0)])
def test_sharded_single_pass_matches_oracle(env, world, m, n, k, ell, q):
    """single_pass (sketch.hpp:54-58) over row blocks: Q1^T T1 needs the sketch T1 after its sharded QR."""
    P, torch = env
    A = O.gen_lowrank_decay(m, n, 30, lambda j: 2.0 ** (-j / 3), 1e-4, m + 11 * world)
    ref = O.sor_svd_power(A, k, O.SketchConfig(ell, q, 41, single_pass=True))
    out = _sharded_call(P, torch, A, world, lambda blk, ctx, mg: P.sor_svd_power(
        blk, k, P.SketchConfig(ell, q, 41, single_pass=True), ctx=ctx, m_global=mg))
    s0 = out[0].sigma.cpu().numpy()
    assert O.sigma_rel_err(s0, ref.sigma).max() <= 1e-9
    assert out[0].passes == 2 * q + 2


@pytest.mark.parametrize("world,m,n", [(2, 2000, 300), (3, 1501, 640)])
def test_sharded_spectral_norm_and_error_match_lapack(env, world, m, n):
    """norm(a, spectral) and approx_error(a, x, spectral) (dense.hpp:173-176, sketch.hpp:168-172) over
    row blocks: the Gram matrix is summed over the ranks; every rank returns the same value, equal to
    LAPACK's sigma_1 of the full matrix / of the full difference."""
    P, torch = env
    A = O.gen_lowrank_decay(m, n, 25, lambda j: 2.0 ** (-j / 3), 1e-3, 1000 + m)
    k = 12
    x = O.sor_svd_power(A, k, O.SketchConfig(16, 1, 9))
    ref_n = np.linalg.norm(A, 2)
    ref_e = np.linalg.norm(A - (x.u * x.sigma) @ x.v.T, 2)
    base, extra = divmod(m, world)
    starts = np.cumsum([0] + [base + (1 if r < extra else 0) for r in range(world)])

    def fn(blk, ctx, mg):
        r = ctx.rank
        xr = O.LowRankApprox(x.u[starts[r]:starts[r + 1]], x.sigma, x.v, 0, 0, k, 1, 9)
        return P.norm(blk, "spectral", ctx=ctx), P.approx_error(blk, xr, "spectral", ctx=ctx)

    out = _sharded_call(P, torch, A, world, fn)
    assert all(o == out[0] for o in out)
    assert abs(out[0][0] - ref_n) <= 1e-11 * ref_n
    assert abs(out[0][1] - ref_e) <= 1e-9 * ref_e


@pytest.mark.parametrize("world,m,n,r", [(2, 1200, 96, 7), (4, 4000, 200, 30)])
def test_sharded_estimate_rank_bound_matches_oracle(env, world, m, n, r):
    """estimate_rank_bound of a row-sharded matrix: local thin QR, the ranks' R
    factors gathered and factored again; the bound equals the single-matrix value on every rank."""
    P, torch = env
    A = O.gen_lowrank_decay(m, n, r, lambda j: 1.0 / j, 1e-6, 31 + m)
    ref = O.estimate_rank_bound(A)
    out = _sharded_call(P, torch, A, world, lambda blk, ctx, mg: P.estimate_rank_bound(blk, ctx=ctx))
    assert out == [ref] * world
    # rpca_default_config from a row block: lambda and the ell cap use the global row count
    cfgs = _sharded_call(P, torch, A, world, lambda blk, ctx, mg: P.rpca_default_config(blk, ctx=ctx, m_global=mg))
    one = P.rpca_default_config(torch.from_numpy(A).cuda())
    assert all(c.ell == one.ell and c.lam == one.lam for c in cfgs)
    single = P.estimate_rank_bound(torch.from_numpy(A).cuda())
    assert single == ref


def test_sharded_spectral_norm_wide_n_unsupported(env):
    P, torch = env
    A = np.ones((64, 1100))
    with pytest.raises(P.UnsupportedError):
        _sharded_call(P, torch, A, 2, lambda blk, ctx, mg: P.norm(blk, "spectral", ctx=ctx))


def test_nccl_binding_selftest_one_rank(env):
    """The NCCL calls of the row-sharded contexts (libnccl resolved by dlopen inside the library: unique id,
    ncclCommInitRank, in-place ncclAllReduce(ncclDouble, ncclSum), ncclAllGather, ncclCommDestroy) run on the
    one GPU that is reachable here as a one-rank communicator and return their input unchanged; a 128-byte id
    comes back from nccl_unique_id."""
    P, torch = env
    assert P.Context.nccl_selftest(0, 1 << 16) == 0.0
    assert P.Context.nccl_selftest(0, 3) == 0.0
    assert len(P.Context.nccl_unique_id()) == 128
