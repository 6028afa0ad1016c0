"""Generate the committed golden vectors from the COMPILED REFERENCE
(oracle/_ref/libsorsvd_ref.so = the unmodified /root/reference headers).

Run in the build container (needs /root/reference at build time only):
    python tests/golden/make_golden.py
The .npz written here is what tests/test_oracle.py pins the numpy/C
restatement against, and what the GPU parity tests use as fixed expectations.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import sorsvd_oracle as O  # noqa: E402

Ref = O.Ref
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    Ref.set_threads(1)
    g = {}
    meta = {}
    # random.hpp: gaussian_matrix / sub_seed (external contract, bit-exact)
    g["gauss_7x5_s123"] = Ref.gaussian_matrix(7, 5, 123)
    g["gauss_3x3_s0"] = Ref.gaussian_matrix(3, 3, 0)
    g["gauss_1x9_smax"] = Ref.gaussian_matrix(1, 9, 2**64 - 1)
    g["sub_seeds"] = np.array([Ref.sub_seed(s, t) for s in (0, 1, 42, 2**63) for t in (0, 1, 2, 3)], dtype=np.uint64)
    # sketch.hpp:178 flop_estimate (SPEC.md:224 KAT + all variants)
    fl = []
    for args in [(1000, 1000, 38, 20, 0), (4000, 4000, 100, 100, 1), (200000, 20000, 256, 256, 1), (25344, 300, 10, 10, 1)]:
        fl.append([Ref.flop_estimate(*args, v) for v in range(4)])
    g["flops"] = np.array(fl, dtype=np.int64)
    # dense.hpp KATs
    g["matmul_kat"] = Ref.matmul(np.array([[1.0, 2], [3, 4]]), np.array([[5.0], [6]]))
    q, r = Ref.thin_qr(np.array([[3.0], [4.0]]))
    g["qr34_q"], g["qr34_r"] = q, r
    u, s, v = Ref.full_svd(np.diag([3.0, 2.0, 1.0]))
    g["svd321_u"], g["svd321_s"], g["svd321_v"] = u, s, v
    a = O.gaussian_matrix(50, 10, 777)
    q, r = Ref.thin_qr(a)
    g["qr50x10_a"], g["qr50x10_q"], g["qr50x10_r"] = a, q, r
    mm = O.gaussian_matrix(20, 20, 4242)
    u, s, v = Ref.full_svd(mm)
    g["svd20_m"], g["svd20_u"], g["svd20_s"], g["svd20_v"] = mm, u, s, v
    # sor_svd_power on small seeded instances (sketch.hpp:87)
    cases = []
    for (m, n, k, ell, q, seed, aseed) in [(60, 40, 5, 8, 0, 11, 1), (60, 40, 5, 8, 1, 12, 2), (40, 70, 6, 6, 2, 13, 3),
                                            (100, 80, 1, 4, 0, 14, 4), (129, 65, 16, 24, 1, 15, 5)]:
        name = f"sor_{m}x{n}_k{k}_l{ell}_q{q}"
        x = O.gaussian_matrix(m, 6, O.sub_seed(aseed, 1))
        y = O.gaussian_matrix(n, 6, O.sub_seed(aseed, 2))
        e = O.gaussian_matrix(m, n, O.sub_seed(aseed, 3))
        A = x @ y.T + 1e-3 * e
        f = Ref.sor_svd_power(A, k, O.SketchConfig(ell, q, seed))
        g[name + "_A"] = A
        g[name + "_u"], g[name + "_s"], g[name + "_v"] = f.u, f.sigma, f.v
        meta[name] = dict(m=m, n=n, k=k, ell=ell, q=q, seed=seed, passes=f.passes, method=f.method)
        cases.append(name)
    # single_pass = true (sketch.hpp:54-58,100-104): M_approx core, 2q+2 passes
    sp_cases = []
    for (m, n, k, ell, q, seed, aseed) in [(60, 40, 5, 8, 0, 21, 6), (80, 50, 6, 10, 1, 22, 7), (50, 90, 4, 6, 2, 23, 8)]:
        name = f"sp_{m}x{n}_k{k}_l{ell}_q{q}"
        x = O.gaussian_matrix(m, 6, O.sub_seed(aseed, 1))
        y = O.gaussian_matrix(n, 6, O.sub_seed(aseed, 2))
        e = O.gaussian_matrix(m, n, O.sub_seed(aseed, 3))
        A = x @ y.T + 1e-3 * e
        f = Ref.sor_svd_power(A, k, O.SketchConfig(ell, q, seed, single_pass=True))
        g[name + "_A"] = A
        g[name + "_u"], g[name + "_s"], g[name + "_v"] = f.u, f.sigma, f.v
        meta[name] = dict(m=m, n=n, k=k, ell=ell, q=q, seed=seed, passes=f.passes, method=f.method, single_pass=True)
        sp_cases.append(name)
    # baselines r_svd (sketch.hpp:124) and tsr_svd (sketch.hpp:139): all ell triplets
    bl_cases = []
    for (kind, m, n, ell, q, seed, aseed) in [("rsvd", 60, 40, 8, 0, 31, 9), ("rsvd", 70, 50, 10, 1, 32, 10),
                                               ("rsvd", 40, 90, 6, 2, 33, 11), ("tsr", 60, 40, 8, 0, 34, 12),
                                               ("tsr", 50, 80, 10, 0, 35, 13), ("tsr", 129, 65, 16, 0, 36, 14)]:
        name = f"{kind}_{m}x{n}_l{ell}_q{q}"
        x = O.gaussian_matrix(m, 6, O.sub_seed(aseed, 1))
        y = O.gaussian_matrix(n, 6, O.sub_seed(aseed, 2))
        e = O.gaussian_matrix(m, n, O.sub_seed(aseed, 3))
        A = x @ y.T + 1e-3 * e
        f = Ref.r_svd(A, ell, q, seed) if kind == "rsvd" else Ref.tsr_svd(A, ell, seed)
        g[name + "_A"] = A
        g[name + "_u"], g[name + "_s"], g[name + "_v"] = f.u, f.sigma, f.v
        meta[name] = dict(kind=kind, m=m, n=n, ell=ell, q=q, seed=seed, passes=f.passes, method=f.method)
        bl_cases.append(name)
    # rank-1: 100 x 80, k = 1, ell = 4
    uu = O.gaussian_matrix(100, 1, 91)
    vv = O.gaussian_matrix(80, 1, 92)
    g["rank1_A"] = uu @ vv.T
    f = Ref.sor_svd_power(g["rank1_A"], 1, O.SketchConfig(4, 0, 93))
    g["rank1_u"], g["rank1_s"], g["rank1_v"] = f.u, f.sigma, f.v
    # Config 1 at full size (BASELINE.json configs[0])
    A1 = O.gen_c1(1)
    f = Ref.sor_svd_power(A1, 20, O.SketchConfig(20, 0, 7))
    g["c1_s"], g["c1_u"], g["c1_v"] = f.sigma, f.u, f.v
    g["c1_A_checksum"] = np.array([A1.sum(), (A1 * A1).sum(), A1[123, 456]])
    meta["c1"] = dict(seed=7, gen_seed=1, k=20, ell=20, q=0)
    # RPCA restatement around the reference sor_svd_power
    X, L0, S0 = Ref.gen_rpca_instance(100, 5, 500, 31)
    cfg = O.RpcaConfig(lam=1 / np.sqrt(100), mu0=0.0, mu_bar_factor=1e7, rho=1.6, tol=1e-7, max_iter=100, ell=10, q=1, seed=5)
    rr = Ref.rpca_alm(X, cfg)
    g["rpca100_X"] = X
    g["rpca100_L"], g["rpca100_S"] = rr.l, rr.s
    meta["rpca100"] = dict(iterations=rr.iterations, rank=rr.rank_l, nnz=rr.nnz_s, rel=rr.rel_error,
                           converged=rr.converged, mu0=rr.mu0, ell=10, q=1, seed=5, lam=float(cfg.lam))
    np.savez_compressed(os.path.join(OUT, "golden_ref.npz"), **g)
    with open(os.path.join(OUT, "golden_meta.json"), "w") as fh:
        json.dump({"cases": cases, "sp_cases": sp_cases, "bl_cases": bl_cases, "meta": meta, "blas": Ref and O.ref_lib().ref_blas_config().decode()}, fh, indent=1)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
