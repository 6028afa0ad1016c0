// TEST: the drop-in C++ front end (include/sorsvd_b200.hpp) used exactly as a
// reference caller would, on the reference's own types, next to the
// reference's CPU sor_svd_power. Built by tests/cpp/Makefile against the
// unmodified reference headers (needs /root/reference at build time only).
#include <sorsvd/matrixgen.hpp>
#include <sorsvd/sketch.hpp>

#include "sorsvd_b200.hpp"

#include <cmath>
#include <cstdio>

using namespace sorsvd;

static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
    double m = 0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a[i] - b[i]) / std::fabs(b[i]));
    return m;
}

int main() {
    int fails = 0;
    // Config 1 shape (BASELINE.json configs[0]): A = X Y^T + 1e-2 E
    Matrix x = gaussian_matrix(1000, 20, sub_seed(1, 1));
    Matrix y = gaussian_matrix(1000, 20, sub_seed(1, 2));
    Matrix a = matmul(x, y, Trans::none, Trans::transpose) + 1e-2 * gaussian_matrix(1000, 1000, sub_seed(1, 3));
    SketchConfig cfg;
    cfg.ell = 20;
    cfg.q = 0;
    cfg.seed = 7;
    LowRankApprox ref = sor_svd_power(a, 20, cfg);
    LowRankApprox gpu = cuda::sor_svd_power(a, 20, cfg);
    const double es = max_rel(gpu.sigma, ref.sigma);
    const double ea = std::sqrt(std::pow(norm(a - reconstruct(gpu), NormKind::frobenius), 2)) /
                      norm(a, NormKind::frobenius);
    const double er = norm(a - reconstruct(ref), NormKind::frobenius) / norm(a, NormKind::frobenius);
    std::printf("C1 sigma max rel err %.3e, approx err gpu %.6e ref %.6e, passes %d/%d, method %s/%s\n", es, ea, er,
                gpu.passes, ref.passes, to_string(gpu.method), to_string(ref.method));
    fails += !(es <= 1e-10) + (gpu.passes != ref.passes) + (gpu.method != ref.method) +
             !(std::fabs(ea - er) <= 1e-9 * er + 1e-12);
    // power form on a polynomial-decay matrix (matrixgen.hpp:80)
    Matrix p = gen_polydecay(300, 5);
    cfg.ell = 12;
    cfg.q = 2;
    cfg.seed = 3;
    LowRankApprox r2 = sor_svd_power(p, 10, cfg), g2 = cuda::sor_svd_power(p, 10, cfg);
    std::printf("polydecay sigma max rel err %.3e\n", max_rel(g2.sigma, r2.sigma));
    fails += !(max_rel(g2.sigma, r2.sigma) <= 1e-8);
    // single-pass core (sketch.hpp:54-58): M_approx, 2q+2 passes
    cfg.ell = 12;
    cfg.q = 1;
    cfg.seed = 5;
    cfg.single_pass = true;
    LowRankApprox r3 = sor_svd_power(a, 10, cfg), g3 = cuda::sor_svd_power(a, 10, cfg);
    std::printf("single_pass sigma max rel err %.3e, passes %d/%d\n", max_rel(g3.sigma, r3.sigma), g3.passes,
                r3.passes);
    fails += !(max_rel(g3.sigma, r3.sigma) <= 1e-10) + (g3.passes != r3.passes);
    cfg.single_pass = false;
    // baselines (sketch.hpp:124, :139): all ell triplets
    LowRankApprox r4 = r_svd(a, 12, 1, 9), g4 = cuda::r_svd(a, 12, 1, 9);
    LowRankApprox r5 = tsr_svd(a, 12, 9), g5 = cuda::tsr_svd(a, 12, 9);
    std::printf("r_svd sigma max rel err %.3e (passes %d/%d), tsr_svd %.3e (passes %d/%d)\n",
                max_rel(std::vector<double>(g4.sigma.begin(), g4.sigma.begin() + 10),
                        std::vector<double>(r4.sigma.begin(), r4.sigma.begin() + 10)),
                g4.passes, r4.passes,
                max_rel(std::vector<double>(g5.sigma.begin(), g5.sigma.begin() + 10),
                        std::vector<double>(r5.sigma.begin(), r5.sigma.begin() + 10)),
                g5.passes, r5.passes);
    fails += (g4.passes != r4.passes) + (g5.passes != r5.passes) + (g4.method != r4.method) +
             (g5.method != r5.method) + (g4.u.cols() != 12) + (g5.v.cols() != 12);
    fails += !(max_rel(std::vector<double>(g4.sigma.begin(), g4.sigma.begin() + 10),
                       std::vector<double>(r4.sigma.begin(), r4.sigma.begin() + 10)) <= 1e-10);
    fails += !(max_rel(std::vector<double>(g5.sigma.begin(), g5.sigma.begin() + 10),
                       std::vector<double>(r5.sigma.begin(), r5.sigma.begin() + 10)) <= 1e-10);
    try {
        cuda::r_svd(p, 300, 0, 1);
        ++fails;
    } catch (const parameter_error& e) {
        std::printf("parameter_error: %s\n", e.what());
    }
    // error behaviour mirrors the reference exceptions
    try {
        cfg.ell = 400;
        cuda::sor_svd_power(p, 10, cfg);
        ++fails;
    } catch (const parameter_error& e) {
        std::printf("parameter_error: %s\n", e.what());
    }
    try {
        cfg.ell = 12;
        cfg.q = 1;
        cuda::sor_svd(p, 10, cfg);
        ++fails;
    } catch (const parameter_error& e) {
        std::printf("parameter_error: %s\n", e.what());
    }
    // RPCA drop-in on a matrixgen instance (matrixgen.hpp:99): n = 100, r = 5, s = 0.05 n^2
    {
        RpcaInstance inst = gen_rpca_instance(100, 5, 500, 77);
        cuda::RpcaConfig rc = cuda::rpca_default_config(inst.l_true);
        std::printf("rank bound of the rank-5 L0: %lld, default ell %d\n", cuda::estimate_rank_bound(inst.l_true), rc.ell);
        fails += (cuda::estimate_rank_bound(inst.l_true) > 5) + (rc.ell > 10) + (rc.ell < 2);
        rc.ell = 10;
        rc.seed = 3;
        cuda::RpcaResult rr = cuda::rpca_alm(inst.x, rc);
        const double el = norm(rr.l - inst.l_true, NormKind::frobenius) / norm(inst.l_true, NormKind::frobenius);
        std::printf("rpca: %d iterations, rank %d, nnz %lld, rel %.2e, |L-L0|/|L0| %.2e, telemetry rows %zu\n",
                    rr.iterations, rr.rank_l, rr.nnz_s, rr.rel_error, el, rr.telemetry.size());
        fails += !rr.converged + (rr.rank_l != 5) + (rr.nnz_s != 500) + !(el <= 1e-5) +
                 (rr.telemetry.size() != (std::size_t)rr.iterations) + !(rr.rel_error < 1e-7);
        if (!rr.telemetry.empty())
            fails += (rr.telemetry.back().rank_l != rr.rank_l) + (rr.telemetry.back().nnz_s != rr.nnz_s) +
                     (rr.telemetry.front().iter != 1);
        try {
            cuda::estimate_rank_bound(Matrix(4, 3));
            ++fails;
        } catch (const parameter_error& e) {
            std::printf("parameter_error: %s\n", e.what());
        }
    }
    std::printf(fails ? "FAIL (%d)\n" : "OK\n", fails);
    return fails ? 1 : 0;
}
