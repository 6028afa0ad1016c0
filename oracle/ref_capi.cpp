// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// C-ABI shim over the UNMODIFIED reference headers, compiled in place from
// /root/reference/proj/include (see oracle/Makefile; output only into
// oracle/_ref/). Nothing here re-implements the reference's SOR-SVD: every
// sorsvd::* call below is the reference's own inline code linked against the
// in-image OpenBLAS 0.3.15 (BLAS/LAPACK is un-vendored upstream:
// /root/reference/proj/CMakeLists.txt:5, .gitignore:2).
//
// The one restatement is ref_rpca_alm: the reference ships no RPCA code, so
// the inexact-ALM loop of SPEC.md:386-398 / PAPER.md:3138-3148 is restated
// here around the reference's own sor_svd_power (sketch.hpp:87), with the
// ambiguity ledger frozen as in SURVEY.md Appendix B (S0=Y0=0, mu capped with
// min, k=ell, seed+it per iteration, mu0 passed in).
#include <sorsvd/bounds.hpp>
#include <sorsvd/dense.hpp>
#include <sorsvd/matrix.hpp>
#include <sorsvd/matrixgen.hpp>
#include <sorsvd/random.hpp>
#include <sorsvd/sketch.hpp>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

// 0 ok, 1 shape, 2 parameter, 3 numerical, 4 other
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const sorsvd::shape_error& e) {
        g_err = e.what();
        return 1;
    } catch (const sorsvd::parameter_error& e) {
        g_err = e.what();
        return 2;
    } catch (const sorsvd::numerical_error& e) {
        g_err = e.what();
        return 3;
    } catch (const sorsvd::bound_inapplicable_error& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

sorsvd::Matrix wrap(std::int64_t rows, std::int64_t cols, const double* p) {
    return sorsvd::Matrix((std::size_t)rows, (std::size_t)cols,
                          std::vector<double>(p, p + rows * cols));
}

void put(const sorsvd::Matrix& m, double* out) {
    std::memcpy(out, m.data().data(), m.size() * sizeof(double));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) { openblas_set_num_threads(n); }

const char* ref_blas_config() { return openblas_get_config(); }

// random.hpp:24
std::uint64_t ref_sub_seed(std::uint64_t seed, std::uint64_t stream) {
    return sorsvd::sub_seed(seed, stream);
}

// random.hpp:60
int ref_gaussian_matrix(std::int64_t rows, std::int64_t cols, std::uint64_t seed, double* out) {
    return guarded([&] { put(sorsvd::gaussian_matrix((std::size_t)rows, (std::size_t)cols, seed), out); });
}

// dense.hpp:20 (matmul), trans flags 0/1
int ref_matmul(std::int64_t ar, std::int64_t ac, const double* a, int ta, std::int64_t br,
               std::int64_t bc, const double* b, int tb, double* c) {
    return guarded([&] {
        auto m = sorsvd::matmul(wrap(ar, ac, a), wrap(br, bc, b),
                                ta ? sorsvd::Trans::transpose : sorsvd::Trans::none,
                                tb ? sorsvd::Trans::transpose : sorsvd::Trans::none);
        put(m, c);
    });
}

// dense.hpp:114 (thin_qr): q m x n, r n x n
int ref_thin_qr(std::int64_t m, std::int64_t n, const double* a, double* q, double* r) {
    return guarded([&] {
        auto f = sorsvd::thin_qr(wrap(m, n, a));
        put(f.q, q);
        put(f.r, r);
    });
}

// dense.hpp:65 (full_svd): u m x r, s r, v n x r, r = min(m,n)
int ref_full_svd(std::int64_t m, std::int64_t n, const double* a, double* u, double* s, double* v) {
    return guarded([&] {
        auto f = sorsvd::full_svd(wrap(m, n, a));
        put(f.u, u);
        std::memcpy(s, f.sigma.data(), f.sigma.size() * sizeof(double));
        put(f.v, v);
    });
}

// dense.hpp:161 (norm): kind 0 frobenius, 1 spectral, 2 nuclear, 3 l1
int ref_norm(std::int64_t m, std::int64_t n, const double* a, int kind, double* out) {
    return guarded([&] {
        *out = sorsvd::norm(wrap(m, n, a), static_cast<sorsvd::NormKind>(kind));
    });
}

// sketch.hpp:87 (sor_svd_power) / :116 (sor_svd when use_basic != 0)
int ref_sor_svd_power(std::int64_t m, std::int64_t n, const double* a, int k, int ell, int q,
                      std::uint64_t seed, int single_pass, int use_basic, double* u, double* sigma,
                      double* v, int* passes, int* method) {
    return guarded([&] {
        sorsvd::SketchConfig cfg;
        cfg.ell = ell;
        cfg.q = q;
        cfg.seed = seed;
        cfg.single_pass = single_pass != 0;
        sorsvd::Matrix am = wrap(m, n, a);
        auto r = use_basic ? sorsvd::sor_svd(am, k, cfg) : sorsvd::sor_svd_power(am, k, cfg);
        put(r.u, u);
        std::memcpy(sigma, r.sigma.data(), r.sigma.size() * sizeof(double));
        put(r.v, v);
        *passes = r.passes;
        *method = (int)r.method;
    });
}

// sketch.hpp:124 (r_svd) / :139 (tsr_svd): all ell triplets, U m x ell, V n x ell
int ref_r_svd(std::int64_t m, std::int64_t n, const double* a, int ell, int q, std::uint64_t seed, double* u,
              double* sigma, double* v, int* passes, int* method) {
    return guarded([&] {
        auto r = sorsvd::r_svd(wrap(m, n, a), ell, q, seed);
        put(r.u, u);
        std::memcpy(sigma, r.sigma.data(), r.sigma.size() * sizeof(double));
        put(r.v, v);
        *passes = r.passes;
        *method = (int)r.method;
    });
}

int ref_tsr_svd(std::int64_t m, std::int64_t n, const double* a, int ell, std::uint64_t seed, double* u,
                double* sigma, double* v, int* passes, int* method) {
    return guarded([&] {
        auto r = sorsvd::tsr_svd(wrap(m, n, a), ell, seed);
        put(r.u, u);
        std::memcpy(sigma, r.sigma.data(), r.sigma.size() * sizeof(double));
        put(r.v, v);
        *passes = r.passes;
        *method = (int)r.method;
    });
}

// sketch.hpp:168-172: approx_error(a, x, kind) on a given factorisation
int ref_approx_error(std::int64_t m, std::int64_t n, const double* a, int k, const double* u, const double* sigma,
                     const double* v, int kind, double* out) {
    return guarded([&] {
        sorsvd::LowRankApprox x{wrap(m, k, u), std::vector<double>(sigma, sigma + k), wrap(n, k, v),
                                sorsvd::SketchMethod::sor, 0, k, 0, 0};
        *out = sorsvd::approx_error(wrap(m, n, a), x, kind == 0 ? sorsvd::NormKind::frobenius
                                                                : sorsvd::NormKind::spectral);
    });
}

// sketch.hpp:178
long long ref_flop_estimate(long long m, long long n, long long ell, long long k, long long q,
                            int variant) {
    long long out = -1;
    guarded([&] {
        out = sorsvd::flop_estimate(m, n, ell, k, q, static_cast<sorsvd::FlopVariant>(variant));
    });
    return out;
}

// matrixgen.hpp:44
int ref_random_orthonormal(std::int64_t n, std::uint64_t seed, double* out) {
    return guarded([&] { put(sorsvd::random_orthonormal((std::size_t)n, seed), out); });
}

// matrixgen.hpp:99
int ref_gen_rpca_instance(std::int64_t n, std::int64_t r, long long s, std::uint64_t seed,
                          double* x, double* l, double* sp) {
    return guarded([&] {
        auto inst = sorsvd::gen_rpca_instance((std::size_t)n, (std::size_t)r, s, seed);
        put(inst.x, x);
        put(inst.l_true, l);
        put(inst.s_true, sp);
    });
}

// bounds.hpp:94-222: the formula evaluators on a given spectrum and split norms
// (det_*: Phi from the two norms; avg_*: NaN when p < 2).
int ref_bound_formulas(int nsig, const double* sigma, int k, int ell, int p, int q, double norm_omega2,
                       double norm_omega1_pinv, int full_row_rank, double* det_sv, double* det_fro2,
                       double* avg_sv, double* avg_fro2, double* best_p_fro2) {
    return guarded([&] {
        std::vector<double> sg(sigma, sigma + nsig);
        sorsvd::BoundParams bp{k, ell, p, q};
        sorsvd::OmegaSplit sp{sorsvd::Matrix(1, 1), sorsvd::Matrix(1, 1), norm_omega2, norm_omega1_pinv,
                              full_row_rank != 0};
        std::vector<double> d = sorsvd::det_sv_lower_bound(sg, bp, sp);
        std::memcpy(det_sv, d.data(), d.size() * sizeof(double));
        det_fro2[0] = sorsvd::det_lowrank_bound(sg, bp, sp, sorsvd::NormKind::frobenius);
        det_fro2[1] = sorsvd::det_lowrank_bound(sg, bp, sp, sorsvd::NormKind::spectral);
        if (p >= 2) {
            std::vector<double> a = sorsvd::avg_sv_lower_bound(sg, bp);
            std::memcpy(avg_sv, a.data(), a.size() * sizeof(double));
            avg_fro2[0] = sorsvd::avg_lowrank_bound(sg, bp, sorsvd::NormKind::frobenius);
            avg_fro2[1] = sorsvd::avg_lowrank_bound(sg, bp, sorsvd::NormKind::spectral);
        } else {
            for (int j = 0; j < k; ++j) avg_sv[j] = NAN;
            avg_fro2[0] = avg_fro2[1] = NAN;
        }
        if (k + 2 <= ell) {
            best_p_fro2[0] = sorsvd::avg_lowrank_bound_best_p(sg, k, ell, q, sorsvd::NormKind::frobenius);
            best_p_fro2[1] = sorsvd::avg_lowrank_bound_best_p(sg, k, ell, q, sorsvd::NormKind::spectral);
        } else {
            best_p_fro2[0] = best_p_fro2[1] = NAN;
        }
    });
}

// RESTATEMENT of bounds.hpp:50-71 from the reference's own matmul / singular_values / norm:
// out = {||Omega_2||_2, ||Omega_1^+||_2, full_row_rank}. The reference function itself cannot
// be called: its return statement (bounds.hpp:65-70) moves omega2 into the result and THEN
// evaluates norm(omega2, spectral) on the moved-from matrix (rows/cols kept, buffer empty), so
// dgesdd is handed a null buffer (a segfault with this OpenBLAS). The intended order -- the
// norm of Omega_2 before it is moved -- is what is restated here; for the same reason
// bound_tightness_experiment (bounds.hpp:265-379, which calls omega_split at :300) is restated
// in oracle/sorsvd_oracle.py around the reference's sor_svd_power, approx_error, gaussian_matrix
// and the evaluators above.
int ref_omega_split(std::int64_t n, const double* v, const double* omega, int k, int ell, int p, int q,
                    double* out3) {
    return guarded([&] {
        sorsvd::BoundParams bp{k, ell, p, q};
        bp.validate();
        const sorsvd::Matrix vm = wrap(n, n, v), om = wrap(n, ell, omega);
        const std::size_t lead = (std::size_t)(ell - p);
        if (lead > (std::size_t)n) throw sorsvd::parameter_error("omega_split: ell - p exceeds n");
        const sorsvd::Matrix o1 = sorsvd::matmul(vm.block(0, 0, (std::size_t)n, lead), om, sorsvd::Trans::transpose,
                                                 sorsvd::Trans::none);
        const sorsvd::Matrix o2 = sorsvd::matmul(vm.block(0, lead, (std::size_t)n, (std::size_t)n - lead), om,
                                                 sorsvd::Trans::transpose, sorsvd::Trans::none);
        const std::vector<double> s1 = sorsvd::singular_values(o1);
        const double smax = s1.empty() ? 0.0 : s1.front(), smin = s1.empty() ? 0.0 : s1.back();
        const bool frr = smin > (double)n * DBL_EPSILON * smax;
        out3[0] = sorsvd::norm(o2, sorsvd::NormKind::spectral);
        out3[1] = frr ? 1.0 / smin : INFINITY;
        out3[2] = frr ? 1.0 : 0.0;
    });
}

// matrixgen.hpp:84-91
int ref_gen_polydecay(std::int64_t n, std::uint64_t seed, double* out) {
    return guarded([&] { put(sorsvd::gen_polydecay((std::size_t)n, seed), out); });
}

// RESTATEMENT (the reference has no RPCA code): SPEC.md:386-398,
// PAPER.md:3138-3148. Calls the reference's own sor_svd_power each iteration.
// mu0 is an input (Appendix B item 5); pass mu0 <= 0 to use 1.25/||X||_2
// computed with the reference's norm(spectral) (dense.hpp:173).
int ref_rpca_alm(std::int64_t m, std::int64_t n, const double* x, double lambda, double mu0,
                 double mu_bar_factor, double rho, double tol, int max_iter, int ell, int q,
                 std::uint64_t seed, double* l_out, double* s_out, int* iterations,
                 double* rel_error, int* rank_l, long long* nnz_s, int* converged,
                 double* mu0_used) {
    return guarded([&] {
        sorsvd::Matrix X = wrap(m, n, x);
        const std::size_t cells = (std::size_t)(m * n);
        const double xnorm = sorsvd::norm(X, sorsvd::NormKind::frobenius);
        std::vector<double> L(cells, 0.0), S(cells, 0.0), Y(cells, 0.0);
        if (xnorm == 0.0) {  // X = 0 -> L = S = 0 after 1 iteration
            std::memset(l_out, 0, cells * sizeof(double));
            std::memset(s_out, 0, cells * sizeof(double));
            *iterations = 1;
            *rel_error = 0.0;
            *rank_l = 0;
            *nnz_s = 0;
            *converged = 1;
            *mu0_used = 0.0;
            return;
        }
        double mu = mu0 > 0.0 ? mu0 : 1.25 / sorsvd::norm(X, sorsvd::NormKind::spectral);
        *mu0_used = mu;
        const double mu_bar = mu_bar_factor * mu;
        const double* xd = X.data().data();
        int it = 0;
        double rel = 0.0;
        int rank = 0;
        bool conv = false;
        while (it < max_iter) {
            // W = X - S + Y/mu
            std::vector<double> w(cells);
            for (std::size_t i = 0; i < cells; ++i) w[i] = xd[i] - S[i] + Y[i] / mu;
            sorsvd::SketchConfig cfg;
            cfg.ell = ell;
            cfg.q = q;
            cfg.seed = seed + (std::uint64_t)it;
            auto f = sorsvd::sor_svd_power(sorsvd::Matrix((std::size_t)m, (std::size_t)n, std::move(w)),
                                           ell, cfg);
            // L = U S_{1/mu}(Z) V^T
            std::vector<double> z(f.sigma.size());
            for (std::size_t j = 0; j < z.size(); ++j) z[j] = std::max(f.sigma[j] - 1.0 / mu, 0.0);
            rank = 0;
            for (std::size_t j = 0; j < z.size(); ++j)
                if (z[j] > 1e-8 * z[0]) ++rank;
            const std::size_t kk = z.size();
            const double* U = f.u.data().data();
            const double* V = f.v.data().data();
            for (std::int64_t i = 0; i < m; ++i)
                for (std::int64_t j = 0; j < n; ++j) {
                    double acc = 0.0;
                    for (std::size_t r = 0; r < kk; ++r) acc += U[i * kk + r] * z[r] * V[j * kk + r];
                    L[(std::size_t)(i * n + j)] = acc;
                }
            // S = S_{lambda/mu}(X - L + Y/mu); Y = Y + mu (X - L - S)
            const double eps = lambda / mu;
            long double res2 = 0.0L;
            for (std::size_t i = 0; i < cells; ++i) {
                const double t = xd[i] - L[i] + Y[i] / mu;
                const double a = std::fabs(t) - eps;
                const double s = a > 0.0 ? (t > 0.0 ? a : -a) : 0.0;
                S[i] = s;
                const double r = xd[i] - L[i] - s;
                Y[i] = Y[i] + mu * r;
                res2 += (long double)r * r;
            }
            mu = std::min(rho * mu, mu_bar);
            ++it;
            rel = std::sqrt((double)res2) / xnorm;
            if (!std::isfinite(rel)) throw sorsvd::numerical_error("rpca: non-finite iterate");
            if (rel < tol) {
                conv = true;
                break;
            }
        }
        std::memcpy(l_out, L.data(), cells * sizeof(double));
        std::memcpy(s_out, S.data(), cells * sizeof(double));
        long long nnz = 0;
        for (std::size_t i = 0; i < cells; ++i) nnz += S[i] != 0.0;
        *iterations = it;
        *rel_error = rel;
        *rank_l = rank;
        *nnz_s = nnz;
        *converged = conv ? 1 : 0;
    });
}

}  // extern "C"
