// sorsvd_b200.hpp — drop-in C++ front end for the reference API.
//
// Include AFTER the reference headers (<sorsvd/sketch.hpp>): this header
// defines sorsvd::cuda::sor_svd_power / sor_svd / r_svd / tsr_svd with exactly
// the reference signatures (sketch.hpp:87, :116, :124, :139) on the reference types (Matrix,
// SketchConfig, LowRankApprox), and rethrows the reference exception types
// (errors.hpp:9-26) from the C-ABI status codes. The arithmetic runs on the
// B200 through include/sorsvd_b200.h (libsorsvd_b200.so).
//
//   #include <sorsvd/sketch.hpp>
//   #include "sorsvd_b200.hpp"
//   auto f = sorsvd::cuda::sor_svd_power(a, k, cfg);   // was sorsvd::sor_svd_power
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sorsvd_b200.h"

namespace sorsvd {
namespace cuda {

namespace detail {

inline std::string strip_tag(std::string msg) {
    // the C ABI messages carry the reference's "shape: " / "parameter: " /
    // "numerical: " tags, which the reference exception constructors add again
    for (const char* tag : {"shape: ", "parameter: ", "numerical: "}) {
        const std::string t(tag);
        if (msg.compare(0, t.size(), t) == 0) return msg.substr(t.size());
    }
    return msg;
}

inline void throw_status(int rc, const sorsvd_ctx* ctx) {
    const std::string msg = strip_tag(sorsvd_last_error(ctx));
    switch (rc) {
        case SORSVD_OK: return;
        case SORSVD_ERR_SHAPE: throw shape_error(msg);
        case SORSVD_ERR_PARAMETER: throw parameter_error(msg);
        case SORSVD_ERR_NUMERICAL: throw numerical_error(msg);
        default: throw std::runtime_error("sorsvd_b200: " + msg);
    }
}

// One context per host thread (the reference functions are re-entrant,
// SPEC.md:127; a context owns a device stream, workspaces and CUDA graphs).
inline sorsvd_ctx* thread_context(int device = 0) {
    struct Holder {
        sorsvd_ctx* c = nullptr;
        ~Holder() {
            if (c) sorsvd_ctx_destroy(c);
        }
    };
    thread_local Holder h;
    if (!h.c) throw_status(sorsvd_ctx_create(device, &h.c), nullptr);
    return h.c;
}

}  // namespace detail

// sketch.hpp:87 — same arguments, same result type, same exceptions.
inline LowRankApprox sor_svd_power(const Matrix& a, int k, const SketchConfig& cfg) {
    sorsvd_ctx* ctx = detail::thread_context();
    sorsvd_desc d{};
    d.m = (int64_t)a.rows();
    d.n = (int64_t)a.cols();
    d.lda = (int64_t)a.cols();
    d.k = k;
    d.ell = cfg.ell;
    d.q = cfg.q;
    d.single_pass = cfg.single_pass ? 1 : 0;
    d.seed = cfg.seed;
    d.dtype = SORSVD_F64;
    if (k < 1 || cfg.ell < k) {  // validate before sizing outputs (sketch.hpp:62-69 messages)
        detail::throw_status(sorsvd_validate_sketch(d.m, d.n, k, cfg.ell, cfg.q), nullptr);
    }
    Matrix u(a.rows(), (std::size_t)k), v(a.cols(), (std::size_t)k);
    std::vector<double> sigma((std::size_t)k);
    sorsvd_stats st{};
    detail::throw_status(sorsvd_sor_svd_power(ctx, &d, a.data().data(), nullptr, u.data().data(), sigma.data(),
                                              v.data().data(), &st),
                         ctx);
    return LowRankApprox{std::move(u), std::move(sigma), std::move(v),
                         cfg.q == 0 ? SketchMethod::sor : SketchMethod::sor_power, st.passes, cfg.ell, cfg.q,
                         cfg.seed};
}

// sketch.hpp:116
inline LowRankApprox sor_svd(const Matrix& a, int k, const SketchConfig& cfg) {
    if (cfg.q != 0) throw parameter_error("sor_svd requires q == 0; use sor_svd_power");
    return ::sorsvd::cuda::sor_svd_power(a, k, cfg);
}

namespace detail {
inline sorsvd_desc baseline_desc(const Matrix& a, int ell, int q, std::uint64_t seed) {
    sorsvd_desc d{};
    d.m = (int64_t)a.rows();
    d.n = (int64_t)a.cols();
    d.lda = (int64_t)a.cols();
    d.k = ell;
    d.ell = ell;
    d.q = q;
    d.seed = seed;
    d.dtype = SORSVD_F64;
    // validate_sketch(a, ell, ell, q) before sizing outputs (sketch.hpp:127,141)
    throw_status(sorsvd_validate_sketch(d.m, d.n, ell, ell, q), nullptr);
    return d;
}
}  // namespace detail

// sketch.hpp:124 — one-sided randomized SVD baseline, all ell triplets, 2q+2 passes.
inline LowRankApprox r_svd(const Matrix& a, int ell, int q, std::uint64_t seed) {
    sorsvd_ctx* ctx = detail::thread_context();
    const sorsvd_desc d = detail::baseline_desc(a, ell, q, seed);
    Matrix u(a.rows(), (std::size_t)ell), v(a.cols(), (std::size_t)ell);
    std::vector<double> sigma((std::size_t)ell);
    sorsvd_stats st{};
    detail::throw_status(
        sorsvd_r_svd(ctx, &d, a.data().data(), nullptr, u.data().data(), sigma.data(), v.data().data(), &st), ctx);
    return LowRankApprox{std::move(u), std::move(sigma), std::move(v), SketchMethod::rsvd, st.passes, ell, q, seed};
}

// sketch.hpp:139 — two-sided randomized SVD baseline (Psi2 from seed ^ 1), 1 pass.
inline LowRankApprox tsr_svd(const Matrix& a, int ell, std::uint64_t seed) {
    sorsvd_ctx* ctx = detail::thread_context();
    const sorsvd_desc d = detail::baseline_desc(a, ell, 0, seed);
    Matrix u(a.rows(), (std::size_t)ell), v(a.cols(), (std::size_t)ell);
    std::vector<double> sigma((std::size_t)ell);
    sorsvd_stats st{};
    detail::throw_status(sorsvd_tsr_svd(ctx, &d, a.data().data(), nullptr, nullptr, u.data().data(), sigma.data(),
                                        v.data().data(), &st),
                         ctx);
    return LowRankApprox{std::move(u), std::move(sigma), std::move(v), SketchMethod::tsr, st.passes, ell, 0, seed};
}

// ---- RPCA (the reference ships the spec but no code for it) ----------------
// Types with the spec's field names and the three operations a caller of the
// spec's rpca module uses: estimate_rank_bound (:377), rpca_default_config (:398), rpca_alm (:386).
struct RpcaConfig {
    double lambda = 0.0;       // <= 0 -> 1/sqrt(max(m,n))
    double mu0 = 0.0;          // <= 0 -> 1.25/sigma_1(X), estimated on the device
    double mu_bar_factor = 1e7;
    double rho = 1.6;
    double tol = 1e-7;
    int max_iter = 500;
    int ell = 10;
    int q = 1;
    std::uint64_t seed = 0;
};

struct RpcaIteration {  // one row of the per-iteration telemetry CSV
    int iter;
    double mu, rel_error;
    int rank_l;
    long long nnz_s;
};

struct RpcaResult {
    Matrix l, s;
    int iterations = 0;
    double rel_error = 0.0;
    int rank_l = 0;
    long long nnz_s = 0;
    bool converged = false;
    std::vector<RpcaIteration> telemetry;
};

// inexact ALM with sor_svd_power (k = ell, seed + it) per iteration.
inline RpcaResult rpca_alm(const Matrix& x, const RpcaConfig& cfg) {
    sorsvd_ctx* ctx = detail::thread_context();
    sorsvd_rpca_desc d{};
    d.m = (int64_t)x.rows();
    d.n = (int64_t)x.cols();
    d.ldd = (int64_t)x.cols();
    d.lambda = cfg.lambda;
    d.mu0 = cfg.mu0;
    d.mu_bar_factor = cfg.mu_bar_factor;
    d.rho = cfg.rho;
    d.tol = cfg.tol;
    d.max_iter = cfg.max_iter;
    d.ell = cfg.ell;
    d.q = cfg.q;
    d.dtype = SORSVD_F64;
    d.seed = cfg.seed;
    RpcaResult out{Matrix(x.rows(), x.cols()), Matrix(x.rows(), x.cols())};
    sorsvd_rpca_result r{};
    detail::throw_status(sorsvd_rpca_alm(ctx, &d, x.data().data(), out.l.data().data(), out.s.data().data(), &r), ctx);
    out.iterations = r.iterations;
    out.rel_error = r.rel_error;
    out.rank_l = r.rank_l;
    out.nnz_s = r.nnz_s;
    out.converged = r.converged != 0;
    int32_t rows = 0;
    detail::throw_status(sorsvd_rpca_telemetry(ctx, 0, nullptr, &rows), ctx);
    std::vector<double> t((std::size_t)rows * 5);
    if (rows) detail::throw_status(sorsvd_rpca_telemetry(ctx, rows, t.data(), &rows), ctx);
    for (int i = 0; i < rows; ++i)
        out.telemetry.push_back(RpcaIteration{(int)t[5 * i], t[5 * i + 1], t[5 * i + 2], (int)t[5 * i + 3],
                                              (long long)t[5 * i + 4]});
    return out;
}

// ceil((||X||_* / ||X||_F)^2); min(m, n) <= 512 on the device.
inline long long estimate_rank_bound(const Matrix& x) {
    sorsvd_ctx* ctx = detail::thread_context();
    int64_t b = 0;
    detail::throw_status(sorsvd_estimate_rank_bound(ctx, (int64_t)x.rows(), (int64_t)x.cols(), x.data().data(),
                                                    (int64_t)x.cols(), &b, nullptr, nullptr),
                         ctx);
    return (long long)b;
}

// SPEC.md:398.
inline RpcaConfig rpca_default_config(const Matrix& x) {
    RpcaConfig c;
    const std::size_t mn = x.rows() < x.cols() ? x.rows() : x.cols();
    const long long two_r = 2 * estimate_rank_bound(x);
    c.ell = (int)(two_r < (long long)mn - 1 ? two_r : (long long)mn - 1);
    if (c.ell < 1) c.ell = 1;
    c.q = 1;
    return c;
}

}  // namespace cuda
}  // namespace sorsvd
