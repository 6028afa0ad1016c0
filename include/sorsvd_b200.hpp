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

}  // namespace cuda
}  // namespace sorsvd
