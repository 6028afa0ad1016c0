// Host mirror of the reference RNG contract (random.hpp:14-65) and of the
// scalar helpers of sketch.hpp (validate_sketch :62-69, flop_estimate
// :178-196). Compiled by the host compiler against glibc libm, so
// gaussian_matrix is bit-identical to the reference's std::log/sqrt/sin/cos.
//
// The splitmix64 stream is counter based (state after t words is
// seed + t*gamma), so the row-major fill parallelises exactly: element e uses
// words 2*floor(e/2)+1 and 2*floor(e/2)+2; even e takes r*cos(t), odd r*sin(t)
// (NormalStream::next, random.hpp:35-48).
#include <cmath>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "host_api.hpp"

namespace sorsvd_host {

static constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

static inline uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t sub_seed(uint64_t seed, uint64_t stream) {
    const uint64_t s = seed + kGamma * (stream + 1);
    return mix(s + kGamma);
}

static void fill_range(double* out, uint64_t e0, uint64_t e1, uint64_t seed) {
    const double two_pi = 2.0 * 3.141592653589793238462643383279502884;
    uint64_t e = e0;
    while (e < e1) {
        const uint64_t p = e >> 1;
        const uint64_t w1 = mix(seed + (2 * p + 1) * kGamma);
        const uint64_t w2 = mix(seed + (2 * p + 2) * kGamma);
        const double u1 = (double)((w1 >> 11) + 1) * 0x1.0p-53;
        const double u2 = (double)(w2 >> 11) * 0x1.0p-53;
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double t = two_pi * u2;
        if ((e & 1) == 0) {
            out[e] = r * std::cos(t);
            if (e + 1 < e1) out[e + 1] = r * std::sin(t);
            e += 2;
        } else {
            out[e] = r * std::sin(t);
            e += 1;
        }
    }
}

void gaussian_fill(double* out, uint64_t count, uint64_t seed, int nthreads) {
    if (nthreads <= 0) {
        nthreads = (int)std::thread::hardware_concurrency();
        if (nthreads <= 0) nthreads = 1;
    }
    const uint64_t min_chunk = 1 << 15;
    uint64_t nt = (uint64_t)nthreads;
    if (count / min_chunk + 1 < nt) nt = count / min_chunk + 1;
    if (nt <= 1) {
        fill_range(out, 0, count, seed);
        return;
    }
    std::vector<std::thread> th;
    const uint64_t per = ((count / nt) + 1) & ~1ULL;  // even chunk starts keep pairs together
    for (uint64_t t = 0; t < nt; ++t) {
        // the last chunk runs to the end: nt * per can fall short of count (per is rounded
        // down to even), which left the last element pair of Omega unwritten
        const uint64_t a = t * per;
        const uint64_t b = (t + 1 == nt || (t + 1) * per > count) ? count : (t + 1) * per;
        if (a >= b) break;
        th.emplace_back(fill_range, out, a, b, seed);
    }
    for (auto& x : th) x.join();
}

long long flop_estimate(long long m, long long n, long long ell, long long k, long long q, int variant) {
    if (m <= 0 || n <= 0 || ell <= 0 || k <= 0 || q < 0) return -1;
    const long long cmult = 2 * m * n;
    switch (variant) {
        case 0: return 3 * ell * cmult + 2 * ell * (m + n) * (ell + k) + 2 * ell * ell * (m + ell);
        case 1: return 2 * ell * cmult + 2 * ell * (m + n) * (2 * ell + k) + 5 * ell * ell * ell;
        case 2: return (2 * q + 3) * ell * cmult + 2 * ell * (m + n) * (ell + k) + 2 * ell * ell * (m + ell);
        case 3: return (2 * q + 2) * ell * cmult + 2 * ell * (m + n) * (2 * ell + k) + 5 * ell * ell * ell;
    }
    return -1;
}

const char* validate_sketch(int64_t m, int64_t n, int k, int ell, int q) {
    const int64_t mn = m < n ? m : n;
    if (m < 2 || n < 2) return "parameter: sketch input must be at least 2x2";
    if (k < 1) return "parameter: target rank k must be positive";
    if (ell < k) return "parameter: sample size ell must satisfy ell >= k";
    if ((int64_t)ell >= mn) return "parameter: sample size ell must be < min(rows, cols)";
    if (q < 0) return "parameter: power iteration count q must be nonnegative";
    return nullptr;
}

}  // namespace sorsvd_host
