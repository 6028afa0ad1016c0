// Host mirror of the reference RNG contract (random.hpp:14-65) and of the
// scalar helpers of sketch.hpp (validate_sketch :62-69, flop_estimate
// :178-196). Compiled by the host compiler against glibc libm, so
// gaussian_matrix is bit-identical to the reference's std::log/sqrt/sin/cos.
//
// The splitmix64 stream is counter based (state after t words is
// seed + t*gamma), so the row-major fill parallelises exactly: element e uses
// words 2*floor(e/2)+1 and 2*floor(e/2)+2; even e takes r*cos(t), odd r*sin(t)
// (NormalStream::next, random.hpp:35-48).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <thread>
#include <unordered_set>
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

// Elements [e0, e1) of the stream of `seed` into out[0 .. e1 - e0): a row block of a larger
// gaussian_matrix (the generators' row-sharded factors).
void gaussian_fill_range(double* out, uint64_t e0, uint64_t e1, uint64_t seed, int nthreads) {
    if (e1 <= e0) return;
    if (nthreads <= 0) {
        nthreads = (int)std::thread::hardware_concurrency();
        if (nthreads <= 0) nthreads = 1;
    }
    const uint64_t count = e1 - e0, min_chunk = 1 << 15;
    uint64_t nt = (uint64_t)nthreads;
    if (count / min_chunk + 1 < nt) nt = count / min_chunk + 1;
    double* base = out - e0;  // fill_range indexes by the absolute element number
    if (nt <= 1) {
        fill_range(base, e0, e1, seed);
        return;
    }
    std::vector<std::thread> th;
    const uint64_t per = ((count / nt) + 2) & ~1ULL;
    for (uint64_t t = 0; t < nt; ++t) {
        // chunk edges on even absolute element numbers keep the Box-Muller pairs together
        uint64_t a = e0 + t * per, b = e0 + (t + 1) * per;
        if (t > 0) a &= ~1ULL;
        b &= ~1ULL;
        if (t + 1 == nt || b > e1) b = e1;
        if (a >= b) break;
        th.emplace_back(fill_range, base, a, b, seed);
        if (b == e1) break;
    }
    for (auto& x : th) x.join();
}

// The sparse component of gen_rpca_instance (matrixgen.hpp:106-121): s distinct cells of
// {0, ..., cells - 1} by Floyd's sampling from the stream of sub_seed(seed, 3), sorted, with values
// +-50 from the words of sub_seed(seed, 4). Integer arithmetic only: identical to the reference.
void rpca_support(long long cells, long long s, uint64_t seed, std::vector<long long>& pos, std::vector<double>& val) {
    pos.clear();
    val.clear();
    if (s <= 0) return;
    uint64_t st = sub_seed(seed, 3);
    std::unordered_set<long long> chosen;
    chosen.reserve((size_t)s * 2);
    for (long long j = cells - s; j < cells; ++j) {
        st += kGamma;
        const long long t = (long long)(mix(st) % (uint64_t)(j + 1));
        if (!chosen.insert(t).second) chosen.insert(j);
    }
    pos.assign(chosen.begin(), chosen.end());
    std::sort(pos.begin(), pos.end());
    uint64_t sg = sub_seed(seed, 4);
    val.resize(pos.size());
    for (size_t i = 0; i < pos.size(); ++i) {
        sg += kGamma;
        val[i] = (mix(sg) & 1ULL) ? 50.0 : -50.0;
    }
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
