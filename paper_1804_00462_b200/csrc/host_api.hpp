// Internal host-side helpers shared by the C-ABI implementation.
#pragma once
#include <cstdint>

namespace sorsvd_host {
uint64_t sub_seed(uint64_t seed, uint64_t stream);
void gaussian_fill(double* out, uint64_t count, uint64_t seed, int nthreads);
long long flop_estimate(long long m, long long n, long long ell, long long k, long long q, int variant);
// nullptr when valid, else the reference's parameter_error message.
const char* validate_sketch(int64_t m, int64_t n, int k, int ell, int q);
}  // namespace sorsvd_host
