// Internal host-side helpers shared by the C-ABI implementation.
#pragma once
#include <cstdint>
#include <vector>

namespace sorsvd_host {
uint64_t sub_seed(uint64_t seed, uint64_t stream);
void gaussian_fill(double* out, uint64_t count, uint64_t seed, int nthreads);
void gaussian_fill_range(double* out, uint64_t e0, uint64_t e1, uint64_t seed, int nthreads);
void rpca_support(long long cells, long long s, uint64_t seed, std::vector<long long>& pos, std::vector<double>& val);
long long flop_estimate(long long m, long long n, long long ell, long long k, long long q, int variant);
// nullptr when valid, else the reference's parameter_error message.
const char* validate_sketch(int64_t m, int64_t n, int k, int ell, int q);
}  // namespace sorsvd_host
