// f4: test-matrix generators on the device (matrixgen.hpp; SURVEY.md 8(d) "generated on the GPU:
// counter splitmix + Box-Muller, only ulp-compatible with the host").
//
// The reference fills every Gaussian matrix from one sequential NormalStream (random.hpp:27-55):
// words 2p+1, 2p+2 of the splitmix64 stream give the normals 2p (r cos t) and 2p+1 (r sin t).
// The stream is counter based (state after w words = seed + w * gamma), so any element can be
// drawn on its own: these kernels evaluate the same words with the device's log / sqrt /
// sincos, which agree with glibc's to a few ulp (the integer part -- words, uniforms -- is
// bit-identical). Factors that must be bit-identical to the host (the n x r Gaussian factors
// of the low-rank families) are drawn by host_rng.cpp and uploaded; only the m x n noise term,
// which dominates the volume (C3: 4e9 normals, C5: 1.7e10), is drawn here.
#pragma once
#include "common.cuh"
#include "rpca_f64.cuh"  // dmma884, kRpcaThreads

namespace sorsvd_dev {

__device__ __forceinline__ uint64_t gen_mix(uint64_t z) {  // splitmix64 finaliser (random.hpp:17-20)
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
constexpr uint64_t kGenGamma = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ uint64_t gen_sub_seed(uint64_t seed, uint64_t stream) {  // random.hpp:24-27
    return gen_mix(seed + kGenGamma * (stream + 1) + kGenGamma);
}

// Normals 2p and 2p+1 of NormalStream(seed) (random.hpp:35-48).
__device__ __forceinline__ void gen_normal_pair(uint64_t seed, uint64_t p, double& z0, double& z1) {
    const uint64_t w1 = gen_mix(seed + (2 * p + 1) * kGenGamma);
    const uint64_t w2 = gen_mix(seed + (2 * p + 2) * kGenGamma);
    const double u1 = (double)((w1 >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(w2 >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincos(6.283185307179586476925286766559 * u2, &sn, &cs);
    z0 = r * cs;
    z1 = r * sn;
}

// gaussian_matrix(rows, cols, seed) (random.hpp:60-65) as a rows x cols row-major fill of `out`
// (pitch ld): element e = i * cols + j of the stream, times `scale`.
__global__ void gaussian_fill_kernel(double* __restrict__ out, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                                     double scale) {
    const int64_t pairs = (rows * cols + 1) / 2;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < pairs; p += (int64_t)gridDim.x * blockDim.x) {
        double z0, z1;
        gen_normal_pair(seed, (uint64_t)p, z0, z1);
        const int64_t e0 = 2 * p, e1 = 2 * p + 1;
        out[(e0 / cols) * ld + e0 % cols] = z0 * scale;
        if (e1 < rows * cols) out[(e1 / cols) * ld + e1 % cols] = z1 * scale;
    }
}

// A (rows [row0, row0 + m) of the global matrix) = X diag(s) Y^T + noise_std * E, E's row i drawn
// from NormalStream(sub_seed(noise_seed, i)) (one stream per global row: shardable by rows).
// The rank-r product is built on DMMA fragments per 64 x 64 tile like approx_err_kernel; a thread's
// two adjacent columns (even, odd) are one Box-Muller pair. AT = double or float storage.
template <typename AT>
__global__ void __launch_bounds__(kRpcaThreads) gen_lowrank_kernel(AT* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                                                  const double* __restrict__ X, int64_t ldx,
                                                                  const double* __restrict__ sig,
                                                                  const double* __restrict__ Y, int64_t ldy, int r,
                                                                  double noise_std, uint64_t noise_seed, int64_t row0) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t i0 = (int64_t)blockIdx.y * 64 + (warp >> 1) * 16;
    const int64_t j0 = (int64_t)blockIdx.x * 64 + (warp & 1) * 32;
    double acc[2][4][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    for (int kk0 = 0; kk0 < r; kk0 += 4) {
        const int kk = kk0 + t4;
        const double z = kk < r ? sig[kk] : 0.0;
        double af[2], bf[4];
#pragma unroll
        for (int fm = 0; fm < 2; ++fm) {
            const int64_t i = i0 + fm * 8 + g;
            af[fm] = (kk < r && i < m) ? X[i * ldx + kk] * z : 0.0;
        }
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
            const int64_t j = j0 + fn * 8 + g;
            bf[fn] = (kk < r && j < n) ? Y[j * ldy + kk] : 0.0;
        }
#pragma unroll
        for (int fm = 0; fm < 2; ++fm)
#pragma unroll
            for (int fn = 0; fn < 4; ++fn) dmma884(acc[fm][fn][0], acc[fm][fn][1], af[fm], bf[fn]);
    }
#pragma unroll
    for (int fm = 0; fm < 2; ++fm) {
        const int64_t i = i0 + fm * 8 + g;
        if (i >= m) continue;
        const uint64_t rs = gen_sub_seed(noise_seed, (uint64_t)(row0 + i));
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
            const int64_t j = j0 + fn * 8 + 2 * t4;
            if (j >= n) continue;
            double z0 = 0.0, z1 = 0.0;
            if (noise_std != 0.0) gen_normal_pair(rs, (uint64_t)(j >> 1), z0, z1);
            A[i * lda + j] = (AT)(acc[fm][fn][0] + noise_std * z0);
            if (j + 1 < n) A[i * lda + j + 1] = (AT)(acc[fm][fn][1] + noise_std * z1);
        }
    }
}

// A[pos[t]] += val[t] over a dense row-major n x n (pitch ld) matrix: the sparse component of
// gen_rpca_instance (matrixgen.hpp:116-120; positions are distinct).
__global__ void scatter_add_kernel(double* __restrict__ A, int64_t ld, int64_t cols, const long long* __restrict__ pos,
                                   const double* __restrict__ val, int64_t count) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        const long long p = pos[t];
        A[(p / cols) * ld + p % cols] += val[t];
    }
}

}  // namespace sorsvd_dev
