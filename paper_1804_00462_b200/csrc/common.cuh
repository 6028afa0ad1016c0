// Shared device helpers for the SOR-SVD sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sorsvd_dev {

constexpr int kWarp = 32;

// Launch predication. A kernel given (pred, skip) is a no-op when *pred == skip
// (CholeskyQR2 accepted / rejected, RPCA converged) or when *pred == kPredDead:
// a QR whose enclosing RPCA iteration is predicated off marks its inner flag
// dead, so both of its paths skip (predicates stack instead of replacing).
constexpr int kPredDead = 2;
__device__ __forceinline__ bool pred_off(const int* p, int skip) {
    if (!p) return false;
    const int v = *p;
    return v == skip || v == kPredDead;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum over aligned groups of `G` lanes (G power of two <= 32).
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Asynchronous global->shared copies (LDGSTS). src_bytes < size zero-fills the tail.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(src_bytes));
}
// one element (8 or 4 bytes), zero-filled when !ok
__device__ __forceinline__ void cp_async_elem(double* smem, const double* gmem, bool ok) {
    cp_async8(smem, gmem, ok ? 8 : 0);
}
__device__ __forceinline__ void cp_async_elem(float* smem, const float* gmem, bool ok) {
    cp_async4(smem, gmem, ok ? 4 : 0);
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// FP64 tensor-core MMA (DMMA.8x8x4 on sm_100a): C[8x8] += A[8x4] * B[4x8].
// Fragment ownership (lane = 4*g + t): a = A[g][t], b = B[t][g],
// c0,c1 = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

}  // namespace sorsvd_dev
