// Small-k Gram matrix for CholeskyQR2 (cholqr_f64.cuh) at k <= 32, where the
// QR of a sketch is latency-bound (C1: k = 20, C4: k = 10, every RPCA
// iteration). gram_tall_kernel<K>: G = T^T T for a tall T (rows x K, pitch
// ldt) in one launch. Each warp accumulates a K x K partial over its rows in
// registers (the row is broadcast from the lane that loaded it), the CTA's
// warps are summed through shared memory in a fixed order, and the last CTA
// to finish (atomic ticket) adds the CTA partials in CTA order --
// deterministic for a given grid -- and writes G. Replaces a split-K TN GEMM
// plus its reduction kernel (C4: 24 -> 17 us per Gram; measured dead ends:
// a one-warp Cholesky and a one-warp Jacobi were 2x slower than the CTA
// kernels, their FP64 sqrt / divide / FMA chains fully exposed).
#pragma once
#include "common.cuh"

namespace sorsvd_dev {

constexpr int kGramThreads = 256;

template <int K>
__global__ void __launch_bounds__(kGramThreads) gram_tall_kernel(const double* __restrict__ T, int64_t ldt, int64_t rows,
                                                                 int k, double* __restrict__ ws,
                                                                 unsigned int* __restrict__ ticket,
                                                                 double* __restrict__ G, int ldg, const int* pred,
                                                                 int pred_skip) {
    static_assert(K == 16 || K == 32, "K");
    if (pred_off(pred, pred_skip)) return;
    constexpr int CPL = K * K / 32;   // G entries per lane: row a = lane % K, columns [b0, b0 + CPL)
    constexpr int NW = kGramThreads / 32;
    static_assert(NW == 8, "the CTA sum below pairs warps w and w + 4");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int a = lane % K, b0 = (lane / K) * CPL;
    double acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
    const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per, r1 = r0 + per < rows ? r0 + per : rows;
    // four rows per trip, all loads issued before any is used
    int64_t r = r0 + warp;
    for (; r + 3 * NW < r1; r += 4 * NW) {
        double x[4], xa[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = lane < k ? T[(r + u * NW) * ldt + lane] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) xa[u] = __shfl_sync(0xffffffffu, x[u], a);
#pragma unroll
        for (int c = 0; c < CPL; ++c)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[c] = fma(xa[u], __shfl_sync(0xffffffffu, x[u], b0 + c), acc[c]);
    }
    for (; r < r1; r += NW) {
        const double x = lane < k ? T[r * ldt + lane] : 0.0;
        const double xa = __shfl_sync(0xffffffffu, x, a);
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = fma(xa, __shfl_sync(0xffffffffu, x, b0 + c), acc[c]);
    }
    // CTA sum in a fixed order: warps 0-3 store, warps 4-7 add onto them, then the 4 slots
    __shared__ double part[4][K * K];
    __shared__ bool last;
    if (warp < 4) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) part[warp][a * K + b0 + c] = acc[c];
    }
    __syncthreads();
    if (warp >= 4) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) part[warp - 4][a * K + b0 + c] += acc[c];
    }
    __syncthreads();
    double* mine = ws + (size_t)blockIdx.x * K * K;
    for (int e = threadIdx.x; e < K * K; e += kGramThreads) mine[e] = (part[0][e] + part[1][e]) + (part[2][e] + part[3][e]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int e = threadIdx.x; e < K * K; e += kGramThreads) {
        // the CTA partials in CTA order, loads issued 8 ahead of the (ordered) adds
        double s = 0.0;
        unsigned int bI = 0;
        for (; bI + 8 <= gridDim.x; bI += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(ws + (size_t)(bI + u) * K * K + e);
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        for (; bI < gridDim.x; ++bI) s += __ldcg(ws + (size_t)bI * K * K + e);
        const int i = e / K, j = e - i * K;
        if (i < k && j < k) G[(size_t)i * ldg + j] = s;
    }
    if (threadIdx.x == 0) *ticket = 0u;  // ready for the next launch (stream order)
}

}  // namespace sorsvd_dev

