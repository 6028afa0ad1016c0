// K1 o K2 for narrow sketches over a narrow matrix (ell <= 16, n <= 512): one power step
//   T1 = A X          (sketch.hpp:95, NN)
//   T2 = A^T T1       (sketch.hpp:96, TN)
// in ONE sweep over A, and the projection M = Q1^T (A Q2) (sketch.hpp:100-102) likewise.
//
// BASELINE config 4 (RPCA, W = 25344 x 300, ell = 10) runs five such passes per ALM iteration. Each
// is 2 m n ell = 0.15 GFLOP over a 60.8 MB matrix: on the generic skinny GEMM (gemm_f64.cuh: 64-row
// DMMA tiles, stream-K and a fix-up launch) a pass took ~35-40 us against 9.3 us of HBM time, and
// the pairs read W twice. Here every CTA owns a contiguous range of row blocks: a block (RB rows x
// n) is staged in shared memory by cp.async (double buffered), T1_b = W_b X is formed from it
// (X resident in shared memory), written out, and immediately contracted again against the SAME
// staged block, T2 += W_b^T T1_b, into DMMA accumulators that live across the CTA's blocks.
// Per-CTA partials of T2 are summed in CTA order by pair_reduce_kernel (deterministic).
// PROJ = true contracts T1_b against a second row-block operand L (Q1) instead: M += L_b^T T1_b.
// Both stages run on DMMA.8x8x4 fragments read from shared memory (pitches chosen so the fragment
// loads are bank-conflict free); a first version on plain FP64 FMAs was shared-memory-bandwidth
// bound (one 8-byte load per FMA) and slower than the two GEMM passes it replaced.
#pragma once
#include "common.cuh"

namespace sorsvd_dev {

constexpr int kPairThreads = 512;  // 16 warps: the two DMMA stages are latency chains, not throughput
constexpr int kPairNP = 16;    // sketch columns per row (zero padded): two 8-wide DMMA column tiles
constexpr int kPairLd = 20;    // shared-memory pitch of the 16-column operands: k rows 4 apart land on
                               // banks 8 apart, so a half-warp's fragment load is conflict free
constexpr int kPairMaxT2 = 4;  // second-stage row tiles per warp: ceil(ceil(n / 8) / 16), n <= 512

struct PairArgs {
    const double* A;   // m x n row-major (lda)
    int64_t lda, m;
    int n;
    const double* X;   // n x np right operand (Omega / T2 / Q2), row pitch ldx
    int ldx, np;       // np = real padded sketch width (8 or 16)
    double* T1;        // m x np output of the first stage (pitch ldt)
    int ldt;
    const double* L;   // PROJ: m x np left operand of the second stage (Q1), pitch ldl
    int ldl;
    double* part;      // [gridDim.x][rows2][16] partial second-stage sums, rows2 = n or 16
    int rb;            // rows per staged block: 16 or 32
    int vec;           // A rows 16-byte aligned: 16-byte cp.async
    const int* pred;
    int pred_skip;
};

// Row pitch of the staged block: n rounded up to 4 mod 8 doubles, so that rows (the k index of the
// second stage, the row index of the first) 1 apart land on banks 8 or 24 apart.
__host__ __device__ inline int pair_nld(int n) { return n + ((4 - n % 8) + 8) % 8; }

inline size_t pair_smem_bytes(int n, int rb, bool proj) {
    // staged blocks (double buffered), X, the K-split partials of T1_b (ksplit * rb = 128 rows), L_b
    return (size_t)(2 * rb * pair_nld(n) + n * kPairLd + 128 * kPairLd + (proj ? rb * kPairLd : 0)) * sizeof(double);
}

template <bool PROJ>
__global__ void __launch_bounds__(kPairThreads, 1) skinny_pair_kernel(PairArgs p) {
    if (pred_off(p.pred, p.pred_skip)) return;
    extern __shared__ __align__(16) double sm[];
    const int n = p.n, rb = p.rb, nld = pair_nld(n);
    const int mt1 = rb >> 3;        // first-stage row tiles (2 or 4)
    const int ksplit = 16 / mt1;    // warps sharing a row tile's K range (8 or 4)
    double* sW = sm;                                  // [2][rb][nld]
    double* sX = sW + 2 * rb * nld;                   // [n][kPairLd]
    double* sT = sX + n * kPairLd;                    // [ksplit][rb][kPairLd] K-split partials; [0] = T1_b
    double* sL = sT + ksplit * rb * kPairLd;          // [rb][kPairLd] (PROJ)
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, g = lane >> 2, t4 = lane & 3;

    for (int e = t; e < n * kPairNP; e += kPairThreads) {
        const int j = e >> 4, cc = e & 15;
        sX[j * kPairLd + cc] = cc < p.np ? p.X[(int64_t)j * p.ldx + cc] : 0.0;
    }
    // this CTA's contiguous range of row blocks
    const int64_t nblk = (p.m + rb - 1) / rb;
    const int64_t per = (nblk + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = (int64_t)blockIdx.x * per, b1 = b0 + per < nblk ? b0 + per : nblk;

    auto stage = [&](int64_t blk, int buf) {
        double* dst = sW + (size_t)buf * rb * nld;
        const int64_t row0 = blk * rb;
        if (p.vec) {
            const int cpr = (n + 1) >> 1;  // 16-byte chunks per row
            const int dr = kPairThreads / cpr, dc = kPairThreads - dr * cpr;
            int r = t / cpr, ch = t - r * cpr;  // this thread's chunks: t, t + 512, ... (no division per chunk)
            while (r < rb) {
                const int64_t row = row0 + r;
                const int rem = n - 2 * ch;  // doubles left in the row from this chunk
                const int bytes = row < p.m ? (rem >= 2 ? 16 : 8) : 0;
                cp_async16(dst + r * nld + 2 * ch, p.A + (row < p.m ? row : 0) * p.lda + 2 * ch, bytes);
                r += dr;
                ch += dc;
                if (ch >= cpr) {
                    ch -= cpr;
                    ++r;
                }
            }
        } else {
            for (int e = t; e < rb * n; e += kPairThreads) {
                const int r = e / n, j = e - r * n;
                const int64_t row = row0 + r;
                cp_async8(dst + r * nld + j, p.A + (row < p.m ? row : 0) * p.lda + j, row < p.m ? 8 : 0);
            }
        }
        cp_async_commit();
    };

    const int ks_all = (n + 3) >> 2;                    // first-stage K steps of 4
    const int ks_per = (ks_all + ksplit - 1) / ksplit;
    const int mt2_all = PROJ ? 2 : (n + 7) >> 3;        // second-stage output row tiles
    double acc2[kPairMaxT2][2][2];
#pragma unroll
    for (int i = 0; i < kPairMaxT2; ++i) acc2[i][0][0] = acc2[i][0][1] = acc2[i][1][0] = acc2[i][1][1] = 0.0;

    if (b0 < b1) stage(b0, 0);
    for (int64_t blk = b0; blk < b1; ++blk) {
        const int buf = (int)((blk - b0) & 1);
        if (blk + 1 < b1) {
            stage(blk + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        const int64_t row0 = blk * rb;
        if (PROJ) {
            for (int e = t; e < rb * kPairNP; e += kPairThreads) {
                const int r = e >> 4, cc = e & 15;
                const int64_t row = row0 + r;
                sL[r * kPairLd + cc] = (row < p.m && cc < p.np) ? p.L[row * p.ldl + cc] : 0.0;
            }
        }
        __syncthreads();  // block `blk` (and sX on the first trip) visible
        const double* W = sW + (size_t)buf * rb * nld;
        // ---- stage 1: T1_b (rb x 16) = W_b X on DMMA tiles; warp = (row tile, K part) ----
        {
            const int mt = warp % mt1, kp = warp / mt1;
            double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;  // even K steps
            double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;  // odd K steps (a second, independent DMMA chain)
            const double* wrow = W + (8 * mt + g) * nld;
            const int k_end = (kp + 1) * ks_per < ks_all ? (kp + 1) * ks_per : ks_all;
            for (int ks = kp * ks_per; ks < k_end; ks += 2) {
                const int j = 4 * ks + t4, j2 = j + 4;
                const bool ok = j < n, ok2 = ks + 1 < k_end && j2 < n;
                const double a = ok ? wrow[j] : 0.0;
                const double x0 = ok ? sX[j * kPairLd + g] : 0.0;
                const double x1 = ok ? sX[j * kPairLd + 8 + g] : 0.0;
                const double a2 = ok2 ? wrow[j2] : 0.0;
                const double y0 = ok2 ? sX[j2 * kPairLd + g] : 0.0;
                const double y1 = ok2 ? sX[j2 * kPairLd + 8 + g] : 0.0;
                dmma884(c00, c01, a, x0);
                dmma884(c10, c11, a, x1);
                dmma884(d00, d01, a2, y0);
                dmma884(d10, d11, a2, y1);
            }
            c00 += d00;
            c01 += d01;
            c10 += d10;
            c11 += d11;
            double* tp = sT + (size_t)kp * rb * kPairLd + (8 * mt + g) * kPairLd + 2 * t4;
            tp[0] = c00;
            tp[1] = c01;
            tp[8] = c10;
            tp[9] = c11;
        }
        __syncthreads();
        for (int e = t; e < rb * kPairNP; e += kPairThreads) {  // sum the K parts in order -> T1_b
            const int r = e >> 4, cc = e & 15;
            double v = sT[r * kPairLd + cc];
            for (int q = 1; q < ksplit; ++q) v += sT[(size_t)q * rb * kPairLd + r * kPairLd + cc];
            sT[r * kPairLd + cc] = v;
            if (cc < p.np && row0 + r < p.m) p.T1[(row0 + r) * p.ldt + cc] = v;
        }
        __syncthreads();  // T1_b complete
        // ---- stage 2: out (rows2 x 16) += left^T T1_b; warp takes output row tiles warp, warp + 8, ... ----
        if (!PROJ) {
            for (int ks = 0; ks < (rb >> 2); ++ks) {  // the tiles' DMMAs of one K step are independent
                const int r = 4 * ks + t4;
                const double y0 = sT[r * kPairLd + g], y1 = sT[r * kPairLd + 8 + g];
#pragma unroll
                for (int i = 0; i < kPairMaxT2; ++i) {
                    const int mt2 = warp + 16 * i;
                    if (mt2 < mt2_all) {
                        const int j = 8 * mt2 + g;
                        const double a = j < n ? W[r * nld + j] : 0.0;
                        dmma884(acc2[i][0][0], acc2[i][0][1], a, y0);
                        dmma884(acc2[i][1][0], acc2[i][1][1], a, y1);
                    }
                }
            }
        } else if (warp < 2) {
            for (int ks = 0; ks < (rb >> 2); ++ks) {
                const int r = 4 * ks + t4;
                const double a = sL[r * kPairLd + 8 * warp + g];
                const double y0 = sT[r * kPairLd + g], y1 = sT[r * kPairLd + 8 + g];
                dmma884(acc2[0][0][0], acc2[0][0][1], a, y0);
                dmma884(acc2[0][1][0], acc2[0][1][1], a, y1);
            }
        }
        __syncthreads();  // buffer `buf`, sT and sL are rewritten by the next trips
    }
    const int rows2 = PROJ ? kPairNP : n;
    double* out = p.part + (size_t)blockIdx.x * rows2 * kPairNP;
    if (!PROJ) {
#pragma unroll
        for (int i = 0; i < kPairMaxT2; ++i) {
            const int mt2 = warp + 16 * i;
            if (mt2 >= mt2_all) break;
            const int j = 8 * mt2 + g;
            if (j < n) {
                double* o = out + j * kPairNP + 2 * t4;
                o[0] = acc2[i][0][0];
                o[1] = acc2[i][0][1];
                o[8] = acc2[i][1][0];
                o[9] = acc2[i][1][1];
            }
        }
    } else if (warp < 2) {
        double* o = out + (8 * warp + g) * kPairNP + 2 * t4;
        o[0] = acc2[0][0][0];
        o[1] = acc2[0][0][1];
        o[8] = acc2[0][1][0];
        o[9] = acc2[0][1][1];
    }
}

// ---- two independent halves per CTA (n <= 320) ------------------------------------------------
// The one-pipeline kernel above leaves the tensor pipe 43% active: stage, contract, sum the K
// parts, contract again are a chain of short phases separated by block-wide barriers on a
// 1-CTA-per-SM kernel (shared memory rules out a second CTA). Here the 16 warps run as two halves
// of 8 warps that walk alternate 16-row blocks of the CTA's range, each with its own double-
// buffered staging area, K-part buffer and named barrier (bar.sync 1 / 2 over 256 threads), and
// share only X: while one half sits in a barrier or waits for cp.async, the other issues DMMAs.
// The halves' accumulators are added through shared memory at the end (half 1 first into the
// buffer, half 0 adds and writes the CTA's partial: fixed order).
constexpr int kPair2MaxT2 = 5;   // output row tiles per warp: ceil(ceil(n / 8) / 8), n <= 320
constexpr int kPair2Rb = 16;

inline size_t pair2_smem_bytes(int n, bool proj) {
    const int per_half = 2 * kPair2Rb * pair_nld(n) + 4 * kPair2Rb * kPairLd + (proj ? kPair2Rb * kPairLd : 0);
    return (size_t)(n * kPairLd + 2 * per_half) * sizeof(double);
}

__device__ __forceinline__ void pair_half_sync(int half) {
    asm volatile("bar.sync %0, 256;\n" ::"r"(1 + half) : "memory");
}

template <bool PROJ>
__global__ void __launch_bounds__(kPairThreads, 1) skinny_pair2_kernel(PairArgs p) {
    if (pred_off(p.pred, p.pred_skip)) return;
    extern __shared__ __align__(16) double sm[];
    constexpr int rb = kPair2Rb, mt1 = 2, ksplit = 4;
    const int n = p.n, nld = pair_nld(n);
    const int per_half = 2 * rb * nld + ksplit * rb * kPairLd + (PROJ ? rb * kPairLd : 0);
    const int t = threadIdx.x, half = t >> 8, ht = t & 255, hw = ht >> 5, lane = t & 31, g = lane >> 2, t4 = lane & 3;
    double* sX = sm;                                    // [n][kPairLd], shared by the halves
    double* sW = sX + n * kPairLd + half * per_half;    // [2][rb][nld]
    double* sT = sW + 2 * rb * nld;                     // [ksplit][rb][kPairLd]
    double* sL = sT + ksplit * rb * kPairLd;            // [rb][kPairLd] (PROJ)

    for (int e = t; e < n * kPairNP; e += kPairThreads) {
        const int j = e >> 4, cc = e & 15;
        sX[j * kPairLd + cc] = cc < p.np ? p.X[(int64_t)j * p.ldx + cc] : 0.0;
    }
    // the CTA's contiguous range of 16-row blocks; half h takes blocks b0 + h, b0 + h + 2, ...
    const int64_t nblk = (p.m + rb - 1) / rb;
    const int64_t per = (nblk + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = (int64_t)blockIdx.x * per + half;
    const int64_t b1 = (int64_t)blockIdx.x * per + per < nblk ? (int64_t)blockIdx.x * per + per : nblk;

    auto stage = [&](int64_t blk, int buf) {
        double* dst = sW + (size_t)buf * rb * nld;
        const int64_t row0 = blk * rb;
        if (p.vec) {
            const int cpr = (n + 1) >> 1;
            const int dr = 256 / cpr, dc = 256 - dr * cpr;
            int r = ht / cpr, ch = ht - r * cpr;
            while (r < rb) {
                const int64_t row = row0 + r;
                const int rem = n - 2 * ch;
                const int bytes = row < p.m ? (rem >= 2 ? 16 : 8) : 0;
                cp_async16(dst + r * nld + 2 * ch, p.A + (row < p.m ? row : 0) * p.lda + 2 * ch, bytes);
                r += dr;
                ch += dc;
                if (ch >= cpr) {
                    ch -= cpr;
                    ++r;
                }
            }
        } else {
            for (int e = ht; e < rb * n; e += 256) {
                const int r = e / n, j = e - r * n;
                const int64_t row = row0 + r;
                cp_async8(dst + r * nld + j, p.A + (row < p.m ? row : 0) * p.lda + j, row < p.m ? 8 : 0);
            }
        }
        cp_async_commit();
    };

    const int ks_all = (n + 3) >> 2;
    const int ks_per = (ks_all + ksplit - 1) / ksplit;
    const int mt2_all = PROJ ? 2 : (n + 7) >> 3;
    double acc2[kPair2MaxT2][2][2];
#pragma unroll
    for (int i = 0; i < kPair2MaxT2; ++i) acc2[i][0][0] = acc2[i][0][1] = acc2[i][1][0] = acc2[i][1][1] = 0.0;

    if (b0 < b1) stage(b0, 0);
    __syncthreads();  // sX complete (the only block-wide barrier before the epilogue)
    int trip = 0;
    for (int64_t blk = b0; blk < b1; blk += 2, ++trip) {
        const int buf = trip & 1;
        if (blk + 2 < b1) {
            stage(blk + 2, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        const int64_t row0 = blk * rb;
        if (PROJ) {
            const int r = ht >> 4, cc = ht & 15;  // rb * 16 = 256 elements: one per thread
            const int64_t row = row0 + r;
            sL[r * kPairLd + cc] = (row < p.m && cc < p.np) ? p.L[row * p.ldl + cc] : 0.0;
        }
        pair_half_sync(half);  // this half's block visible
        const double* W = sW + (size_t)buf * rb * nld;
        {   // stage 1: T1_b (16 x 16) = W_b X; warp = (row tile, K part), two interleaved DMMA chains
            const int mt = hw % mt1, kp = hw / mt1;
            double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0, d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
            const double* wrow = W + (8 * mt + g) * nld;
            const int k_end = (kp + 1) * ks_per < ks_all ? (kp + 1) * ks_per : ks_all;
            for (int ks = kp * ks_per; ks < k_end; ks += 2) {
                const int j = 4 * ks + t4, j2 = j + 4;
                const bool ok = j < n, ok2 = ks + 1 < k_end && j2 < n;
                const double a = ok ? wrow[j] : 0.0;
                const double x0 = ok ? sX[j * kPairLd + g] : 0.0;
                const double x1 = ok ? sX[j * kPairLd + 8 + g] : 0.0;
                const double a2 = ok2 ? wrow[j2] : 0.0;
                const double y0 = ok2 ? sX[j2 * kPairLd + g] : 0.0;
                const double y1 = ok2 ? sX[j2 * kPairLd + 8 + g] : 0.0;
                dmma884(c00, c01, a, x0);
                dmma884(c10, c11, a, x1);
                dmma884(d00, d01, a2, y0);
                dmma884(d10, d11, a2, y1);
            }
            double* tp = sT + (size_t)kp * rb * kPairLd + (8 * mt + g) * kPairLd + 2 * t4;
            tp[0] = c00 + d00;
            tp[1] = c01 + d01;
            tp[8] = c10 + d10;
            tp[9] = c11 + d11;
        }
        pair_half_sync(half);
        {   // sum the K parts in order -> T1_b; 256 elements, one per thread
            const int r = ht >> 4, cc = ht & 15;
            double v = sT[r * kPairLd + cc];
#pragma unroll
            for (int q = 1; q < ksplit; ++q) v += sT[(size_t)q * rb * kPairLd + r * kPairLd + cc];
            sT[r * kPairLd + cc] = v;
            if (cc < p.np && row0 + r < p.m) p.T1[(row0 + r) * p.ldt + cc] = v;
        }
        pair_half_sync(half);
        if (!PROJ) {  // stage 2: T2 (n x 16) += W_b^T T1_b
#pragma unroll
            for (int ks = 0; ks < (rb >> 2); ++ks) {
                const int r = 4 * ks + t4;
                const double y0 = sT[r * kPairLd + g], y1 = sT[r * kPairLd + 8 + g];
#pragma unroll
                for (int i = 0; i < kPair2MaxT2; ++i) {
                    const int mt2 = hw + 8 * i;
                    if (mt2 < mt2_all) {
                        const int j = 8 * mt2 + g;
                        const double a = j < n ? W[r * nld + j] : 0.0;
                        dmma884(acc2[i][0][0], acc2[i][0][1], a, y0);
                        dmma884(acc2[i][1][0], acc2[i][1][1], a, y1);
                    }
                }
            }
        } else if (hw < 2) {
#pragma unroll
            for (int ks = 0; ks < (rb >> 2); ++ks) {
                const int r = 4 * ks + t4;
                const double a = sL[r * kPairLd + 8 * hw + g];
                const double y0 = sT[r * kPairLd + g], y1 = sT[r * kPairLd + 8 + g];
                dmma884(acc2[0][0][0], acc2[0][0][1], a, y0);
                dmma884(acc2[0][1][0], acc2[0][1][1], a, y1);
            }
        }
        pair_half_sync(half);  // this half's buffers are rewritten by its next trips
    }
    // epilogue: half 1's accumulators through shared memory (its own staging area), half 0 adds
    const int rows2 = PROJ ? kPairNP : n;
    double* xch = sm + n * kPairLd + per_half;  // half 1's area: rows2 x 16 doubles fit in its staging buffers
    __syncthreads();
    if (half == 1) {
        if (!PROJ) {
#pragma unroll
            for (int i = 0; i < kPair2MaxT2; ++i) {
                const int mt2 = hw + 8 * i;
                if (mt2 >= mt2_all) break;
                const int j = 8 * mt2 + g;
                if (j < n) {
                    double* o = xch + j * kPairNP + 2 * t4;
                    o[0] = acc2[i][0][0], o[1] = acc2[i][0][1], o[8] = acc2[i][1][0], o[9] = acc2[i][1][1];
                }
            }
        } else if (hw < 2) {
            double* o = xch + (8 * hw + g) * kPairNP + 2 * t4;
            o[0] = acc2[0][0][0], o[1] = acc2[0][0][1], o[8] = acc2[0][1][0], o[9] = acc2[0][1][1];
        }
    }
    __syncthreads();
    if (half == 0) {
        double* out = p.part + (size_t)blockIdx.x * rows2 * kPairNP;
        if (!PROJ) {
#pragma unroll
            for (int i = 0; i < kPair2MaxT2; ++i) {
                const int mt2 = hw + 8 * i;
                if (mt2 >= mt2_all) break;
                const int j = 8 * mt2 + g;
                if (j < n) {
                    const double* x = xch + j * kPairNP + 2 * t4;
                    double* o = out + j * kPairNP + 2 * t4;
                    o[0] = acc2[i][0][0] + x[0];
                    o[1] = acc2[i][0][1] + x[1];
                    o[8] = acc2[i][1][0] + x[8];
                    o[9] = acc2[i][1][1] + x[9];
                }
            }
        } else if (hw < 2) {
            const double* x = xch + (8 * hw + g) * kPairNP + 2 * t4;
            double* o = out + (8 * hw + g) * kPairNP + 2 * t4;
            o[0] = acc2[0][0][0] + x[0];
            o[1] = acc2[0][0][1] + x[1];
            o[8] = acc2[0][1][0] + x[8];
            o[9] = acc2[0][1][1] + x[9];
        }
    }
}

// out[j][c] = sum over CTAs of part[cta][j][c] (c < np, j < rows_out: the projection's partials carry
// 16 rows, M has np). A block owns 32 consecutive outputs; its 8 warps each sum a contiguous slice of
// the CTAs (independent, coalesced loads), and warp 0 adds the 8 slice sums in slice order:
// deterministic, and 8 x shorter than one thread walking all the partials.
__global__ void __launch_bounds__(256) pair_reduce_kernel(const double* __restrict__ part, int nctas, int rows2,
                                                          int rows_out, int np, double* __restrict__ out, int ldo,
                                                          const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    __shared__ double red[8][32];
    const int lane = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int e = blockIdx.x * 32 + lane;
    const int per = (nctas + 7) / 8;
    const int b0 = sl * per, b1 = b0 + per < nctas ? b0 + per : nctas;
    double s = 0.0;
    if (e < rows2 * kPairNP) {
#pragma unroll 4
        for (int b = b0; b < b1; ++b) s += part[(size_t)b * rows2 * kPairNP + e];
    }
    red[sl][lane] = s;
    __syncthreads();
    if (sl == 0 && e < rows2 * kPairNP) {
        double v = red[0][lane];
#pragma unroll
        for (int q = 1; q < 8; ++q) v += red[q][lane];
        const int j = e >> 4, c = e & 15;
        if (c < np && j < rows_out) out[(int64_t)j * ldo + c] = v;
    }
}

}  // namespace sorsvd_dev
