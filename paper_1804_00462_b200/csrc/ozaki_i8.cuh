// K1/K2/K4 on the INT8 tensor cores: FP64 skinny GEMM by the Ozaki scheme.
//
// The A-streaming passes (sketch.hpp:95 T1 = A*X, :96 T2 = A^T*T1, :100-102
// Y = A*Q2 -> cblas_dgemm, dense.hpp:30) have arithmetic intensity 2*ell/8
// FLOP/B: at ell >= 20 they are bound by the FP64 tensor pipe (DMMA.8x8x4,
// 37 TFLOP/s on B200), not by HBM (6.5 TB/s). The INT8 tensor pipe
// (tcgen05.mma.kind::i8, 4.5 POPS dense) is 120x faster, and products of
// 8-bit integers accumulate exactly in 32 bits, so an FP64 product can be
// assembled from int8 slice products without rounding inside the
// contraction (Ozaki, Ogita, Oishi, Rump 2012; the emulation cuBLAS 13 ships
// for DGEMM on Blackwell):
//
//   * Each left row r (a row of A for NN, a column of A for TN) is scaled by
//     2^(54 - e_r), e_r = the exponent bound of the row's largest |entry|
//     (max < 2^e_r), and rounded to an integer X, |X| <= 2^54 (a 2^-55
//     relative grid: finer than the max entry's own 53-bit mantissa). Adding
//     0x80 to each of the six low bytes turns X into seven balanced signed
//     base-256 digits d_0..d_6 (d_t = byte_t ^ 0x80 for t < 6, d_6 = the top
//     byte, |d_6| <= 64): X = sum_t d_t 256^t, every digit an int8. The right
//     operand (X = Omega / T1 / Q2, K x ell) is cut the same way per column c
//     (exponent f_c).
//   * a_rk x_kc = 2^(e_r + f_c - 108) sum_{t,u} d_t(a) d_u(x) 256^(t+u). The
//     slice products with t + u >= 5 (34 of the 49) are int8 MMAs summed in
//     exact int32 per level L = t + u in TMEM (levels 5..12 x 64 columns = the
//     whole 512-column TMEM); |sum| <= 7 * 16384 * 128^2 < 2^31 over a
//     16384-deep K chunk, after which the levels are drained into FP64
//     registers: acc += S_L * 2^(8L - 108) (exact scaling, one rounding each).
//   * Error per output: the representation (2^-55 max|row| |x| per term) and
//     the dropped levels L <= 4 (per term <= 5 * 2^-62 of max|a| max|x|), both
//     at or below the sqrt(K) eps |a||x| rounding of the reference's own dgemm
//     sums (measured: max error / (sqrt(K) max|a| max|x|) ~ 1e-15).
//     Non-finite entries are carried as NaN outputs of their row / column
//     (the integer path would otherwise swallow them).
//
// Kernel (one CTA per SM, 640 threads): a 128-row x 64-column output tile.
//   warp 0      streams the A tile of each K step (128 x 32, FP64 or FP32)
//               with TMA (128B swizzle) into a 2-stage ring;
//   warp 3      bulk-copies the precomputed X digit planes of each K step
//               (7 x 64 x 32 B) into the 3-stage digit ring;
//   warp 1      one lane issues the 34 tcgen05.mma (M 128, N 64, K 32) of
//               each step and frees the stage with tcgen05.commit;
//   warp 2      allocates / frees the 512 TMEM columns;
//   warps 4-19  cut the staged A tile into the 7 digit planes in shared
//               memory (no-swizzle K-major core-matrix layout; thread = row x
//               8-deep K quarter), and at each chunk end drain the TMEM levels
//               of their row x 16 columns, small levels first, into the
//               output (written by the first chunk, added by later ones).
//   (An A whose rows are not 16-byte aligned -- odd lda -- is read by the
//   converters straight from global memory instead: TMA_A = false.)
// The X digit planes and the scale exponents come from ozaki_xdigits_kernel
// and ozaki_absmax_kernel (one read of A per call for both orientations).
#pragma once
#include <climits>

#include "common.cuh"
#include "tc_gemm_f32.cuh"  // mbarrier / descriptor helpers

namespace sorsvd_dev {

constexpr int kOzSlices = 7;            // 7 signed base-256 digits of a 55-bit integer
// Lowest digit-pair level t + u kept. 5: 34 of the 49 products, dropped terms <= 5 * 2^-62 of
// max|a| max|x| (below the 2^-55 grid of the operands themselves). 6: 28 products, dropped terms
// <= 6 * 2^-56 (the size of FP64's own product rounding).
#ifndef OZ_LEVEL0
#define OZ_LEVEL0 5
#endif
constexpr int kOzLevel0 = OZ_LEVEL0;    // lowest level kept
constexpr int kOzLevels = 13 - kOzLevel0;  // t + u in [kOzLevel0, 12]
constexpr int kOzProducts = kOzLevel0 == 5 ? 34 : 28;
static_assert(kOzLevel0 == 5 || kOzLevel0 == 6, "digit-pair lists exist for level 5 and 6 cuts");
constexpr int kOzBM = 128;              // left rows per tile (TMEM lanes)
constexpr int kOzBN = 64;               // right columns per tile (8 levels x 64 = 512 TMEM columns)
constexpr int kOzBK = 32;               // K per step (one i8 MMA)
constexpr int kOzDStages = 3;           // digit-plane ring (A digits + X digits per K step)
constexpr int kOzAStages = 2;           // FP64 / FP32 A tile ring filled by TMA
constexpr int kOzAStageBytes = 32768;   // 128 x 32 doubles (FP32: 16 KB used)
constexpr int kOzThreads = 640;        // 4 control warps + 16 converter warps
constexpr int kOzChunkSteps = 512;      // K steps between TMEM drains (16384 deep: exact int32)
constexpr int kOzAPlane = kOzBM * kOzBK;             // 4096 B per digit plane of the left tile
constexpr int kOzXPlane = kOzBN * kOzBK;             // 2048 B per digit plane of the right tile
constexpr int kOzXStep = kOzSlices * kOzXPlane;      // 14336 B of X digits per (K step, column chunk)
constexpr int kOzStage = kOzSlices * kOzAPlane + kOzXStep;  // 43008 B
constexpr size_t kOzSmem = 1024 + (size_t)kOzDStages * kOzStage + (size_t)kOzAStages * kOzAStageBytes + 512;
constexpr int kOzNonFinite = INT_MAX;   // exponent sentinel: the row / column held NaN or Inf
constexpr long long kOzBias = 0x0000808080808080ll;  // +0x80 in each of the six low bytes: balanced digits

struct OzArgs {
    const void* A;        // double or float, row-major m x n (lda)
    int64_t lda;
    int64_t M;            // left rows: m (NN) or n (TN)
    int64_t K;            // n (NN) or m (TN)
    const int* lexp;      // per left row: e_r (max|row| < 2^e_r), or kOzNonFinite
    const int8_t* Xd;     // digit planes [K step][column chunk][slice][64 x 32 B]
    const int* xexp;      // per right column (padded): f_c, or kOzNonFinite
    int NC;               // column chunks of 64
    int N;                // real output columns (<= NC * 64)
    double* C;            // M x ldc output
    int64_t ldc;
    int vec;              // rows of A start 16-byte aligned (lda % (16 / sizeof(AT)) == 0): vector loads (NN)
    int acc0;             // 1: add to C from the first chunk on (another launch wrote the rest of the K range)
    int dbg;              // timing experiments only: 1 = no MMAs, 2 = no A conversion, 4 = no digit stores
    const int* pred;
    int pred_skip;
};

// kind::i8 instruction descriptor: D s32, A/B s8, both K-major, N, M.
__host__ __device__ constexpr uint32_t i8_idesc(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// The digit-plane words of 4 consecutive (scaled) values: w[t] holds digit t of the
// four values in its bytes 0..3. X_i = rint(v_i) (|X_i| <= 2^54), Y_i = X_i + bias;
// a 4 x 4 byte transpose of the low / high words of Y gathers the planes, and
// XOR 0x80 recentres the six low digits (the top byte is already signed).
__device__ __forceinline__ void oz_digit_words(const double v[4], uint32_t w[kOzSlices]) {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const unsigned long long y = (unsigned long long)(__double2ll_rn(v[i]) + kOzBias);
        lo[i] = (uint32_t)y;
        hi[i] = (uint32_t)(y >> 32);
    }
    const uint32_t a0 = __byte_perm(lo[0], lo[1], 0x5140), a1 = __byte_perm(lo[0], lo[1], 0x7362);
    const uint32_t a2 = __byte_perm(lo[2], lo[3], 0x5140), a3 = __byte_perm(lo[2], lo[3], 0x7362);
    const uint32_t b0 = __byte_perm(hi[0], hi[1], 0x5140), b1 = __byte_perm(hi[0], hi[1], 0x7362);
    const uint32_t b2 = __byte_perm(hi[2], hi[3], 0x5140), b3 = __byte_perm(hi[2], hi[3], 0x7362);
    w[0] = __byte_perm(a0, a2, 0x5410) ^ 0x80808080u;
    w[1] = __byte_perm(a0, a2, 0x7632) ^ 0x80808080u;
    w[2] = __byte_perm(a1, a3, 0x5410) ^ 0x80808080u;
    w[3] = __byte_perm(a1, a3, 0x7632) ^ 0x80808080u;
    w[4] = __byte_perm(b0, b2, 0x5410) ^ 0x80808080u;
    w[5] = __byte_perm(b0, b2, 0x7632) ^ 0x80808080u;
    w[6] = __byte_perm(b1, b3, 0x5410);  // top digit: byte 6, signed as it stands
}

__device__ __forceinline__ double oz_scale(int e) {  // 2^(54 - e) (0 for the sentinel / empty rows)
    return e == kOzNonFinite ? 0.0 : __longlong_as_double((long long)(1023 + 54 - e) << 52);
}

// ---------------------------------------------------------------- scales ----
// Bit patterns of non-negative doubles order like the values (NaN above Inf).
__device__ __forceinline__ void oz_atomic_max(unsigned long long* p, double v) {
    atomicMax(p, (unsigned long long)__double_as_longlong(v));
}

// max |A_ij| over each row (rowmax, m) and over each column (colmax, n) of a
// row-major m x n block: one read of A. Tile: 64 rows x 512 columns per CTA.
template <typename AT>
__global__ void __launch_bounds__(256) ozaki_absmax_kernel(const AT* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                                           unsigned long long* __restrict__ rowmax,
                                                           unsigned long long* __restrict__ colmax) {
    __shared__ unsigned long long srow[64];
    const int64_t r0 = (int64_t)blockIdx.y * 64;
    const int64_t c = (int64_t)blockIdx.x * 512 + 2 * threadIdx.x;
    if (threadIdx.x < 64) srow[threadIdx.x] = 0ull;
    __syncthreads();
    double cm0 = 0.0, cm1 = 0.0;
    const int rows = m - r0 < 64 ? (int)(m - r0) : 64;
    for (int r = 0; r < rows; ++r) {
        const AT* row = A + (r0 + r) * lda;
        double v0 = 0.0, v1 = 0.0;
        if (c < n) v0 = fabs((double)row[c]);
        if (c + 1 < n) v1 = fabs((double)row[c + 1]);
        // NaN must win every max: fmax would drop it
        cm0 = (v0 > cm0 || v0 != v0) ? v0 : cm0;
        cm1 = (v1 > cm1 || v1 != v1) ? v1 : cm1;
        double w = (v1 > v0 || v1 != v1) ? v1 : v0;
        for (int o = 16; o > 0; o >>= 1) {
            const double x = __shfl_xor_sync(0xffffffffu, w, o);
            w = (x > w || x != x) ? x : w;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(&srow[r], (unsigned long long)__double_as_longlong(w));
    }
    __syncthreads();
    if (threadIdx.x < rows) oz_atomic_max(rowmax + r0 + threadIdx.x, __longlong_as_double((long long)srow[threadIdx.x]));
    if (c < n) oz_atomic_max(colmax + c, cm0);
    if (c + 1 < n) oz_atomic_max(colmax + c + 1, cm1);
}

// max |entry| -> exponent e with max < 2^e (frexp), kOzNonFinite for NaN / Inf,
// 0 for an all-zero row (its digits are all zero).
__global__ void ozaki_exp_kernel(const unsigned long long* __restrict__ mx, int64_t count, int* __restrict__ e_out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = __longlong_as_double((long long)mx[i]);
        int e = 0;
        if (!isfinite(v)) {
            e = kOzNonFinite;
        } else if (v > 0.0) {
            frexp(v, &e);  // v = f 2^e, f in [0.5, 1): v < 2^e
        }
        e_out[i] = e;
    }
}

// max |X_kn| over k for each column of the right operand (K x N row-major, ldx). A block takes
// 32 columns x 64 rows (thread = column x one of 8 row lanes, 8 rows each: a warp reads 256
// contiguous bytes of a row), reduces its 8 row lanes through shared memory and issues one
// atomic per column. (The first version gave a thread a column and 256 rows: 16 blocks on C2's
// K = 4000, 34-146 us of serial loads per launch.)
constexpr int kOzCmRows = 64;
__device__ __forceinline__ double oz_nanmax(double a, double b) { return (b > a || b != b) ? b : a; }
__global__ void __launch_bounds__(256) ozaki_colmax_kernel(const double* __restrict__ X, int64_t ldx, int64_t K, int N,
                                                           unsigned long long* __restrict__ xmax) {
    __shared__ double red[8][33];
    const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
    const int n = blockIdx.x * 32 + cx;
    double mv = 0.0;
    if (n < N) {
        for (int64_t k0 = (int64_t)blockIdx.y * kOzCmRows; k0 < K; k0 += (int64_t)gridDim.y * kOzCmRows) {
#pragma unroll
            for (int i = 0; i < kOzCmRows / 8; ++i) {
                const int64_t k = k0 + ry + 8 * i;
                if (k < K) mv = oz_nanmax(mv, fabs(X[k * ldx + n]));
            }
        }
    }
    red[ry][cx] = mv;
    __syncthreads();
    if (ry == 0 && n < N) {
#pragma unroll
        for (int q = 1; q < 8; ++q) mv = oz_nanmax(mv, red[q][cx]);
        oz_atomic_max(xmax + n, mv);
    }
}

// Digit planes of the right operand X (K x N row-major, ldx; columns padded
// to NC * 64 with zeros) with per-column exponents xexp: thread (column n,
// 16-deep K half of a step) writes its 16 bytes of each of the 7 planes.
__global__ void ozaki_xdigits_kernel(const double* __restrict__ X, int64_t ldx, int64_t K, int N, int NC,
                                     const int* __restrict__ xexp, int8_t* __restrict__ Xd) {
    const int64_t KT = (K + kOzBK - 1) / kOzBK;
    const int64_t total = KT * 2 * (int64_t)NC * kOzBN;  // (K step, half, column)
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
        const int ncol = (int)(w % ((int64_t)NC * kOzBN));
        const int64_t kh = w / ((int64_t)NC * kOzBN);
        const int h = (int)(kh & 1);
        const int64_t kt = kh >> 1;
        const int nc = ncol / kOzBN, nl = ncol % kOzBN;
        const double s = ncol < N ? oz_scale(xexp[ncol]) : 0.0;
        uint32_t words[kOzSlices][4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            double v[4];
            uint32_t w[kOzSlices];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t k = kt * kOzBK + 16 * h + 4 * q4 + q;
                v[q] = (k < K && ncol < N) ? X[k * ldx + ncol] * s : 0.0;
            }
            oz_digit_words(v, w);
#pragma unroll
            for (int t = 0; t < kOzSlices; ++t) words[t][q4] = w[t];
        }
        // the 7 planes of a (step, column chunk) stacked along N as one 448 x 32 B K-major
        // operand: core matrices of 8 rows x 16 B, 8-row groups 128 B apart (SBO), the two
        // 16-byte K halves 7168 B apart (LBO); plane u starts at row group 8u
        int8_t* base = Xd + (kt * NC + nc) * (int64_t)kOzXStep + h * (kOzXStep / 2) + (nl / 8) * 128 + (nl % 8) * 16;
#pragma unroll
        for (int t = 0; t < kOzSlices; ++t)
            *reinterpret_cast<uint4*>(base + (int64_t)t * 1024) =
                make_uint4(words[t][0], words[t][1], words[t][2], words[t][3]);
    }
}

__device__ __forceinline__ void oz_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void oz_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
template <bool TA, typename AT, bool TMA_A>
__global__ void __launch_bounds__(kOzThreads, 1)
    ozaki_gemm_kernel(const __grid_constant__ CUtensorMap tmA, OzArgs p) {
    if (pred_off(p.pred, p.pred_skip)) return;
    extern __shared__ __align__(1024) uint8_t smraw[];
    const uint32_t base = (smem_u32(smraw) + 1023u) & ~1023u;
    uint8_t* gbase = smraw + (base - smem_u32(smraw));
    const uint32_t stg0 = base + kOzDStages * kOzStage;  // A staging ring (TMA_A), 1024-aligned
    const uint32_t bar0 = stg0 + kOzAStages * kOzAStageBytes;
    auto full_a = [&](int s) { return bar0 + 8u * s; };
    auto full_x = [&](int s) { return bar0 + 8u * (kOzDStages + s); };
    auto empty = [&](int s) { return bar0 + 8u * (2 * kOzDStages + s); };
    auto a_full = [&](int s) { return bar0 + 8u * (3 * kOzDStages + s); };
    auto a_empty = [&](int s) { return bar0 + 8u * (3 * kOzDStages + kOzAStages + s); };
    const uint32_t drain_full = bar0 + 8u * (3 * kOzDStages + 2 * kOzAStages);
    const uint32_t drain_empty = drain_full + 8u;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (drain_empty + 8u - base));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x / p.NC, nc = blockIdx.x % p.NC;
    const int64_t m0 = (int64_t)mt * kOzBM;
    const int KT = (int)((p.K + kOzBK - 1) / kOzBK);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kOzDStages; ++s) {
            mbar_init(full_a(s), 16);  // one arrive per converter warp
            mbar_init(full_x(s), 1);
            mbar_init(empty(s), 1);
        }
        for (int s = 0; s < kOzAStages; ++s) {
            mbar_init(a_full(s), 1);
            mbar_init(a_empty(s), 16);      // one arrive per converter warp
        }
        mbar_init(drain_full, 1);
        mbar_init(drain_empty, 16);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if (TMA_A) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (TMA_A && lane == 0) {  // ---- A tile producer (TMA, 128B swizzle) ----
            for (int kt = 0; kt < KT; ++kt) {
                const int s = kt % kOzAStages;
                const uint32_t ph = (uint32_t)(kt / kOzAStages) & 1u;
                mbar_wait(a_empty(s), ph ^ 1u);
                const uint32_t dst = stg0 + s * kOzAStageBytes;
                const int k0 = kt * kOzBK;
                if (sizeof(AT) == 8) {
                    mbar_expect_tx(a_full(s), 32768u);
                    if (!TA) {  // {K, M} boxes {16, 128}: the two 16-deep K halves
                        tma_load_2d(dst, &tmA, a_full(s), k0, (int)m0);
                        tma_load_2d(dst + 16384, &tmA, a_full(s), k0 + 16, (int)m0);
                    } else {  // {M, K} boxes {16, 32}: 8 column groups of the 128 left rows
#pragma unroll
                        for (int b = 0; b < 8; ++b) tma_load_2d(dst + b * 4096, &tmA, a_full(s), (int)m0 + 16 * b, k0);
                    }
                } else {
                    mbar_expect_tx(a_full(s), 16384u);
                    if (!TA) {  // {K, M} box {32, 128}
                        tma_load_2d(dst, &tmA, a_full(s), k0, (int)m0);
                    } else {  // {M, K} boxes {32, 32}
#pragma unroll
                        for (int b = 0; b < 4; ++b) tma_load_2d(dst + b * 4096, &tmA, a_full(s), (int)m0 + 32 * b, k0);
                    }
                }
            }
        }
    } else if (warp == 3) {
        if (lane == 0) {  // ---- X digit producer (bulk copies) ----
            const int8_t* xsrc = p.Xd + (size_t)nc * kOzXStep;
            for (int kt = 0; kt < KT; ++kt) {
                const int s = kt % kOzDStages;
                const uint32_t ph = (uint32_t)(kt / kOzDStages) & 1u;
                mbar_wait(empty(s), ph ^ 1u);
                mbar_expect_tx(full_x(s), (uint32_t)kOzXStep);
                oz_bulk_g2s(base + s * kOzStage + kOzSlices * kOzAPlane, xsrc + (size_t)kt * p.NC * kOzXStep,
                            (uint32_t)kOzXStep, full_x(s));
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer ----
            for (int kt = 0; kt < KT; ++kt) {
                const int s = kt % kOzDStages;
                const uint32_t ph = (uint32_t)(kt / kOzDStages) & 1u;
                const int ck = kt % kOzChunkSteps;
                if (ck == 0) mbar_wait(drain_empty, (uint32_t)(kt / kOzChunkSteps) & 1u);  // TMEM zeroed
                mbar_wait(full_a(s), ph);
                mbar_wait(full_x(s), ph);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                const uint32_t a_s = base + s * kOzStage;
                const uint32_t x_s = a_s + kOzSlices * kOzAPlane;
                // A plane t times the X planes u0 .. u0+cnt-1 (stacked along N) in one MMA, its
                // cnt x 64 output columns landing on the consecutive TMEM levels t+u0 .. (TMEM is
                // zeroed by the drainers, so every MMA accumulates)
                auto mma = [&](int t, int u0, int cnt) {
                    const uint64_t da = umma_desc(a_s + t * kOzAPlane, 2048, 128, 0);
                    const uint64_t db = umma_desc(x_s + u0 * 1024, kOzXStep / 2, 128, 0);
                    const uint32_t idesc = i8_idesc(kOzBM, kOzBN * cnt);
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                            tmem + (uint32_t)((t + u0 - kOzLevel0) * kOzBN)),
                        "l"(da), "l"(db), "r"(idesc));
                };
                // all pairs with t + u >= 5 (digits 0..6, 6 = top)
                if (p.dbg & 1) {
                } else if constexpr (kOzLevel0 == 5) {
                    mma(6, 0, 4); mma(6, 4, 3);
                    mma(5, 0, 4); mma(5, 4, 3);
                    mma(4, 1, 4); mma(4, 5, 2);
                    mma(3, 2, 4); mma(3, 6, 1);
                    mma(2, 3, 4);
                    mma(1, 4, 3);
                    mma(0, 5, 2);
                } else {  // t + u >= 6
                    mma(6, 0, 4); mma(6, 4, 3);
                    mma(5, 1, 4); mma(5, 5, 2);
                    mma(4, 2, 4); mma(4, 6, 1);
                    mma(3, 3, 4);
                    mma(2, 4, 3);
                    mma(1, 5, 2);
                    mma(0, 6, 1);
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                 empty(s))
                             : "memory");
                if (ck == kOzChunkSteps - 1 || kt == KT - 1)
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(drain_full)
                        : "memory");
            }
        }
    } else if (warp >= 4) {
        // ---- converters / drainers: row r of the tile, K quarter kq of each step ----
        const int q = warp & 3;             // TMEM lane quarter
        const int kq = (warp - 4) >> 2;     // K quarter (conversion) and 16-column quarter (drain)
        const int r = 32 * q + lane;
        const int64_t row = m0 + r;
        const bool row_ok = row < p.M;
        const int e_row = row_ok ? p.lexp[row] : 0;
        const double sr = row_ok ? oz_scale(e_row) : 0.0;
        const AT* Ap = static_cast<const AT*>(p.A);
        // this thread's 8 bytes inside a digit plane: core matrix (row group, K half), row, K quarter
        const uint32_t a_off = (uint32_t)((r >> 3) * 128 + (kq >> 1) * 2048 + (r & 7) * 16 + (kq & 1) * 8);
        // this thread's TMEM row (lane) and 16-column quarter of every level
        const uint32_t t_row = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(16 * kq);
        auto zero_levels = [&]() {
#pragma unroll 1
            for (int L = 0; L < kOzLevels; ++L) {
                const uint32_t ta = t_row + (uint32_t)(L * kOzBN);
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(ta),
                    "r"(0u)
                    : "memory");
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            __syncwarp();
            if (lane == 0) oz_arrive(drain_empty);
        };
        zero_levels();
        const int c0 = nc * kOzBN + 16 * kq;  // this thread's output columns c0 .. c0+15
        int chunk = 0;
        for (int kt = 0; kt < KT; ++kt) {
            const int s = kt % kOzDStages;
            const uint32_t ph = (uint32_t)(kt / kOzDStages) & 1u;
            const int64_t k0 = (int64_t)kt * kOzBK + 8 * kq;
            double v[8];
            if (p.dbg & 2) {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = (double)(kt + i);
                if (TMA_A) {
                    const int sa = kt % kOzAStages;
                    mbar_wait(a_full(sa), (uint32_t)(kt / kOzAStages) & 1u);
                    __syncwarp();
                    if (lane == 0) oz_arrive(a_empty(sa));
                }
            } else if (TMA_A) {
                const int sa = kt % kOzAStages;
                mbar_wait(a_full(sa), (uint32_t)(kt / kOzAStages) & 1u);
                const uint8_t* stg = gbase + (stg0 - base) + (size_t)sa * kOzAStageBytes;
                if (sizeof(AT) == 8) {
                    if (!TA) {  // row r, K elements 8kq..8kq+7: box kq/2, 16-byte chunks 4(kq&1)..+3 (swizzled)
                        const uint8_t* rowp = stg + (kq >> 1) * 16384 + r * 128;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const double2 x = *reinterpret_cast<const double2*>(rowp + (((4 * (kq & 1) + j) ^ (r & 7)) << 4));
                            v[2 * j] = x.x;
                            v[2 * j + 1] = x.y;
                        }
                    } else {  // column r of rows 8kq..8kq+7: box r / 16, element r % 16
                        const uint8_t* bp = stg + (r >> 4) * 4096 + (r & 1) * 8;
                        const int jc = (r & 15) >> 1;
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int il = 8 * kq + i;
                            v[i] = *reinterpret_cast<const double*>(bp + il * 128 + ((jc ^ (il & 7)) << 4));
                        }
                    }
                } else {
                    if (!TA) {  // floats 8kq..8kq+7 of row r: chunks 2kq, 2kq+1
                        const uint8_t* rowp = stg + r * 128;
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            const float4 x = *reinterpret_cast<const float4*>(rowp + (((2 * kq + j) ^ (r & 7)) << 4));
                            v[4 * j] = x.x;
                            v[4 * j + 1] = x.y;
                            v[4 * j + 2] = x.z;
                            v[4 * j + 3] = x.w;
                        }
                    } else {  // column r: box r / 32, element r % 32
                        const uint8_t* bp = stg + (r >> 5) * 4096 + (r & 3) * 4;
                        const int jc = (r & 31) >> 2;
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int il = 8 * kq + i;
                            v[i] = *reinterpret_cast<const float*>(bp + il * 128 + ((jc ^ (il & 7)) << 4));
                        }
                    }
                }
            } else if (!TA) {
                const AT* src = Ap + row * p.lda + k0;
                if (p.vec && row_ok && k0 + 8 <= p.K) {  // 16-byte vectors
                    if constexpr (sizeof(AT) == 8) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const double2 x = __ldg(reinterpret_cast<const double2*>(src) + i);
                            v[2 * i] = x.x;
                            v[2 * i + 1] = x.y;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            const float4 x = __ldg(reinterpret_cast<const float4*>(src) + i);
                            v[4 * i] = x.x;
                            v[4 * i + 1] = x.y;
                            v[4 * i + 2] = x.z;
                            v[4 * i + 3] = x.w;
                        }
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = (row_ok && k0 + i < p.K) ? (double)__ldg(src + i) : 0.0;
                }
            } else {
                const AT* src = Ap + k0 * p.lda + row;
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = (row_ok && k0 + i < p.K) ? (double)__ldg(src + (int64_t)i * p.lda) : 0.0;
            }
            uint32_t words[kOzSlices][2];
#pragma unroll
            for (int q4 = 0; q4 < 2; ++q4) {
                double vs[4];
                uint32_t w[kOzSlices];
#pragma unroll
                for (int i = 0; i < 4; ++i) vs[i] = v[4 * q4 + i] * sr;
                oz_digit_words(vs, w);
#pragma unroll
                for (int t = 0; t < kOzSlices; ++t) words[t][q4] = w[t];
            }
            if (TMA_A && !(p.dbg & 2)) {
                // the staged values have been consumed (the digits depend on every load), so
                // the slot can be refilled: an arrive right after the loads could let the TMA
                // overwrite a value a lane's load had not yet returned
                __syncwarp();
                if (lane == 0) oz_arrive(a_empty(kt % kOzAStages));
            }
            mbar_wait(empty(s), ph ^ 1u);
            uint8_t* ap = gbase + (size_t)s * kOzStage + a_off;
            if (!(p.dbg & 4)) {
#pragma unroll
                for (int t = 0; t < kOzSlices; ++t)
                    *reinterpret_cast<uint2*>(ap + t * kOzAPlane) = make_uint2(words[t][0], words[t][1]);
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) oz_arrive(full_a(s));
            if ((kt % kOzChunkSteps) == kOzChunkSteps - 1 || kt == KT - 1) {
                // drain the 8 int32 levels of this thread's row x 16 columns, small levels
                // first, into the output row (written by the first chunk, added by the others)
                mbar_wait(drain_full, (uint32_t)chunk & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                double part[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) part[c] = 0.0;
#pragma unroll 1
                for (int L = kOzLevel0; L < kOzLevel0 + kOzLevels; ++L) {
                    uint32_t d[16];
                    const uint32_t taddr = t_row + (uint32_t)((L - kOzLevel0) * kOzBN);
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
                          "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]),
                          "=r"(d[14]), "=r"(d[15])
                        : "r"(taddr));
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                    const double w = __longlong_as_double((long long)(1023 + 8 * L - 108) << 52);  // 2^(8L - 108)
#pragma unroll
                    for (int c = 0; c < 16; ++c) part[c] = fma((double)(int)d[c], w, part[c]);
                }
                if (kt < KT - 1) zero_levels();  // the next chunk starts from zero
                if (row_ok) {
                    double* crow = p.C + row * p.ldc;
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const int col = c0 + c;
                        if (col < p.N) {
                            const int f = p.xexp[col];
                            double out;
                            if (e_row == kOzNonFinite || f == kOzNonFinite) out = __longlong_as_double(0x7ff8000000000000ll);
                            else out = scalbn(part[c], e_row + f);
                            crow[col] = (chunk == 0 && !p.acc0) ? out : crow[col] + out;
                        }
                    }
                }
                ++chunk;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

}  // namespace sorsvd_dev
