// K1/K2/K4 on the INT8 tensor cores, second engine: the digit planes of A are
// cut ONCE per call and every pass streams them straight into the MMAs.
//
// ozaki_i8.cuh cuts A's FP64 tiles into int8 digit planes inside the pass
// kernel: every one of the 2q+3 passes (sketch.hpp:95, :96, :100-102 ->
// cblas_dgemm, dense.hpp:30) repeats that conversion, and the 4 column-chunk
// CTAs of a row tile each repeat it again (16 converter warps per CTA; the
// MMA pipe was ~46% active). Here the conversion is hoisted out of the passes:
//
//   * ozaki_rowplanes_kernel: one read of A (FP64 or FP32 storage) per call ->
//     the row exponents and 7 int8 planes P_t (m x n bytes each, row pitch padded to 16): row i is
//     scaled by 2^(54 - e_i) (e_i the exponent bound of its largest |entry|),
//     rounded to a 55-bit integer and split into balanced base-256 digits
//     exactly as ozaki_i8.cuh does. 7/8 of A's FP64 bytes, kept for the call.
//   * ONE representation serves both orientations. NN (T1 = A X): the row
//     scale 2^(e_i - 54) multiplies the output row. TN (T2 = A^T T1): the row
//     scale rides on the right operand instead, Z_ic = 2^(e_i) T1_ic, cut per
//     column like every other right operand; the left "rows" (columns of A)
//     then need no scale of their own. The TN representation error is 2^-55 of
//     each ROW's maximum (not each column's): the same normwise bound,
//     |err| <= K 2^-55 max|a| max|z|.
//   * ozaki_planes_gemm_kernel (one CTA per SM, 384 threads, a 128 x 64 output
//     tile like ozaki_i8.cuh): warp 0 streams, per 32-deep K step, the 7 planes
//     of the tile with ONE 3-D TMA box (NN: {32 K, 128 rows, 7} with the 32-byte
//     swizzle = K-major operand; TN: {128 columns, 32 K, 7} with the 128-byte
//     swizzle = MN-major operand, legal for kind::i8 from shared memory) plus
//     the X digit planes by bulk copy into a 5-stage ring; warp 1's elected lane
//     issues the same 11 stacked tcgen05.mma.kind::i8 per step (34 digit
//     products) into the 8 TMEM levels and frees the stage by tcgen05.commit;
//     warps 4-11 only drain TMEM every 16384 K. No converter warps, no A
//     re-conversion, A's HBM bytes per pass 7/8 of the FP64 matrix.
//   * split-K over grid.y for short grids (TN: n/128 x 4 tiles is 4.2 waves on
//     148 SMs): partial tiles summed in split order by reduce_splits_kernel.
#pragma once
#include <type_traits>

#include "ozaki_i8.cuh"

namespace sorsvd_dev {

constexpr int kOzpStages = 5;     // (A planes + X planes) ring: 5 x 43008 B
constexpr int kOzpThreads = 384;  // 4 control warps + 8 drain warps
#ifndef OZP_COLLECTOR
#define OZP_COLLECTOR 1
#endif
constexpr bool kOzpCollector = OZP_COLLECTOR != 0;  // A-collector reuse between the two MMAs of planes 3-6
#ifndef OZP_ISSUERS
#define OZP_ISSUERS 2
#endif
constexpr int kOzpIssuers = OZP_ISSUERS;  // MMA-issuing threads per CTA (1, 2 or 3; measured best: 2)
constexpr int kOzpMaxRegs = 96;   // 384 x 96 registers leave room for one 512-thread block of the conversion kernel
                                  // on the same SM (the first pass runs while the next row chunk is being cut)
constexpr size_t kOzpSmem = 1024 + (size_t)kOzpStages * kOzStage + 256;

struct OzpArgs {
    int64_t M;             // left rows of this launch: m (NN) or the column block's width (TN)
    int64_t K;             // n (NN) or m (TN)
    int mn0;               // first left row of this launch inside the planes (tensor-map coordinate): TN the
                           // column block's first column, NN the row block's first row
    const int* lexp;       // NN: exponent bounds of the left rows; TN: null (the row scales ride on X)
    const int8_t* Xd;      // digit planes of the right operand [K step][column chunk][slice][64 x 32 B]
    const int* xexp;       // per right column
    int NC, N;
    double* C;             // M x ldc (split s writes C + s * c_split_stride)
    int64_t ldc, c_split_stride;
    int kt_split;          // K steps per split (grid.y splits)
    int kt0;               // first K step of this launch inside the planes (a K range of the TN pass: rows [32 kt0, ..))
    int acc0;              // 1: add to C from the first drain on (an earlier launch wrote the preceding K range)
    int dbg;               // timing experiments (tools/oz_pass.py): 1 = no MMAs, 2 = no A-plane TMA
    const int* pred;
    int pred_skip;
};

// The same box delivered to the same shared-memory offset of every CTA in `mask` (cluster ranks),
// each destination's mbarrier (same offset) credited with the bytes.
__device__ __forceinline__ void tma_load_3d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y, int z,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%4, "
        "%5, %6}], [%2], %3;\n" ::"r"(dst),
        "l"(map), "r"(bar), "h"(mask), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(x), "r"(y), "r"(z)
        : "memory");
}

// A (m x n, FP64 or FP32 storage) -> row exponents e_i and the 7 digit planes,
// row-scaled by 2^(54 - e_i), in ONE read of A from HBM: G threads own a row
// (G = 512: the whole block, long rows; G = 32: a warp, short rows), first
// reduce max|a_ij| over it (bit patterns of |x| order like the values, NaN
// above Inf, so a non-finite entry wins the integer max), then re-read the
// row -- still in L1 / L2: at most 2 blocks x 148 SMs x one 160 KB row are in
// flight -- and cut it. A thread takes 4 consecutive values: 32 (16) bytes of
// loads, one 4-byte store per plane, a warp 128 contiguous bytes per plane.
template <typename AT, bool LAST = false>
__device__ __forceinline__ void oz_load4(const AT* __restrict__ src, int64_t col, int64_t n, int vec, double v[4]) {
    if (vec && col + 4 <= n) {
        if constexpr (sizeof(AT) == 8) {
            const double2* q = reinterpret_cast<const double2*>(src + col);
            const double2 x0 = LAST ? __ldcs(q) : __ldg(q);      // LAST: the row's second (final) read, evict first
            const double2 x1 = LAST ? __ldcs(q + 1) : __ldg(q + 1);
            v[0] = x0.x, v[1] = x0.y, v[2] = x1.x, v[3] = x1.y;
        } else {
            const float4* q = reinterpret_cast<const float4*>(src + col);
            const float4 x = LAST ? __ldcs(q) : __ldg(q);
            v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = col + i < n ? (double)__ldg(src + col + i) : 0.0;
    }
}

template <typename AT, int G, int THREADS = 512>
__global__ void __launch_bounds__(THREADS, 1024 / THREADS) ozaki_rowplanes_kernel(const AT* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                                                 int* __restrict__ row_e, int8_t* __restrict__ planes,
                                                                 int64_t pitch, int64_t plane_stride, int vec,
                                                                 const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    constexpr int RPB = THREADS / G;  // rows per block
    __shared__ unsigned long long sred[THREADS / 32];
    const int gi = threadIdx.x % G, gr = threadIdx.x / G;
    const int64_t ngroups = (n + 3) / 4;
    for (int64_t row0 = (int64_t)blockIdx.x * RPB; row0 < m; row0 += (int64_t)gridDim.x * RPB) {
        const int64_t row = row0 + gr;
        const bool ok = row < m;
        const AT* src = A + (ok ? row : 0) * lda;
        unsigned long long mx = 0ull;
        if (ok) {
#pragma unroll 8
            for (int64_t g = gi; g < ngroups; g += G) {
                double v[4];
                oz_load4(src, 4 * g, n, vec, v);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const unsigned long long b = (unsigned long long)__double_as_longlong(v[i]) & 0x7fffffffffffffffull;
                    mx = b > mx ? b : mx;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = x > mx ? x : mx;
        }
        if (G > 32) {
            if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = mx;
            __syncthreads();
#pragma unroll
            for (int w = 0; w < THREADS / 32; ++w) mx = sred[w] > mx ? sred[w] : mx;
        }
        // max < 2^e (frexp); the sentinel for NaN / Inf; 0 for an all-zero row (ozaki_exp_kernel)
        int e = 0;
        {
            const double vmax = __longlong_as_double((long long)mx);
            if (!isfinite(vmax)) e = kOzNonFinite;
            else if (vmax > 0.0) frexp(vmax, &e);
        }
        if (ok) {
            if (gi == 0) row_e[row] = e;
            const double s = oz_scale(e);
            int8_t* drow = planes + row * pitch;
#pragma unroll 4
            for (int64_t g = gi; g < ngroups; g += G) {
                double v[4];
                oz_load4<AT, true>(src, 4 * g, n, vec, v);
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = e == kOzNonFinite ? 0.0 : v[i] * s;
                uint32_t wd[kOzSlices];
                oz_digit_words(v, wd);
#pragma unroll
                for (int t = 0; t < kOzSlices; ++t)
                    __stcs(reinterpret_cast<uint32_t*>(drow + 4 * g + t * plane_stride), wd[t]);
            }
        }
        if (G > 32) __syncthreads();  // sred is reused by the next row
    }
}

// max_k |X_kn 2^(kexp_k)| per column (the TN right operand with A's row scales folded in); the
// block shape of ozaki_colmax_kernel.
__global__ void __launch_bounds__(256) ozaki_colmax_scaled_kernel(const double* __restrict__ X, int64_t ldx, int64_t K,
                                                                  int N, const int* __restrict__ kexp,
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
                if (k < K) {
                    const int e = kexp[k];
                    const double v =
                        e == kOzNonFinite ? __longlong_as_double(0x7ff8000000000000ll) : fabs(scalbn(X[k * ldx + n], e));
                    mv = oz_nanmax(mv, v);
                }
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

// ozaki_xdigits_kernel with the per-K-row factor 2^(kexp_k) applied first.
__global__ void ozaki_xdigits_scaled_kernel(const double* __restrict__ X, int64_t ldx, int64_t K, int N, int NC,
                                            const int* __restrict__ kexp, const int* __restrict__ xexp,
                                            int8_t* __restrict__ Xd) {
    const int64_t KT = (K + kOzBK - 1) / kOzBK;
    const int64_t total = KT * 2 * (int64_t)NC * kOzBN;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
        const int ncol = (int)(w % ((int64_t)NC * kOzBN));
        const int64_t kh = w / ((int64_t)NC * kOzBN);
        const int h = (int)(kh & 1);
        const int64_t kt = kh >> 1;
        const int nc = ncol / kOzBN, nl = ncol % kOzBN;
        const int f = ncol < N ? xexp[ncol] : 0;
        uint32_t words[kOzSlices][4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            double v[4];
            uint32_t wd[kOzSlices];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t k = kt * kOzBK + 16 * h + 4 * q4 + q;
                double x = 0.0;
                if (k < K && ncol < N && f != kOzNonFinite) {
                    const int e = kexp[k];
                    // 2^(e_k) x 2^(54 - f_c) in one exact scaling (no intermediate overflow)
                    x = e == kOzNonFinite ? 0.0 : scalbn(X[k * ldx + ncol], e + 54 - f);
                }
                v[q] = x;
            }
            oz_digit_words(v, wd);
#pragma unroll
            for (int t = 0; t < kOzSlices; ++t) words[t][q4] = wd[t];
        }
        int8_t* base = Xd + (kt * NC + nc) * (int64_t)kOzXStep + h * (kOzXStep / 2) + (nl / 8) * 128 + (nl % 8) * 16;
#pragma unroll
        for (int t = 0; t < kOzSlices; ++t)
            *reinterpret_cast<uint4*>(base + (int64_t)t * 1024) =
                make_uint4(words[t][0], words[t][1], words[t][2], words[t][3]);
    }
}

// MC = true: the NC column-chunk CTAs of a row tile form a thread-block cluster (cluster = NC <= 8
// CTAs along x). They need the SAME 7 A planes every K step, so cluster rank r loads planes r,
// r + NC, ... once (one-plane boxes) and multicasts them into every CTA's ring: the L2 -> SM traffic
// of A falls by NC. A stage is refilled when all NC CTAs' MMAs have retired it: each CTA's
// tcgen05.commit arrives on the empty barrier of every CTA in the cluster (multicast commit, count
// NC). Measured on B200 (m = 1e5 of C3): pass 11.67 -> 11.95 ms, the copy skeleton alone 7.84 ->
// 8.92 ms: NOT faster, so it is off by default (SORSVD_OPT_OZAKI_MULTICAST). The pass is bound by
// shared-memory bandwidth instead: per K step the MMAs read 44 KB of A planes and 68 KB of X planes
// (each X plane is an operand of up to 7 MMAs) while TMA writes 42 KB -- 154 KB against
// 128 B/clk x 1088 clk of MMA time.
template <bool TA, bool MC>
__global__ void __maxnreg__(kOzpMaxRegs)
    ozaki_planes_gemm_kernel(const __grid_constant__ CUtensorMap tmA, OzpArgs p) {
    if (pred_off(p.pred, p.pred_skip)) return;
    extern __shared__ __align__(1024) uint8_t smraw[];
    const uint32_t base = (smem_u32(smraw) + 1023u) & ~1023u;
    uint8_t* gbase = smraw + (base - smem_u32(smraw));
    const uint32_t bar0 = base + kOzpStages * kOzStage;
    auto full = [&](int s) { return bar0 + 8u * s; };
    auto empty = [&](int s) { return bar0 + 8u * (kOzpStages + s); };
    const uint32_t drain_full = bar0 + 8u * (2 * kOzpStages);
    const uint32_t drain_empty = drain_full + 8u;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (drain_empty + 8u - base));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x / p.NC, nc = blockIdx.x % p.NC;
    const int64_t m0 = (int64_t)mt * kOzBM;
    const int KT_all = (int)((p.K + kOzBK - 1) / kOzBK);
    const int kt_b = (int)blockIdx.y * p.kt_split;
    const int KT = (KT_all - kt_b < p.kt_split ? KT_all - kt_b : p.kt_split);  // >= 1 (host)

    const uint32_t crank = MC ? cluster_ctarank() : 0u;
    const uint32_t csize = MC ? (uint32_t)p.NC : 1u;
    const uint16_t cmask = (uint16_t)((1u << csize) - 1u);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kOzpStages; ++s) {
            mbar_init(full(s), 1);
            mbar_init(empty(s), kOzpIssuers * csize);  // one commit per issuing thread per CTA of the cluster
        }
        mbar_init(drain_full, kOzpIssuers);
        mbar_init(drain_empty, 8);  // one arrive per drain warp
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (MC) cluster_sync_all();  // every CTA's barriers are initialised before any multicast lands
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- producer: A planes (one 3-D TMA box) + X planes (bulk copy) per K step ----
            const int8_t* xsrc = p.Xd + (size_t)nc * kOzXStep;
            for (int i = 0; i < KT; ++i) {
                const int s = i % kOzpStages;
                const uint32_t ph = (uint32_t)(i / kOzpStages) & 1u;
                mbar_wait(empty(s), ph ^ 1u);
                mbar_expect_tx(full(s), (p.dbg & 2) ? (uint32_t)kOzXStep : (uint32_t)kOzStage);
                const uint32_t dst = base + s * kOzStage;
                const int kt = kt_b + i;
                if (p.dbg & 2) {
                } else if (MC) {  // this rank's planes, multicast to the whole cluster
                    for (int t = (int)crank; t < kOzSlices; t += (int)csize) {
                        if (!TA) tma_load_3d_mc(dst + t * kOzAPlane, &tmA, full(s), kt * kOzBK, p.mn0 + (int)m0, t, cmask);
                        else tma_load_3d_mc(dst + t * kOzAPlane, &tmA, full(s), p.mn0 + (int)m0, (p.kt0 + kt) * kOzBK, t, cmask);
                    }
                } else if (!TA) tma_load_3d(dst, &tmA, full(s), kt * kOzBK, p.mn0 + (int)m0, 0);
                else tma_load_3d(dst, &tmA, full(s), p.mn0 + (int)m0, (p.kt0 + kt) * kOzBK, 0);
                oz_bulk_g2s(dst + kOzSlices * kOzAPlane, xsrc + (size_t)kt * p.NC * kOzXStep, (uint32_t)kOzXStep, full(s));
            }
        }
    } else if (warp >= 1 && warp <= kOzpIssuers) {
        // ---- MMA issuers: kOzpIssuers threads (warps 1.., one lane each) share the 11 MMAs of a K step by A
        // plane (two: planes 6-4 / 3-0). The int32 levels are exact, so the order in which the streams of
        // MMAs land does not matter; one thread alone was close to issue-bound (a run-time branch in its
        // loop cost 16% of the pass; two threads: 24.8 -> 23.3 ms on C3; three: no better).
        const int who = warp - 1;
        if (lane == 0) {
            for (int i = 0; i < KT; ++i) {
                const int s = i % kOzpStages;
                const uint32_t ph = (uint32_t)(i / kOzpStages) & 1u;
                const int ck = i % kOzChunkSteps;
                if (ck == 0) mbar_wait(drain_empty, (uint32_t)(i / kOzChunkSteps) & 1u);  // TMEM zeroed
                mbar_wait(full(s), ph);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                const uint32_t a_s = base + s * kOzStage;
                const uint32_t x_s = a_s + kOzSlices * kOzAPlane;
                // COLL: 0 = plain; 1 = keep this A plane in the MMA's A collector (collector::a::fill); 2 = the
                // next MMA on the same plane takes it from there (collector::a::lastuse) instead of reading
                // its 4 KB from shared memory again (planes 3-6 are operands of two MMAs: N <= 256 each).
                // Compile-time: a run-time selector in this one-thread issue loop cost 16% of the pass.
                auto mma = [&](int t, int u0, int cnt, auto coll_tag) {
                    constexpr int COLL = decltype(coll_tag)::value;
                    // NN: K-major, 32-byte swizzle atoms (8 rows x 32 B), 8-row groups 256 B apart.
                    // TN: MN-major, 128-byte swizzle atoms (8 K rows x 128 columns), K groups 1024 B apart.
                    const uint64_t da = TA ? umma_desc(a_s + t * kOzAPlane, 4096, 1024, 2)
                                           : umma_desc(a_s + t * kOzAPlane, 0, 256, 6);
                    const uint64_t db = umma_desc(x_s + u0 * 1024, kOzXStep / 2, 128, 0);
                    const uint32_t idesc = i8_idesc(kOzBM, kOzBN * cnt) | (TA ? (1u << 15) : 0u);
                    const uint32_t d = tmem + (uint32_t)((t + u0 - kOzLevel0) * kOzBN);
                    if constexpr (COLL == 1)
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                            "l"(da), "l"(db), "r"(idesc));
                    else if constexpr (COLL == 2)
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::i8.collector::a::lastuse [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                            "l"(da), "l"(db), "r"(idesc));
                    else
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                            "l"(da), "l"(db), "r"(idesc));
                };
                using C0 = std::integral_constant<int, 0>;
                using C1 = std::integral_constant<int, kOzpCollector ? 1 : 0>;
                using C2 = std::integral_constant<int, kOzpCollector ? 2 : 0>;
                // all digit pairs with t + u >= 5, split over the issuing threads by A plane (straight-line
                // blocks: the loop-invariant choice is one branch per step)
                if (p.dbg & 1) {
                } else if constexpr (kOzLevel0 == 6) {  // the 28 pairs with t + u >= 6
                    if (kOzpIssuers == 1 || who == 0) {  // 13 products
                        mma(6, 0, 4, C1{}); mma(6, 4, 3, C2{});
                        mma(5, 1, 4, C1{}); mma(5, 5, 2, C2{});
                    }
                    if (kOzpIssuers == 1 || who == 1) {  // 15 products
                        mma(4, 2, 4, C1{}); mma(4, 6, 1, C2{});
                        mma(3, 3, 4, C0{});
                        mma(2, 4, 3, C0{});
                        mma(1, 5, 2, C0{});
                        mma(0, 6, 1, C0{});
                    }
                } else if constexpr (kOzpIssuers == 1) {
                    mma(6, 0, 4, C1{}); mma(6, 4, 3, C2{});
                    mma(5, 0, 4, C1{}); mma(5, 4, 3, C2{});
                    mma(4, 1, 4, C1{}); mma(4, 5, 2, C2{});
                    mma(3, 2, 4, C1{}); mma(3, 6, 1, C2{});
                    mma(2, 3, 4, C0{});
                    mma(1, 4, 3, C0{});
                    mma(0, 5, 2, C0{});
                } else if constexpr (kOzpIssuers == 2) {
                    if (who == 0) {  // 20 products
                        mma(6, 0, 4, C1{}); mma(6, 4, 3, C2{});
                        mma(5, 0, 4, C1{}); mma(5, 4, 3, C2{});
                        mma(4, 1, 4, C1{}); mma(4, 5, 2, C2{});
                    } else {         // 14 products
                        mma(3, 2, 4, C1{}); mma(3, 6, 1, C2{});
                        mma(2, 3, 4, C0{});
                        mma(1, 4, 3, C0{});
                        mma(0, 5, 2, C0{});
                    }
                } else {
                    if (who == 0) {
                        mma(6, 0, 4, C1{}); mma(6, 4, 3, C2{});
                        mma(5, 0, 4, C1{}); mma(5, 4, 3, C2{});
                    } else if (who == 1) {
                        mma(4, 1, 4, C1{}); mma(4, 5, 2, C2{});
                        mma(3, 2, 4, C1{}); mma(3, 6, 1, C2{});
                    } else {
                        mma(2, 3, 4, C0{});
                        mma(1, 4, 3, C0{});
                        mma(0, 5, 2, C0{});
                    }
                }
                if (MC)
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                            empty(s)),
                        "h"(cmask)
                        : "memory");
                else
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                     empty(s))
                                 : "memory");
                if (ck == kOzChunkSteps - 1 || i == KT - 1)
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(drain_full)
                        : "memory");
            }
        }
    } else if (warp >= 4) {
        // ---- drainers: thread = TMEM lane (tile row) x 32 of the 64 columns of every level ----
        const int q = warp & 3;          // TMEM lane quarter
        const int hc = (warp - 4) >> 2;  // column half
        const int r = 32 * q + lane;
        const int64_t row = m0 + r;
        const bool row_ok = row < p.M;
        const int e_row = (row_ok && p.lexp) ? p.lexp[row] : 0;
        const uint32_t t_row = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(32 * hc);
        auto zero_levels = [&]() {
#pragma unroll 1
            for (int L = 0; L < kOzLevels; ++L) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t ta = t_row + (uint32_t)(L * kOzBN + 16 * h);
                    asm volatile(
                        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(
                            ta),
                        "r"(0u)
                        : "memory");
                }
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            __syncwarp();
            if (lane == 0) oz_arrive(drain_empty);
        };
        zero_levels();
        double* crow = p.C + (int64_t)blockIdx.y * p.c_split_stride + row * p.ldc;
        const int chunks = (KT + kOzChunkSteps - 1) / kOzChunkSteps;
        for (int chunk = 0; chunk < chunks; ++chunk) {
            mbar_wait(drain_full, (uint32_t)chunk & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            double part[2][16];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 16; ++c) part[h][c] = 0.0;
#pragma unroll 1
            for (int L = kOzLevel0; L < kOzLevel0 + kOzLevels; ++L) {
                const double w = __longlong_as_double((long long)(1023 + 8 * L - 108) << 52);  // 2^(8L - 108)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t d[16];
                    const uint32_t taddr = t_row + (uint32_t)((L - kOzLevel0) * kOzBN + 16 * h);
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
                          "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]),
                          "=r"(d[14]), "=r"(d[15])
                        : "r"(taddr));
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                    for (int c = 0; c < 16; ++c) part[h][c] = fma((double)(int)d[c], w, part[h][c]);
                }
            }
            if (chunk < chunks - 1) zero_levels();  // the next chunk starts from zero
            if (row_ok) {
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const int col = nc * kOzBN + 32 * hc + 16 * h + c;
                        if (col < p.N) {
                            const int f = p.xexp[col];
                            double out;
                            if (e_row == kOzNonFinite || f == kOzNonFinite) out = __longlong_as_double(0x7ff8000000000000ll);
                            else out = scalbn(part[h][c], e_row + f);
                            crow[col] = (chunk == 0 && !p.acc0) ? out : crow[col] + out;
                        }
                    }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (MC) cluster_sync_all();  // no CTA leaves while a peer may still multicast into it / signal its barriers
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

// out = (acc ? out : 0) + sum of the S split partials, in split order (a K range of the TN pass added
// to the ranges before it).
__global__ void oz_reduce_acc_kernel(const double* __restrict__ ws, int64_t count, int S, int64_t stride,
                                     double* __restrict__ out, int acc, const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        double v = acc ? out[i] : 0.0;
        for (int sidx = 0; sidx < S; ++sidx) v += ws[(int64_t)sidx * stride + i];
        out[i] = v;
    }
}

}  // namespace sorsvd_dev
