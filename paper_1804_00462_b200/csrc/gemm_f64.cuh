// K1/K2/K4/K6: FP64 skinny-GEMM engine on the sm_100a DMMA pipe.
//
// Every product on the SOR-SVD path (sketch.hpp:95,96,100-102,105,107 ->
// cblas_dgemm, dense.hpp:30) has one huge dimension (m or n of A), one huge
// reduction or output dimension, and one narrow dimension (k <= 256). This
// kernel computes
//     C[M x N] = alpha * op(A)[M x K] * B[K x N]
// with op(A) = A (A row-major M x K, "NN": T1 = A*Omega, Y = A*Q2, U = Q1*Ut)
//   or op(A) = A^T (A stored K x M row-major, "TN": T2 = A^T*T1, M = Q1^T*Y),
// B row-major with its columns zero-padded to a multiple of 8 (N chunks of
// up to 128 columns per CTA, grid.y), and split-K over grid.z with
// deterministic partial buffers reduced by reduce_splits_kernel.
//
// Tiles: 8 warps along M, each owning an (8*FM) x (8*FN) accumulator block of
// m8n8k4 DMMA fragments (FP64 tensor core, 37 TFLOP/s measured on B200);
// A and B tiles are staged through a 4-stage cp.async (LDGSTS) ring in shared
// memory with +4-double row padding so every fragment read is bank-conflict
// free. A is streamed exactly once per pass (the dominant HBM traffic).
//
// A may also be FP32 (AT = float: Config 3/5 inputs stored in single
// precision): the tile is staged as floats (half the HBM bytes) and widened
// to FP64 when the fragments are read, so the arithmetic is the same FP64
// DMMA as for double inputs (the power iteration needs it: see DESIGN.md,
// "FP32 inputs").
#pragma once
#include "common.cuh"

namespace sorsvd_dev {

struct GemmArgs {
    const void* A;  // double, or float for the FP32-storage kernels
    int64_t lda;
    const double* B;
    int64_t ldb;
    int64_t b_seg_stride;  // segmented GEMM: B for segment s is B + s*b_seg_stride
    double* C;
    int64_t ldc;
    int64_t c_split_stride;  // split z writes C + z*c_split_stride
    int64_t M;
    int64_t K;
    int64_t k_chunk;        // K range per split (multiple of BK)
    const int* tile_row0;   // optional explicit M-tile table (segmented GEMM)
    const int* tile_rows;
    const int* tile_seg;
    double alpha;
    const int* pred;  // optional device flag: the launch is a no-op when *pred == pred_skip
    int pred_skip;
    // stream-K (grid underfilled by whole tiles, or a partial last wave): CTA c runs
    // segments [sk_cta_seg[c], sk_cta_seg[c+1]) of the (tile, k-range) list; a segment
    // covering a whole tile writes C directly, partial ones go to workspace slot
    // sk_seg_slot[g] of `sk_ws` (BM x BN each) and streamk_fixup_kernel sums them in
    // slot order
    const int* sk_cta_seg;
    const int* sk_seg_tile;
    const int* sk_seg_k0;  // in BK units
    const int* sk_seg_k1;
    const int* sk_seg_slot;  // workspace slot of a partial segment (-1: whole tile, written to C)
    int sk_units;            // BK units per tile
    int sk_gy;             // column chunks per row tile
    double* sk_ws;
    int gy_fused;          // > 0: blockIdx.x = row_tile * gy_fused + column chunk (chunks of a row tile
                           // run back to back, so A's tile is served from L2 the second time)
};

constexpr int kGemmThreads = 256;
// K depth per smem stage and ring depth: the wide tiles (FM = 2, N up to 128)
// take BK = 32 with 3 stages (half the barriers per flop; <= 212 KB), the
// narrow-N tiles (FM = 4) BK = 16 with 4 stages.
__host__ __device__ constexpr int gemm_bk(int FM) { return FM >= 4 ? 16 : 32; }
__host__ __device__ constexpr int gemm_stages(int FM) { return FM >= 4 ? 4 : 3; }

template <int FM, int FN, bool TA, typename AT = double>
struct GemmShape {
    static constexpr int BM = 8 * 8 * FM;
    static constexpr int BN = 8 * FN;
    static constexpr int BK = gemm_bk(FM);
    static constexpr int STAGES = gemm_stages(FM);
    static constexpr int EPV = 16 / (int)sizeof(AT);  // A elements per 16-byte vector
    // padded smem strides: fragment reads conflict free (doubles: == 4 mod 8; floats: +4 / +8 words)
    static constexpr int LDA_S = TA ? (BM + (sizeof(AT) == 4 ? 8 : 4)) : (BK + 4);
    static constexpr int LDB_S = BN + 4;
    static constexpr int A_STAGE = TA ? BK * LDA_S : BM * LDA_S;  // elements of AT
    static constexpr int A_BYTES = ((A_STAGE * (int)sizeof(AT) + 15) / 16) * 16;
    static constexpr int B_STAGE = BK * LDB_S;
    static constexpr int STAGE_BYTES = A_BYTES + B_STAGE * 8;
    static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES;
};

// One output tile (rows [row0, row0+rows), columns [ncol0, ncol0+BN)) over the
// K range [kBegin, kEnd); the result goes to Cbase + (row_base + r) * ldc.
template <int FM, int FN, bool TA, bool V16, typename AT>
__device__ __forceinline__ void gemm_tile(const GemmArgs& p, unsigned char* smem_raw, int64_t row0, int64_t rows,
                                          int seg, int ncol0, int64_t kBegin, int64_t kEnd, double* Cbase,
                                          int64_t row_base, int64_t ldc) {
    using S = GemmShape<FM, FN, TA, AT>;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const double* __restrict__ Bp = p.B + seg * p.b_seg_stride + ncol0;
    const AT* __restrict__ Ap = static_cast<const AT*>(p.A);
    constexpr int EPV = S::EPV;
    const int KT = kEnd > kBegin ? (int)((kEnd - kBegin + S::BK - 1) / S::BK) : 0;

    auto a_stage = [&](int slot) { return reinterpret_cast<AT*>(smem_raw + (size_t)slot * S::STAGE_BYTES); };
    auto b_stage = [&](int slot) {
        return reinterpret_cast<double*>(smem_raw + (size_t)slot * S::STAGE_BYTES + S::A_BYTES);
    };
    // Interior stages (whole row tile, whole BK slab, 16-byte rows) take the
    // fast path: every thread's A chunks sit in one fixed column of the tile
    // (CPR chunks per tile row divides the 256 threads), so the global source
    // is a per-tile base plus a per-stage offset plus a constant stride, and
    // no bounds arithmetic is issued inside the DMMA loop's stage refill.
    constexpr int CPR = (TA ? S::BM : S::BK) / EPV;           // 16-byte chunks per smem tile row
    constexpr int RSTEP = kGemmThreads / CPR;                  // tile rows between a thread's chunks
    constexpr int NA = (TA ? S::BK : S::BM) / RSTEP;           // chunks per thread
    static_assert(kGemmThreads % CPR == 0 && (TA ? S::BK : S::BM) % RSTEP == 0, "A chunk map");
    const bool full_rows = V16 && rows == S::BM;
    const int ac = tid % CPR, ar0 = tid / CPR;
    const AT* __restrict__ abase =
        TA ? Ap + (int64_t)ar0 * p.lda + row0 + EPV * ac : Ap + (row0 + ar0) * p.lda + EPV * ac;
    const int64_t astride = (int64_t)RSTEP * p.lda;
    const int asoff = ar0 * S::LDA_S + EPV * ac;
    auto load_stage = [&](int slot, int kt) {
        AT* As = a_stage(slot);
        double* Bs = b_stage(slot);
        const int64_t k0 = kBegin + (int64_t)kt * S::BK;
        if (full_rows && k0 + S::BK <= kEnd) {
            const AT* src = abase + (TA ? k0 * p.lda : k0);
#pragma unroll
            for (int i = 0; i < NA; ++i) cp_async16(As + asoff + i * RSTEP * S::LDA_S, src + i * astride, 16);
            const double* bsrc = Bp + k0 * p.ldb;
#pragma unroll
            for (int i = 0; i < (S::BK * (S::BN / 2) + kGemmThreads - 1) / kGemmThreads; ++i) {
                const int id = tid + i * kGemmThreads;
                if (id < S::BK * (S::BN / 2)) {
                    const int kr = id / (S::BN / 2), c = id - kr * (S::BN / 2);
                    cp_async16(Bs + kr * S::LDB_S + 2 * c, bsrc + (int64_t)kr * p.ldb + 2 * c, 16);
                }
            }
            return;
        }
        if (!TA) {
            if (V16) {
                for (int id = tid; id < S::BM * (S::BK / EPV); id += kGemmThreads) {
                    const int r = id / (S::BK / EPV), c = id % (S::BK / EPV);
                    const int64_t kk = k0 + EPV * c;
                    int bytes = 0;
                    const AT* src = Ap;
                    if (r < rows && kk < kEnd) {
                        const int64_t rem = (kEnd - kk) * (int64_t)sizeof(AT);
                        bytes = rem >= 16 ? 16 : (int)rem;
                        src = Ap + (row0 + r) * p.lda + kk;
                    }
                    cp_async16(As + r * S::LDA_S + EPV * c, src, bytes);
                }
            } else {
                for (int id = tid; id < S::BM * S::BK; id += kGemmThreads) {
                    const int r = id / S::BK, c = id % S::BK;
                    const int64_t kk = k0 + c;
                    const bool ok = r < rows && kk < kEnd;
                    cp_async_elem(As + r * S::LDA_S + c, ok ? Ap + (row0 + r) * p.lda + kk : Ap, ok);
                }
            }
        } else {
            if (V16) {
                for (int id = tid; id < S::BK * (S::BM / EPV); id += kGemmThreads) {
                    const int kr = id / (S::BM / EPV), c = id % (S::BM / EPV);
                    const int64_t kk = k0 + kr;
                    int bytes = 0;
                    const AT* src = Ap;
                    if (kk < kEnd && EPV * c < rows) {
                        const int64_t rem = (rows - EPV * c) * (int64_t)sizeof(AT);
                        bytes = rem >= 16 ? 16 : (int)rem;
                        src = Ap + kk * p.lda + row0 + EPV * c;
                    }
                    cp_async16(As + kr * S::LDA_S + EPV * c, src, bytes);
                }
            } else {
                for (int id = tid; id < S::BK * S::BM; id += kGemmThreads) {
                    const int kr = id / S::BM, c = id % S::BM;
                    const int64_t kk = k0 + kr;
                    const bool ok = kk < kEnd && c < rows;
                    cp_async_elem(As + kr * S::LDA_S + c, ok ? Ap + kk * p.lda + row0 + c : Ap, ok);
                }
            }
        }
        for (int id = tid; id < S::BK * (S::BN / 2); id += kGemmThreads) {
            const int kr = id / (S::BN / 2), c = id % (S::BN / 2);
            const int64_t kk = k0 + kr;
            const bool ok = kk < kEnd;
            cp_async16(Bs + kr * S::LDB_S + 2 * c, ok ? Bp + kk * p.ldb + 2 * c : Bp, ok ? 16 : 0);
        }
    };

    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < S::STAGES - 1; ++s) {
        if (s < KT) load_stage(s, s);
        cp_async_commit();
    }
    const int wrow = warp * 8 * FM;
    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<S::STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + S::STAGES - 1;
            if (nk < KT) load_stage(nk % S::STAGES, nk);
            cp_async_commit();
        }
        const AT* As = a_stage(kt % S::STAGES);
        const double* Bs = b_stage(kt % S::STAGES);
#pragma unroll
        for (int ks = 0; ks < S::BK / 4; ++ks) {
            double a[FM], b[FN];
#pragma unroll
            for (int fm = 0; fm < FM; ++fm)
                a[fm] = (double)(TA ? As[(ks * 4 + t4) * S::LDA_S + wrow + fm * 8 + g]
                                    : As[(wrow + fm * 8 + g) * S::LDA_S + ks * 4 + t4]);
#pragma unroll
            for (int fn = 0; fn < FN; ++fn) b[fn] = Bs[(ks * 4 + t4) * S::LDB_S + fn * 8 + g];
#pragma unroll
            for (int fm = 0; fm < FM; ++fm)
#pragma unroll
                for (int fn = 0; fn < FN; ++fn) dmma884(acc[fm][fn][0], acc[fm][fn][1], a[fm], b[fn]);
        }
    }
    cp_async_wait<0>();
    __syncthreads();  // the smem ring may be reused by the next segment

#pragma unroll
    for (int fm = 0; fm < FM; ++fm) {
        const int r = wrow + fm * 8 + g;
        if (r < rows) {
            double* crow = Cbase + (row_base + r) * ldc + 2 * t4;
#pragma unroll
            for (int fn = 0; fn < FN; ++fn)
                *reinterpret_cast<double2*>(crow + fn * 8) =
                    make_double2(p.alpha * acc[fm][fn][0], p.alpha * acc[fm][fn][1]);
        }
    }
}


template <int FM, int FN, bool TA, bool V16, typename AT = double>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_f64_kernel(GemmArgs p) {
    using S = GemmShape<FM, FN, TA, AT>;
    if (pred_off(p.pred, p.pred_skip)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    if (p.sk_cta_seg) {  // stream-K
        const int g0 = p.sk_cta_seg[blockIdx.x], g1 = p.sk_cta_seg[blockIdx.x + 1];
        for (int gs = g0; gs < g1; ++gs) {
            const int tile = p.sk_seg_tile[gs];
            const int mt = tile / p.sk_gy, nt = tile - mt * p.sk_gy;
            const int64_t row0 = (int64_t)mt * S::BM;
            const int64_t rows = p.M - row0 < S::BM ? p.M - row0 : S::BM;
            const int ku0 = p.sk_seg_k0[gs], ku1 = p.sk_seg_k1[gs];
            const int64_t kBegin = (int64_t)ku0 * S::BK;
            const int64_t kEnd = min((int64_t)ku1 * S::BK, p.K);
            if (ku0 == 0 && ku1 == p.sk_units)  // whole tile: straight to C
                gemm_tile<FM, FN, TA, V16, AT>(p, smem_raw, row0, rows, 0, nt * S::BN, kBegin, kEnd,
                                               p.C + nt * S::BN, row0, p.ldc);
            else
                gemm_tile<FM, FN, TA, V16, AT>(p, smem_raw, row0, rows, 0, nt * S::BN, kBegin, kEnd,
                                               p.sk_ws + (size_t)p.sk_seg_slot[gs] * S::BM * S::BN, 0, S::BN);
        }
        return;
    }
    int64_t row0, rows;
    int seg = 0;
    if (p.tile_row0) {
        row0 = p.tile_row0[blockIdx.x];
        rows = p.tile_rows[blockIdx.x];
        seg = p.tile_seg[blockIdx.x];
    } else {
        const int mt = p.gy_fused > 0 ? (int)(blockIdx.x / p.gy_fused) : (int)blockIdx.x;
        row0 = (int64_t)mt * S::BM;
        rows = p.M - row0 < S::BM ? p.M - row0 : S::BM;
    }
    const int64_t kBegin = (int64_t)blockIdx.z * p.k_chunk;
    const int64_t kEnd = min(kBegin + p.k_chunk, p.K);
    const int ncol0 = (p.gy_fused > 0 ? (int)(blockIdx.x % p.gy_fused) : (int)blockIdx.y) * S::BN;
    gemm_tile<FM, FN, TA, V16, AT>(p, smem_raw, row0, rows, seg, ncol0, kBegin, kEnd,
                                   p.C + (int64_t)blockIdx.z * p.c_split_stride + ncol0, row0, p.ldc);
}

// Stream-K fix-up: every tile split over several segments gets the sum of
// its partial slots in slot order (deterministic: 0 + s_0 + s_1 + ...).
// grid.y = split tile, grid.x covers the tile's elements one per thread; the
// slot loads are issued 16 ahead of the ordered adds, since a tile split over
// ~100 segments (a K = m reduction onto one tile) is otherwise a chain of
// dependent L2 round trips.
__global__ void streamk_fixup_kernel(const double* __restrict__ ws, const int* __restrict__ split_slot0,
                                     const int* __restrict__ split_tiles, int nsplit, int BM, int BN, int gy,
                                     int64_t M, double* __restrict__ C, int64_t ldc, const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    const int per = BM * BN;  // one tile's elements (< 2^31)
    for (int st = blockIdx.y; st < nsplit; st += gridDim.y) {
        const int tile = split_tiles[st];
        const int mt = tile / gy, nt = tile - mt * gy;
        const int g0 = split_slot0[st], g1 = split_slot0[st + 1];  // the tile's partial slots, in order
        for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < per; w += gridDim.x * blockDim.x) {
            const int r = w / BN, col = w - r * BN;
            const int64_t row = (int64_t)mt * BM + r;
            if (row >= M) continue;
            const double* src = ws + (size_t)g0 * per + w;
            double acc = 0.0;
            int gs = g0;
            for (; gs + 16 <= g1; gs += 16, src += (size_t)16 * per) {
                double v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = __ldcg(src + (size_t)u * per);
#pragma unroll
                for (int u = 0; u < 16; ++u) acc += v[u];
            }
            for (; gs < g1; ++gs, src += per) acc += __ldcg(src);
            C[row * ldc + (int64_t)nt * BN + col] = acc;
        }
    }
}

// out[i] = sum_{s<S} ws[s*stride + i], fixed summation order (deterministic).
// The partial loads are issued 16 at a time ahead of the (ordered) adds: with
// many splits and few outputs (K = m reductions) the loop is L2-latency bound.
__global__ void reduce_splits_kernel(const double* __restrict__ ws, int64_t count2, int S, int64_t stride,
                                     double* __restrict__ out, const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    const int64_t n2 = count2;
    const double2* __restrict__ w2 = reinterpret_cast<const double2*>(ws);
    const int64_t st2 = stride / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
        double2 acc = w2[i];
        int s = 1;
        for (; s + 16 <= S; s += 16) {
            double2 v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = w2[(int64_t)(s + u) * st2 + i];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                acc.x += v[u].x;
                acc.y += v[u].y;
            }
        }
        for (; s < S; ++s) {
            const double2 v = w2[(int64_t)s * st2 + i];
            acc.x += v.x;
            acc.y += v.y;
        }
        reinterpret_cast<double2*>(out)[i] = acc;
    }
}

// Few outputs, many splits (Gram matrices of the CholeskyQR gates, the n x ell TN
// passes of C4): one warp per double2 output, lane l adds splits l, l+32, ... in
// order (independent loads across lanes, S/32 dependent L2 trips instead of S/16),
// then a fixed butterfly across the lanes. Deterministic for a given S.
__global__ void reduce_splits_warp_kernel(const double* __restrict__ ws, int64_t count2, int S, int64_t stride,
                                          double* __restrict__ out, const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    const int lane = threadIdx.x & 31;
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (i >= count2) return;
    const double2* __restrict__ w2 = reinterpret_cast<const double2*>(ws);
    const int64_t st2 = stride / 2;
    double2 acc = make_double2(0.0, 0.0);
    int s = lane;
    for (; s + 96 < S; s += 128) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = w2[(int64_t)(s + 32 * u) * st2 + i];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            acc.x += v[u].x;
            acc.y += v[u].y;
        }
    }
    for (; s < S; s += 32) {
        const double2 v = w2[(int64_t)s * st2 + i];
        acc.x += v.x;
        acc.y += v.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) reinterpret_cast<double2*>(out)[i] = acc;
}

}  // namespace sorsvd_dev
