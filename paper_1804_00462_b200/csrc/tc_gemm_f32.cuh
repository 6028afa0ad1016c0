// K1/K2 (FP32 A): the A-streaming passes on the 5th-generation tensor cores.
//
// For fp32 matrices (BASELINE configs 3-fp32 and 5) the passes T1 = A*X
// (sketch.hpp:95, NN) and T2 = A^T*T1 (sketch.hpp:96, TN) run as
// tcgen05.mma.kind::tf32 with FP32 accumulation in TMEM:
//   * warp 0 (one elected lane) streams A and X/T1 tiles with TMA
//     (cp.async.bulk.tensor, 128B swizzle) into a 4-stage shared-memory ring,
//     completion tracked by mbarrier transaction counts;
//   * warp 1 (one lane) issues tcgen05.mma (M = 128, N = BN <= 256, K = 8 per
//     instruction, 4 per 32-deep stage) and frees each stage with
//     tcgen05.commit -> mbarrier when its MMAs retire;
//   * warp 2 allocates / frees the TMEM accumulator (BN columns);
//   * warps 4-7 read the 128 x BN accumulator back with tcgen05.ld
//     (32x32b, one row per thread) and store FP32 rows.
// A is K-major for NN (rows of A contiguous in K) and MN-major for TN (the
// M index of A^T is contiguous); X / T1 are MN-major (N contiguous), both
// legal for kind::tf32. Split-K over grid.z writes partial tiles.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace sorsvd_dev {

constexpr int kTcBM = 128;
constexpr int kTcBK = 32;  // 128 bytes of fp32 = one 128B swizzle row
constexpr int kTcStages = 4;
constexpr int kTcThreads = 256;

template <int BN>
struct TcShape {
    static constexpr int A_BYTES = kTcBM * kTcBK * 4;  // 16 KB
    static constexpr int B_BYTES = kTcBK * BN * 4;     // BN/32 boxes of 4 KB
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    static constexpr size_t SMEM = 1024 /*align slack*/ + (size_t)kTcStages * STAGE + 256 /*barriers*/;
};

struct TcArgs {
    float* C;               // output rows (row-major, ldc) or split partials
    int64_t ldc;
    int64_t c_split_stride;
    int64_t M;              // rows of C
    int64_t K;
    int64_t k_chunk;        // K per split, multiple of kTcBK
    const int* pred;        // optional predication (see gemm_f64.cuh)
    int pred_skip;
};

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(x), "r"(y)
        : "memory");
}
// UMMA shared-memory descriptor. layout: 2 = SWIZZLE_128B (K-major fp32 rows of
// 128 B), 1 = SWIZZLE_128B_BASE32B (MN-major fp32: 32-byte swizzle atoms, the
// layout the TMA writes with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
    d |= (uint64_t)layout << 61;
    return d;
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, majors, N, M.
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

#ifdef TC_DEBUG
__device__ float* tc_dbg;
#endif

template <int BN, bool TA>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs p) {
    using S = TcShape<BN>;
    if (pred_off(p.pred, p.pred_skip)) return;
    extern __shared__ __align__(1024) uint8_t smraw[];
    const uint32_t base = (smem_u32(smraw) + 1023u) & ~1023u;
    uint8_t* gbase = smraw + (base - smem_u32(smraw));
    const uint32_t bar0 = base + kTcStages * S::STAGE;  // full[ST], empty[ST], done
    auto full = [&](int s) { return bar0 + 8u * s; };
    auto empty = [&](int s) { return bar0 + 8u * (kTcStages + s); };
    const uint32_t done = bar0 + 8u * (2 * kTcStages);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + kTcStages * S::STAGE + 8 * (2 * kTcStages + 1));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m0 = (int64_t)blockIdx.x * kTcBM;
    const int n0 = blockIdx.y * BN;
    const int64_t kb = (int64_t)blockIdx.z * p.k_chunk;
    int64_t ke = kb + p.k_chunk;
    if (ke > p.K) ke = p.K;
    const int KT = ke > kb ? (int)((ke - kb + kTcBK - 1) / kTcBK) : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(full(s), 1);
            mbar_init(empty(s), 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(S::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        for (int kt = 0; kt < KT; ++kt) {
            const int s = kt % kTcStages;
            const uint32_t ph = (uint32_t)(kt / kTcStages) & 1u;
            mbar_wait(empty(s), ph ^ 1u);
            mbar_expect_tx(full(s), (uint32_t)S::STAGE);
            const uint32_t a_dst = base + s * S::STAGE;
            const uint32_t b_dst = a_dst + S::A_BYTES;
            const int k0 = (int)(kb + (int64_t)kt * kTcBK);
            if (!TA) {
                tma_load_2d(a_dst, &tmA, full(s), k0, (int)m0);  // {K, M} box {32, 128}
            } else {
#pragma unroll
                for (int c = 0; c < kTcBM / 32; ++c)  // {M, K} boxes {32, 32}
                    tma_load_2d(a_dst + c * 4096, &tmA, full(s), (int)m0 + 32 * c, k0);
            }
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) tma_load_2d(b_dst + c * 4096, &tmB, full(s), n0 + 32 * c, k0);
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = tf32_idesc(kTcBM, BN, TA ? 1 : 0, 1);
        for (int kt = 0; kt < KT; ++kt) {
            const int s = kt % kTcStages;
            const uint32_t ph = (uint32_t)(kt / kTcStages) & 1u;
            mbar_wait(full(s), ph);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const uint32_t a_s = base + s * S::STAGE;
            const uint32_t b_s = a_s + S::A_BYTES;
#ifdef TC_DEBUG
            if (kt == 0 && tc_dbg) {
                const float* af = reinterpret_cast<const float*>(gbase + s * S::STAGE);
                for (int q = 0; q < 8; ++q) tc_dbg[2 + q] = af[q];
                for (int q = 0; q < 8; ++q) tc_dbg[10 + q] = af[S::A_BYTES / 4 + q];
                tc_dbg[0] = (float)tmem;
                tc_dbg[1] = (float)a_s;
            }
#endif
#pragma unroll
            for (int kk = 0; kk < kTcBK / 8; ++kk) {
                // A: K-major -> advance 32 B inside the 128 B swizzle row; MN-major -> next 8-row K group
                // MN-major: 32-element (128 B) MN atoms every 4 KB (LBO), 4-row K atoms every 512 B (SBO)
                const uint64_t da = TA ? umma_desc(a_s + kk * 1024, 4096, 512, 1) : umma_desc(a_s + kk * 32, 0, 1024, 2);
                const uint64_t db = umma_desc(b_s + kk * 1024, 4096, 512, 1);
                const uint32_t acc = (kt | kk) ? 1u : 0u;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             empty(s))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(done)
                     : "memory");
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> global ----------------
        const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
        const int64_t row = m0 + 32 * quarter + lane;
        float* crow = p.C + (int64_t)blockIdx.z * p.c_split_stride + row * p.ldc + n0;
        if (KT > 0) {
            mbar_wait(done, 0);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
        }
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            if (KT > 0) {
                const uint32_t taddr = tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(32 * c);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                      "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                      "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
                      "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                      "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            } else {
#pragma unroll
                for (int q = 0; q < 32; ++q) r[q] = 0u;
            }
            if (row < p.M) {
                float4* dst = reinterpret_cast<float4*>(crow + 32 * c);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                         __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(S::TMEM_COLS));
    }
}

// out[i] = sum_s ws[s*stride + i] (fp32 partials, fixed order).
__global__ void reduce_splits_f32_kernel(const float* __restrict__ ws, int64_t count4, int S, int64_t stride,
                                         float* __restrict__ out, const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 acc = reinterpret_cast<const float4*>(ws)[i];
        for (int s = 1; s < S; ++s) {
            const float4 v = reinterpret_cast<const float4*>(ws + s * stride)[i];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        reinterpret_cast<float4*>(out)[i] = acc;
    }
}

// Precision conversions between the FP32 passes and the FP64 QR / SVD stages.
__global__ void cast_f32_to_f64_kernel(const float* __restrict__ in, int64_t ldi, double* __restrict__ out,
                                       int64_t ldo, int64_t rows, int cols) {
    const int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / cols, j = e - i * cols;
        out[i * ldo + j] = (double)in[i * ldi + j];
    }
}
__global__ void cast_f64_to_f32_kernel(const double* __restrict__ in, int64_t ldi, float* __restrict__ out,
                                       int64_t ldo, int64_t rows, int cols) {
    const int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / cols, j = e - i * cols;
        out[i * ldo + j] = (float)in[i * ldi + j];
    }
}

}  // namespace sorsvd_dev
