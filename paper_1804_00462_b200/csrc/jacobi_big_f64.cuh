// K5 for 256 < k <= 512: one-sided Jacobi with the rotations logged.
//
// Same algorithm and output contract as jacobi_f64.cuh (Brent-Luk ring on a
// thread-block cluster, tol = sqrt(k) eps, descending sigma with index
// tie-break, largest-|u| sign canonicalisation; dense.hpp:65-110), re-laid
// out for the sizes where G and V together no longer fit a cluster's shared
// memory (k = 512: 2 x 2 MB):
//
//  * jacobi_big_kernel keeps only G on chip. A warp owns two adjacent pair
//    slots (4 columns, KP doubles per lane each, all in registers); of its 4
//    columns only one top and one bottom column leave the warp per round, so
//    the ring shift is mostly register renaming and only 2 columns per warp
//    cross shared memory / DSMEM: st.async into the neighbour's
//    double-buffered mailbox, completion tracked by the neighbour's mbarrier
//    (no cluster-wide barrier inside a sweep). The ring shift itself is free:
//    the loop body exists in two copies with the register arrays' roles
//    swapped. Each rotation's tangent t is appended to a log (round-major,
//    one double per slot; t = 0 when the pair was skipped).
//  * jb_vrec_kernel rebuilds V = J_1 J_2 ... J_R row by row: the rows of V
//    are independent, so every SM replays the log on its own block of rows
//    of the identity (c and s are recomputed from t bit-identically to the
//    forward kernel). V's columns are kept in ring order (position y of the
//    2P-1 moving columns, plus the fixed one), so a slot's two columns at
//    round t are (s-1-t) and (2P-2-s-t) mod 2P-1: no per-round table.
//  * jb_sigma_kernel / jb_rank_kernel finish U, sigma and the permutation.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace sorsvd_dev {

namespace cgb = cooperative_groups;

constexpr int kJbWarps = 8;  // warps per CTA; 2 pair slots per warp

struct JacobiBigArgs {
    const double* M;  // k x ldm row-major
    int ldm;
    int k;
    int kk;           // k rounded up to a multiple of 4 (P = kk/2 pair slots, even)
    double* Gout;     // final G, column id c at Gout + c*kk (kk rows, zero padded)
    double* tlog;     // [round][P] tangents
    int max_sweeps;
    int* info;        // [0] sweeps, [1] rounds
    const int* pred;  // optional predication (see JacobiArgs)
    int pred_skip;
};

// Column id held by ring position (slot, h) after `t_mod` shifts (t mod (2P-1)).
__device__ __forceinline__ int jb_origin(int slot, int h, int t_mod, int P) {
    const int L = 2 * P - 1;
    const int x = h == 0 ? slot - 1 : 2 * P - 2 - slot;
    if (x < 0) return 0;  // top of slot 0 never moves: column 0
    int y = x - t_mod;
    if (y < 0) y += L;
    return y < P - 1 ? 2 * (y + 1) : 2 * (2 * P - 2 - y) + 1;
}

__device__ __forceinline__ uint32_t jb_mapa(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
template <int OFF>
__device__ __forceinline__ void jb_st_async(uint32_t addr, double x, double y, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0+%4], {%1, %2}, [%3];\n" ::"r"(addr),
                 "d"(x), "d"(y), "r"(bar), "n"(OFF)
                 : "memory");
}
__device__ __forceinline__ void jb_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void jb_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "JB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra JB_WAIT;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void jb_bulk_send(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        "cp.async.bulk.commit_group;\n" ::"r"(dst),
        "r"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void jb_bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

constexpr int kJbMaxSweeps = 40;

template <int Q, int KP>
__device__ __forceinline__ void jb_send(uint32_t base, const double (&x)[KP], uint32_t bar) {
    if constexpr (Q < KP / 2) {  // 16-byte stores (each st.async carries its own complete_tx)
        jb_st_async<512 * Q>(base, x[2 * Q], x[2 * Q + 1], bar);
        jb_send<Q + 1, KP>(base, x, bar);
    }
}

// Per-warp constants of the ring (mailbox and mbarrier addresses per parity).
struct JbWarp {
    uint32_t sendT[2], barT[2];  // right neighbour's inT mailbox / mbarrier (+16*lane folded in)
    uint32_t sendB[2], barB[2];  // left neighbour's inB mailbox / mbarrier
    uint32_t mybar[2];
    const double* in[2];         // own mailbox for parity 0/1 (+2*lane folded in)
    uint32_t in_bytes;
    bool has_l, has_r;
    int kind;                    // 0 interior, 1 first warp, 2 last warp
    int slot0;                   // first pair slot of this warp
    double tol2;
    double* outT;                // local staging for the outgoing top / bottom column (+2*lane)
    double* outB;
    uint32_t outT_s, outB_s;     // their shared-window addresses (no lane offset)
    uint32_t col_bytes;
};

// Stage a column in the warp's local outbox and ship it with one bulk
// shared::cta -> shared::cluster copy that signals the receiver's mbarrier.
template <int KP>
__device__ __forceinline__ void jb_ship(const double (&x)[KP], double* out, uint32_t out_s, uint32_t dst,
                                        uint32_t bar, uint32_t bytes, int lane) {
#pragma unroll
    for (int q = 0; q < KP / 2; ++q) *reinterpret_cast<double2*>(out + 64 * q) = make_double2(x[2 * q], x[2 * q + 1]);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) jb_bulk_send(dst, out_s, bytes, bar);
}

// One ring round on the arrays in their current roles. On return the arrays
// hold the next round's columns in the SWAPPED roles (T0<->T1, B0<->B1), so
// the caller alternates jb_round(T0,T1,B0,B1) / jb_round(T1,T0,B1,B0).
template <int KP, int PAR>
__device__ __forceinline__ void jb_round(double (&T0)[KP], double (&T1)[KP], double (&B0)[KP], double (&B1)[KP],
                                         const JbWarp& w, double* tlog_round, int lane, int& rotated) {
    if (lane == 0 && w.in_bytes) jb_expect(w.mybar[PAR], w.in_bytes);
    double al0 = 0.0, be0 = 0.0, ga0 = 0.0, al1 = 0.0, be1 = 0.0, ga1 = 0.0;
#pragma unroll
    for (int p = 0; p < KP; ++p) {
        al0 = fma(T0[p], T0[p], al0);
        be0 = fma(B0[p], B0[p], be0);
        ga0 = fma(T0[p], B0[p], ga0);
        al1 = fma(T1[p], T1[p], al1);
        be1 = fma(B1[p], B1[p], be1);
        ga1 = fma(T1[p], B1[p], ga1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        al0 += __shfl_xor_sync(0xffffffffu, al0, o);
        be0 += __shfl_xor_sync(0xffffffffu, be0, o);
        ga0 += __shfl_xor_sync(0xffffffffu, ga0, o);
        al1 += __shfl_xor_sync(0xffffffffu, al1, o);
        be1 += __shfl_xor_sync(0xffffffffu, be1, o);
        ga1 += __shfl_xor_sync(0xffffffffu, ga1, o);
    }
    double t0 = 0.0, t1 = 0.0;
    if (ga0 != 0.0 && ga0 * ga0 > w.tol2 * al0 * be0) {
        const double d = be0 - al0;
        t0 = (2.0 * ga0 * (d < 0.0 ? -1.0 : 1.0)) / (fabs(d) + sqrt(fma(d, d, 4.0 * ga0 * ga0)));
    }
    if (ga1 != 0.0 && ga1 * ga1 > w.tol2 * al1 * be1) {
        const double d = be1 - al1;
        t1 = (2.0 * ga1 * (d < 0.0 ? -1.0 : 1.0)) / (fabs(d) + sqrt(fma(d, d, 4.0 * ga1 * ga1)));
    }
    if (t0 != 0.0) {
        rotated = 1;
        const double c = rsqrt(fma(t0, t0, 1.0)), sn = c * t0;
#pragma unroll
        for (int p = 0; p < KP; ++p) {
            const double x = T0[p], y = B0[p];
            T0[p] = c * x - sn * y;
            B0[p] = sn * x + c * y;
        }
    }
    if (t1 != 0.0) {
        rotated = 1;
        const double c = rsqrt(fma(t1, t1, 1.0)), sn = c * t1;
#pragma unroll
        for (int p = 0; p < KP; ++p) {
            const double x = T1[p], y = B1[p];
            T1[p] = c * x - sn * y;
            B1[p] = sn * x + c * y;
        }
    }
    if (lane < 2) tlog_round[w.slot0 + lane] = lane ? t1 : t0;
    // ring shift: top[i] -> top[i+1], bot[i] -> bot[i-1]; top[0] fixed,
    // top[P-1] -> bot[P-1], bot[0] -> top[1] (same ring as jacobi_cluster_kernel)
    // the previous round's bulk copies must have finished reading the outbox
    if (lane == 0) jb_bulk_wait_read();
    __syncwarp();
    if (w.has_r) jb_ship<KP>(T1, w.outT, w.outT_s, w.sendT[PAR], w.barT[PAR], w.col_bytes, lane);
    if (w.has_l) jb_ship<KP>(B0, w.outB, w.outB_s, w.sendB[PAR], w.barB[PAR], w.col_bytes, lane);
    // next roles: T0' = T1 array, T1' = T0 array, B0' = B1 array, B1' = B0 array
    if (w.kind == 1) {  // T0 fixed, T1' = old B0, B1' = incoming
#pragma unroll
        for (int p = 0; p < KP; ++p) {
            T1[p] = T0[p];
            T0[p] = B0[p];
        }
    } else if (w.kind == 2) {  // B1' = old T1, T0' = incoming
#pragma unroll
        for (int p = 0; p < KP; ++p) B0[p] = T1[p];
    }
}

template <int KP>
__device__ __forceinline__ void jb_recv(double (&dst)[KP], const double* src) {
#pragma unroll
    for (int q = 0; q < KP / 2; ++q) {
        dst[2 * q] = src[64 * q];
        dst[2 * q + 1] = src[64 * q + 1];
    }
}

// Lane `lane` holds column elements i = 64*(p/2) + 2*lane + (p%2), p < KP, so
// each lane's pairs are contiguous and a column moves as 16-byte st.async.
template <int KP>
__global__ void __launch_bounds__(kJbWarps * 32, 1) jacobi_big_kernel(JacobiBigArgs a) {
    if (pred_off(a.pred, a.pred_skip)) return;  // uniform over the cluster
    static_assert(KP % 2 == 0, "KP must be even");
    cgb::cluster_group cl = cgb::this_cluster();
    const int C = (int)cl.num_blocks();
    const int r = (int)cl.block_rank();
    const int k = a.k, kk = a.kk, P = kk / 2, W = P / 2;
    constexpr int KPAD = 32 * KP;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = r * kJbWarps + warp;
    const bool active = gw < W;
    extern __shared__ __align__(128) double mb[];  // [2 parity][kJbWarps][2: inT, inB][KPAD], then outbox [kJbWarps][2][KPAD]
    __shared__ __align__(8) uint64_t bar[2][kJbWarps];
    __shared__ int flags[kJbMaxSweeps];
    double* outbox = mb + (size_t)2 * kJbWarps * 2 * KPAD;

    auto elem = [&](int p) { return 64 * (p >> 1) + 2 * lane + (p & 1); };
    double X0[KP], X1[KP], Y0[KP], Y1[KP];  // (T0, T1, B0, B1) in even rounds, (T1, T0, B1, B0) in odd
    {
        const int s0 = 2 * gw, s1 = 2 * gw + 1;
        const int c00 = 2 * s0, c01 = 2 * s0 + 1, c10 = 2 * s1, c11 = 2 * s1 + 1;
#pragma unroll
        for (int p = 0; p < KP; ++p) {
            const int i = elem(p);
            const bool ri = active && i < k;
            const double* row = a.M + (size_t)(ri ? i : 0) * a.ldm;
            X0[p] = (ri && c00 < k) ? row[c00] : 0.0;
            Y0[p] = (ri && c01 < k) ? row[c01] : 0.0;
            X1[p] = (ri && c10 < k) ? row[c10] : 0.0;
            Y1[p] = (ri && c11 < k) ? row[c11] : 0.0;
        }
    }
    for (int i = threadIdx.x; i < kJbMaxSweeps; i += blockDim.x) flags[i] = 0;
    if (threadIdx.x < 2 * kJbWarps)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[0][0] + threadIdx.x)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    JbWarp w{};
    w.has_r = active && gw + 1 < W;
    w.has_l = active && gw > 0;
    w.kind = gw == 0 ? 1 : (gw == W - 1 ? 2 : 0);
    w.slot0 = 2 * gw;
    w.tol2 = (double)k * 2.220446049250313e-16 * 2.220446049250313e-16;  // tol = sqrt(k) eps
    for (int par = 0; par < 2; ++par) {
        w.mybar[par] = smem_u32(&bar[par][warp]);
        w.in[par] = mb + (size_t)(par * kJbWarps + warp) * 2 * KPAD + 2 * lane;
        if (w.has_r) {
            const int rw = (gw + 1) % kJbWarps, rc = (gw + 1) / kJbWarps;
            w.sendT[par] = jb_mapa(smem_u32(mb + ((size_t)(par * kJbWarps + rw) * 2 + 0) * KPAD), rc);
            w.barT[par] = jb_mapa(smem_u32(&bar[par][rw]), rc);
        }
        if (w.has_l) {
            const int lw = (gw - 1) % kJbWarps, lc = (gw - 1) / kJbWarps;
            w.sendB[par] = jb_mapa(smem_u32(mb + ((size_t)(par * kJbWarps + lw) * 2 + 1) * KPAD), lc);
            w.barB[par] = jb_mapa(smem_u32(&bar[par][lw]), lc);
        }
    }
    w.in_bytes = (uint32_t)((w.has_l ? 1 : 0) + (w.has_r ? 1 : 0)) * KPAD * 8;
    w.col_bytes = KPAD * 8;
    w.outT = outbox + (size_t)(warp * 2 + 0) * KPAD + 2 * lane;
    w.outB = outbox + (size_t)(warp * 2 + 1) * KPAD + 2 * lane;
    w.outT_s = smem_u32(outbox + (size_t)(warp * 2 + 0) * KPAD);
    w.outB_s = smem_u32(outbox + (size_t)(warp * 2 + 1) * KPAD);
    cl.sync();

    const int max_sweeps = a.max_sweeps < kJbMaxSweeps ? a.max_sweeps : kJbMaxSweeps;
    int sweep = 0, rounds = 0, rd = 0, rotated = 0;
    bool swapped = false;  // true when the current roles are (T0,T1,B0,B1) = (X1,X0,Y1,Y0)
    // end of a sweep: cluster-wide "anything rotated?"; returns true to stop
    auto end_sweep = [&]() {
        if (rotated && lane == 0) atomicOr(&flags[sweep], 1);
        cl.sync();
        int any = 0;
        for (int q = 0; q < C; ++q) any |= *cl.map_shared_rank(&flags[sweep], q);
        ++sweep;
        rotated = 0;
        rd = 0;
        return !any || sweep >= max_sweeps;
    };
    // the mbarrier of parity PAR completes once every two rounds: its n-th
    // phase (n = rounds/2) has parity n & 1
    for (;;) {
        if (active) {
            jb_round<KP, 0>(X0, X1, Y0, Y1, w, a.tlog + (size_t)rounds * P, lane, rotated);
            if (w.in_bytes) {
                jb_wait(w.mybar[0], (uint32_t)((rounds >> 1) & 1));
                if (w.has_l) jb_recv<KP>(X1, w.in[0]);
                if (w.has_r) jb_recv<KP>(Y0, w.in[0] + KPAD);
            }
        }
        ++rounds;
        swapped = true;
        if (++rd == kk - 1 && end_sweep()) break;
        if (active) {
            jb_round<KP, 1>(X1, X0, Y1, Y0, w, a.tlog + (size_t)rounds * P, lane, rotated);
            if (w.in_bytes) {
                jb_wait(w.mybar[1], (uint32_t)((rounds >> 1) & 1));
                if (w.has_l) jb_recv<KP>(X0, w.in[1]);
                if (w.has_r) jb_recv<KP>(Y1, w.in[1] + KPAD);
            }
        }
        ++rounds;
        swapped = false;
        if (++rd == kk - 1 && end_sweep()) break;
    }
    if (active) {
        const int tm = rounds % (2 * P - 1);
        const int s0 = 2 * gw, s1 = 2 * gw + 1;
        const int i0 = jb_origin(s0, 0, tm, P), i1 = jb_origin(s0, 1, tm, P), i2 = jb_origin(s1, 0, tm, P),
                  i3 = jb_origin(s1, 1, tm, P);
#pragma unroll
        for (int p = 0; p < KP; ++p) {
            const int i = elem(p);
            if (i < kk) {
                a.Gout[(size_t)i0 * kk + i] = swapped ? X1[p] : X0[p];
                a.Gout[(size_t)i1 * kk + i] = swapped ? Y1[p] : Y0[p];
                a.Gout[(size_t)i2 * kk + i] = swapped ? X0[p] : X1[p];
                a.Gout[(size_t)i3 * kk + i] = swapped ? Y0[p] : Y1[p];
            }
        }
    }
    if (r == 0 && threadIdx.x == 0) {
        a.info[0] = sweep;
        a.info[1] = rounds;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    // no CTA may exit while a peer can still read its flags
    cl.sync();
}

// sigma_c = ||G_c|| for every column id (one warp per column).
__global__ void jb_sigma_kernel(const double* __restrict__ G, int k, int kk, double* __restrict__ sig) {
    const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (c >= k) return;
    double ss = 0.0;
    for (int i = lane; i < k; i += 32) ss = fma(G[(size_t)c * kk + i], G[(size_t)c * kk + i], ss);
    ss = warp_sum(ss);
    if (lane == 0) sig[c] = sqrt(ss);
}

// Stable descending rank, sign canonicalisation (largest |u|, first index),
// U[:, rank] and S[rank]; perm / sgn for the V rebuild.
__global__ void jb_rank_kernel(const double* __restrict__ G, int k, int kk, const double* __restrict__ sig,
                               double* __restrict__ U, int ldu, double* __restrict__ S, int* __restrict__ perm,
                               double* __restrict__ sgn) {
    const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (c >= k) return;
    const double sv = sig[c];
    int rk = 0;
    for (int f = lane; f < k; f += 32) rk += (sig[f] > sv) || (sig[f] == sv && f < c);
    for (int o = 16; o > 0; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
    const double* Gc = G + (size_t)c * kk;
    double best = -1.0;
    int bi = 0;
    for (int i = lane; i < k; i += 32) {
        const double av = fabs(Gc[i]);
        if (av > best) {
            best = av;
            bi = i;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    const double sg = Gc[bi] < 0.0 ? -1.0 : 1.0;
    for (int i = lane; i < k; i += 32) U[(size_t)i * ldu + rk] = sv > 0.0 ? sg * Gc[i] / sv : 0.0;
    if (lane == 0) {
        S[rk] = sv;
        perm[c] = rk;
        sgn[c] = sg;
    }
}

constexpr int kJbRows = 4;   // rows of V per CTA in the rebuild
constexpr int kJbBatch = 8;  // log rounds per prefetch batch

// Storage index of column `id` in ring order: the fixed column 0 at L, the
// moving ones by their ring position y at round 0.
__device__ __forceinline__ int jb_idx_of(int id, int P) {
    const int L = 2 * P - 1;
    if (id == 0) return L;
    return (id & 1) ? 2 * P - 2 - (id - 1) / 2 : id / 2 - 1;
}

// V = J_1 ... J_R applied to rows of the identity; one thread per pair slot.
__global__ void __launch_bounds__(256) jb_vrec_kernel(const double* __restrict__ tlog, const int* __restrict__ info,
                                                      int k, int kk, const int* __restrict__ perm,
                                                      const double* __restrict__ sgn, double* __restrict__ V,
                                                      int ldv) {
    extern __shared__ __align__(16) double vr[];  // [kJbRows][kk], columns in ring order
    const int P = kk / 2, L = 2 * P - 1, s = threadIdx.x;
    const int row0 = blockIdx.x * kJbRows;
    for (int e = threadIdx.x; e < kJbRows * kk; e += blockDim.x) vr[e] = 0.0;
    __syncthreads();
    if (threadIdx.x < kJbRows && row0 + threadIdx.x < k)
        vr[threadIdx.x * kk + jb_idx_of(row0 + threadIdx.x, P)] = 1.0;
    __syncthreads();
    const int RT = info[1];
    const bool act = s < P;
    const int xt = s - 1, xb = 2 * P - 2 - s;  // ring positions of the slot's top / bottom
    double tv[kJbBatch], tn[kJbBatch];
#pragma unroll
    for (int u = 0; u < kJbBatch; ++u) tv[u] = (act && u < RT) ? tlog[(size_t)u * P + s] : 0.0;
    int tm = 0;
    for (int t0 = 0; t0 < RT; t0 += kJbBatch) {
#pragma unroll
        for (int u = 0; u < kJbBatch; ++u)
            tn[u] = (act && t0 + kJbBatch + u < RT) ? tlog[(size_t)(t0 + kJbBatch + u) * P + s] : 0.0;
#pragma unroll
        for (int u = 0; u < kJbBatch; ++u) {
            if (t0 + u >= RT) break;  // uniform
            const double t = tv[u];
            if (t != 0.0) {
                int ya = xt - tm, yb = xb - tm;
                ya = xt < 0 ? L : (ya < 0 ? ya + L : ya);
                yb = yb < 0 ? yb + L : yb;
                const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
#pragma unroll
                for (int rr = 0; rr < kJbRows; ++rr) {
                    double* v = vr + rr * kk;
                    const double x = v[ya], y = v[yb];
                    v[ya] = c * x - sn * y;
                    v[yb] = sn * x + c * y;
                }
            }
            tm = (tm + 1 == L) ? 0 : tm + 1;
            __syncthreads();
        }
#pragma unroll
        for (int u = 0; u < kJbBatch; ++u) tv[u] = tn[u];
    }
    for (int e = threadIdx.x; e < kJbRows * k; e += blockDim.x) {
        const int rr = e / k, id = e - rr * k;
        if (row0 + rr < k) V[(size_t)(row0 + rr) * ldv + perm[id]] = sgn[id] * vr[rr * kk + jb_idx_of(id, P)];
    }
}

}  // namespace sorsvd_dev
