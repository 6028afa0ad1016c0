// K5: small dense SVD of the k x k core M by one-sided (Hestenes) Jacobi.
//
// Replaces truncated_svd(M, k) -> full_svd -> LAPACKE_dgesdd('S')
// (sketch.hpp:103, dense.hpp:65-110). Output contract is the reference's:
// sigma nonincreasing (ties by column index), U and V orthonormal, each
// column of U canonicalised so its largest-magnitude entry is positive
// (dense.hpp:80-95: first maximal index wins), V flipped with it.
//
// Parallel layout (Brent-Luk ring ordering on a thread-block cluster): the
// columns of G = M (and of the accumulated rotation V) sit in P = ceil(k/2)
// pair slots; one warp owns one slot and holds its two columns of G and V in
// registers for the round. Each round every warp computes alpha, beta, gamma
// with warp shuffles, rotates its pair, and writes the two columns to their
// next slots of the ring (top[i] -> top[i+1], bot[i] -> bot[i-1], with the
// ends wrapping), so only the columns at CTA boundaries travel over DSMEM.
// Double-buffered slots make one cluster barrier per round sufficient. A
// sweep is kk-1 rounds (kk = k rounded up to even, the extra column is a
// zero dummy); sweeps stop when no pair exceeded |g_p.g_q| > tol ||g_p|| ||g_q||
// with tol = sqrt(k) eps (the dgesvj criterion; high relative accuracy).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace sorsvd_dev {

namespace cgj = cooperative_groups;

struct JacobiArgs {
    const double* M;  // k x ldm row-major
    int ldm;
    int k;
    double* U;        // k x ldu row-major (first k columns written)
    int ldu;
    double* S;        // k
    double* V;        // k x ldv row-major
    int ldv;
    int ppc;          // pair slots (= warps) per CTA
    int max_sweeps;
    int* sweeps_out;  // optional
    const int* pred;  // optional: no-op when pred_off(pred, pred_skip) (RPCA iteration after convergence)
    int pred_skip;
};

// smem per CTA (doubles): 2 buffers x ppc slots x 2 columns x (G, V) x kpad
//   + ids (2 x ppc x 2 ints, as doubles) + sigma/rank scratch
// Column length held per ring slot: 32 * KP, KP = the kernel's per-lane element count
// (1, 2, 4, 8 by k, as run_jacobi selects it). Every lane reads KP elements per column,
// so the slot must span all 32 * KP of them (zero padded past k).
__host__ __device__ inline int jac_kpad(int k) {
    const int kp = (k + 31) / 32;
    return 32 * (kp <= 1 ? 1 : kp <= 2 ? 2 : kp <= 4 ? 4 : 8);
}
__host__ __device__ inline size_t jacobi_smem_bytes(int k, int ppc) {
    const size_t slot = 4 * (size_t)jac_kpad(k);
    return (2 * (size_t)ppc * slot + 2 * 2 * (size_t)ppc + 4 * (size_t)ppc + 64) * sizeof(double);
}


// Jacobi rotation of a column pair from its Gram entries al = |p|^2, be = |q|^2,
// ga = p.q: tan = 2 ga sgn(d) / (|d| + sqrt(d^2 + 4 ga^2)), d = be - al (the smaller
// angle). Computed from two reciprocal square roots (cos 2th = |d| r1,
// c = sqrt((1 + cos 2th) / 2), s = ga sgn(d) r1 / c) instead of a division, a square
// root and a reciprocal square root in sequence: a shorter FP64 dependency chain on
// the critical path of every ring round.
__device__ __forceinline__ void jac_rotation(double al, double be, double ga, double& c, double& sn) {
    const double d = be - al;
    const double r1 = rsqrt(fma(d, d, 4.0 * ga * ga));
    const double x = fma(0.5 * fabs(d), r1, 0.5);
    const double r2 = rsqrt(x);
    c = x * r2;
    sn = (d < 0.0 ? -ga : ga) * r1 * r2;
}

template <int KP>
__global__ void jacobi_cluster_kernel(JacobiArgs a) {
    if (pred_off(a.pred, a.pred_skip)) return;  // uniform over the cluster
    cgj::cluster_group cl = cgj::this_cluster();
    const int C = (int)cl.num_blocks();
    const int r = (int)cl.block_rank();
    const int k = a.k, ppc = a.ppc;
    const int kk = (k + 1) & ~1;
    const int P = kk / 2;
    constexpr int KPAD = 32 * KP;  // == jac_kpad(k) for the KP run_jacobi picks
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = r * ppc + warp;  // global pair slot of this warp
    const bool active = warp < ppc && slot < P;

    extern __shared__ __align__(16) double sm[];
    const size_t SLOT = 4 * (size_t)KPAD;  // [top G | top V | bot G | bot V]
    double* buf0 = sm;
    double* buf1 = sm + (size_t)ppc * SLOT;
    int* ids = reinterpret_cast<int*>(sm + 2 * (size_t)ppc * SLOT);  // [2][ppc][2]
    double* sig = sm + 2 * (size_t)ppc * SLOT + 2 * (size_t)ppc;     // [ppc][2]
    int* rnk = reinterpret_cast<int*>(sig + 2 * ppc);                 // [ppc][2]
    __shared__ int flag[2];
    __shared__ int s_sweeps;

    // initial placement: top[i] = column 2i, bot[i] = column 2i+1
    if (active) {
        for (int h = 0; h < 2; ++h) {
            const int col = 2 * slot + h;
            double* G = buf0 + (size_t)warp * SLOT + (size_t)h * 2 * KPAD;
            double* Vv = G + KPAD;
            for (int i = lane; i < KPAD; i += 32) {
                G[i] = (col < k && i < k) ? a.M[(size_t)i * a.ldm + col] : 0.0;
                Vv[i] = (col < k && i == col) ? 1.0 : 0.0;
            }
            if (lane == 0) ids[(0 * ppc + warp) * 2 + h] = col;
        }
    }
    if (threadIdx.x == 0) {
        flag[0] = flag[1] = 0;
        s_sweeps = 0;
    }
    cl.sync();

    const double tol = sqrt((double)k) * 2.220446049250313e-16;
    const double tol2 = tol * tol;
    // ring destinations of this slot's two columns (fixed for the whole run):
    // top[i] -> top[i+1] (top[0] fixed, top[P-1] -> bot[P-1]); bot[i] -> bot[i-1] (bot[0] -> top[1])
    int dts = 0, dth = 0, dbs = 0, dbh = 1;
    if (P > 1) {
        if (slot == 0) { dts = 0; dth = 0; }
        else if (slot < P - 1) { dts = slot + 1; dth = 0; }
        else { dts = P - 1; dth = 1; }
        if (slot == 0) { dbs = 1; dbh = 0; }
        else { dbs = slot - 1; dbh = 1; }
    }
    double* dstT[2];
    double* dstB[2];
    {
        const size_t offT = (size_t)(dts % ppc) * SLOT + (size_t)dth * 2 * KPAD;
        const size_t offB = (size_t)(dbs % ppc) * SLOT + (size_t)dbh * 2 * KPAD;
        dstT[0] = cl.map_shared_rank(buf0, dts / ppc) + offT;
        dstT[1] = cl.map_shared_rank(buf1, dts / ppc) + offT;
        dstB[0] = cl.map_shared_rank(buf0, dbs / ppc) + offB;
        dstB[1] = cl.map_shared_rank(buf1, dbs / ppc) + offB;
    }
    int cur = 0;
    int sweep = 0, rounds = 0;
    for (; sweep < a.max_sweeps; ++sweep) {
        int rotated = 0;
        for (int rd = 0; rd < kk - 1; ++rd, ++rounds) {
            const double* src = cur ? buf1 : buf0;
            if (active) {
                const double* base = src + (size_t)warp * SLOT;
                double gt[KP], vt[KP], gb[KP], vb[KP];
#pragma unroll
                for (int p = 0; p < KP; ++p) {
                    const int i = lane + 32 * p;
                    gt[p] = base[i];
                    vt[p] = base[KPAD + i];
                    gb[p] = base[2 * KPAD + i];
                    vb[p] = base[3 * KPAD + i];
                }
                double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
                for (int p = 0; p < KP; ++p) {
                    al = fma(gt[p], gt[p], al);
                    be = fma(gb[p], gb[p], be);
                    ga = fma(gt[p], gb[p], ga);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (ga != 0.0 && ga * ga > tol2 * al * be) {
                    rotated = 1;
                    double c, sn;
                    jac_rotation(al, be, ga, c, sn);
#pragma unroll
                    for (int p = 0; p < KP; ++p) {
                        const double x = gt[p], y = gb[p];
                        gt[p] = c * x - sn * y;
                        gb[p] = sn * x + c * y;
                        const double u = vt[p], w = vb[p];
                        vt[p] = c * u - sn * w;
                        vb[p] = sn * u + c * w;
                    }
                }
                const int nxt = cur ^ 1;
                double* dT = nxt ? dstT[1] : dstT[0];  // selects keep the pointers in registers
                double* dB = nxt ? dstB[1] : dstB[0];
#pragma unroll
                for (int p = 0; p < KP; ++p) {
                    const int i = lane + 32 * p;
                    dT[i] = gt[p];
                    dT[KPAD + i] = vt[p];
                    dB[i] = gb[p];
                    dB[KPAD + i] = vb[p];
                }
            }
            if (C > 1) cl.sync();
            else __syncthreads();
            cur ^= 1;
            // flag[(sweep+1)&1] was last read by peers before this barrier
            if (rd == 0 && threadIdx.x == 0) flag[(sweep + 1) & 1] = 0;
        }
        if (rotated && lane == 0) atomicOr(&flag[sweep & 1], 1);
        cl.sync();
        int any = 0;
        for (int q = 0; q < C; ++q) any |= *cl.map_shared_rank(&flag[sweep & 1], q);
        if (!any) {
            ++sweep;
            break;
        }
    }
    if (threadIdx.x == 0) s_sweeps = sweep;
    // column origins after `rounds` ring shifts of the 2P-1 non-fixed positions
    if (active && lane < 2) {
        const int h = lane;
        const int Lc = 2 * P - 1;
        const int x = (h == 0) ? (slot == 0 ? -1 : slot - 1) : (2 * P - 2 - slot);
        int os = 0, oh = 0;
        if (x >= 0) {
            const int y = ((x - rounds % Lc) % Lc + Lc) % Lc;
            if (y < P - 1) { os = y + 1; oh = 0; }
            else { os = 2 * P - 2 - y; oh = 1; }
        }
        ids[(cur * ppc + warp) * 2 + h] = 2 * os + oh;
    }
    __syncthreads();

    // sigma of every local column, then a cluster-wide stable rank
    double* src = cur ? buf1 : buf0;
    if (active) {
        for (int h = 0; h < 2; ++h) {
            const double* G = src + (size_t)warp * SLOT + (size_t)h * 2 * KPAD;
            double ss = 0.0;
            for (int i = lane; i < KPAD; i += 32) ss = fma(G[i], G[i], ss);
            ss = warp_sum(ss);
            if (lane == 0) sig[warp * 2 + h] = sqrt(ss);
        }
    }
    cl.sync();
    if (active && lane < 2) {
        const int h = lane;
        const int id = ids[(cur * ppc + warp) * 2 + h];
        const double sv = sig[warp * 2 + h];
        int rk = 0;
        for (int q = 0; q < C; ++q) {
            const double* rs = cl.map_shared_rank(sig, q);
            const int* ri = cl.map_shared_rank(ids, q);
            for (int w = 0; w < ppc; ++w) {
                if (q * ppc + w >= P) break;
                for (int hh = 0; hh < 2; ++hh) {
                    const int oid = ri[(cur * ppc + w) * 2 + hh];
                    if (oid >= k || oid == id) continue;
                    const double os = rs[w * 2 + hh];
                    rk += (os > sv) || (os == sv && oid < id);
                }
            }
        }
        rnk[warp * 2 + h] = id < k ? rk : -1;
    }
    cl.sync();  // peers done reading sig / ids
    if (active) {
        for (int h = 0; h < 2; ++h) {
            const int rk = rnk[warp * 2 + h];
            if (rk < 0) continue;
            const double* G = src + (size_t)warp * SLOT + (size_t)h * 2 * KPAD;
            const double* Vv = G + KPAD;
            const double sv = sig[warp * 2 + h];
            double best = -1.0;
            int bi = 0;
            for (int i = lane; i < k; i += 32) {
                const double av = fabs(G[i]);
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
            const double sg = G[bi] < 0.0 ? -1.0 : 1.0;
            for (int i = lane; i < k; i += 32) {
                a.U[(size_t)i * a.ldu + rk] = sv > 0.0 ? sg * G[i] / sv : 0.0;
                a.V[(size_t)i * a.ldv + rk] = sg * Vv[i];
            }
            if (lane == 0) a.S[rk] = sv;
        }
    }
    if (r == 0 && threadIdx.x == 0 && a.sweeps_out) *a.sweeps_out = s_sweeps;
}

// Single-CTA variant (2 k^2 doubles fit in shared memory, k <= ~116): G and V
// columns stay at fixed places (column-major by column id); round r pairs the
// columns of the circle ordering directly (no data movement), one warp per
// pair holds the pair's two G columns in registers, the V columns are
// rotated in place (each column belongs to one pair per round), and rounds
// are separated by one __syncthreads. PPW pairs per warp are interleaved so
// their shuffle chains and square roots overlap.
__device__ __forceinline__ void jac_round_pair(int r, int i, int kk, int& p, int& q) {
    auto pos = [&](int t) { return t == 0 ? 0 : ((t - 1 + r) % (kk - 1)) + 1; };
    p = pos(i);
    q = pos(kk - 1 - i);
}

template <int KP, int PPW>
__global__ void __launch_bounds__(PPW == 1 ? 1024 : 512, 1) jacobi_cta_kernel(JacobiArgs a) {
    if (pred_off(a.pred, a.pred_skip)) return;  // uniform over the cluster
    const int k = a.k;
    const int kk = (k + 1) & ~1;
    const int P = kk / 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    extern __shared__ __align__(16) double sm[];
    double* G = sm;                         // column c at G + c*k
    double* V = sm + (size_t)k * k;
    double* sig = V + (size_t)k * k;        // [k]
    int* rnk = reinterpret_cast<int*>(sig + k);
    __shared__ int flag;
    __shared__ int s_sweeps;

    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int i = e / k, c = e - i * k;
        G[(size_t)c * k + i] = a.M[(size_t)i * a.ldm + c];
        V[(size_t)c * k + i] = (i == c) ? 1.0 : 0.0;
    }
    if (threadIdx.x == 0) s_sweeps = 0;
    __syncthreads();

    const double tol = sqrt((double)k) * 2.220446049250313e-16;
    const double tol2 = tol * tol;
    int sweep = 0;
    for (; sweep < a.max_sweeps; ++sweep) {
        if (threadIdx.x == 0) flag = 0;
        int rotated = 0;
        for (int rd = 0; rd < kk - 1; ++rd) {
            for (int pb = warp * PPW; pb < P; pb += nwarp * PPW) {
                int cp[PPW], cq[PPW];
                bool act[PPW];
                double gp[PPW][KP], gq[PPW][KP];
                double al[PPW], be[PPW], ga[PPW];
#pragma unroll
                for (int t = 0; t < PPW; ++t) {
                    int pp = 0, qq = 0;
                    act[t] = pb + t < P;
                    if (act[t]) jac_round_pair(rd, pb + t, kk, pp, qq);
                    act[t] = act[t] && pp < k && qq < k;  // dummy column for odd k
                    cp[t] = act[t] ? pp : 0;
                    cq[t] = act[t] ? qq : 0;
                    al[t] = be[t] = ga[t] = 0.0;
#pragma unroll
                    for (int p = 0; p < KP; ++p) {
                        const int i = lane + 32 * p;
                        const bool in = act[t] && i < k;
                        gp[t][p] = in ? G[(size_t)cp[t] * k + i] : 0.0;
                        gq[t][p] = in ? G[(size_t)cq[t] * k + i] : 0.0;
                        al[t] = fma(gp[t][p], gp[t][p], al[t]);
                        be[t] = fma(gq[t][p], gq[t][p], be[t]);
                        ga[t] = fma(gp[t][p], gq[t][p], ga[t]);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                    for (int t = 0; t < PPW; ++t) {
                        al[t] += __shfl_xor_sync(0xffffffffu, al[t], o);
                        be[t] += __shfl_xor_sync(0xffffffffu, be[t], o);
                        ga[t] += __shfl_xor_sync(0xffffffffu, ga[t], o);
                    }
                }
#pragma unroll
                for (int t = 0; t < PPW; ++t) {
                    if (!(act[t] && ga[t] != 0.0 && ga[t] * ga[t] > tol2 * al[t] * be[t])) continue;
                    rotated = 1;
                    double c, sn;
                    jac_rotation(al[t], be[t], ga[t], c, sn);
                    double* Gp = G + (size_t)cp[t] * k;
                    double* Gq = G + (size_t)cq[t] * k;
                    double* Vp = V + (size_t)cp[t] * k;
                    double* Vq = V + (size_t)cq[t] * k;
#pragma unroll
                    for (int p = 0; p < KP; ++p) {
                        const int i = lane + 32 * p;
                        if (i < k) {
                            const double x = gp[t][p], y = gq[t][p];
                            Gp[i] = c * x - sn * y;
                            Gq[i] = sn * x + c * y;
                            const double u = Vp[i], w = Vq[i];
                            Vp[i] = c * u - sn * w;
                            Vq[i] = sn * u + c * w;
                        }
                    }
                }
            }
            __syncthreads();
        }
        if (rotated && lane == 0) atomicOr(&flag, 1);
        __syncthreads();
        const int any = flag;
        __syncthreads();
        if (!any) {
            ++sweep;
            break;
        }
    }
    if (threadIdx.x == 0) s_sweeps = sweep;
    for (int c = warp; c < k; c += nwarp) {
        double ss = 0.0;
        for (int i = lane; i < k; i += 32) ss = fma(G[(size_t)c * k + i], G[(size_t)c * k + i], ss);
        ss = warp_sum(ss);
        if (lane == 0) sig[c] = sqrt(ss);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const double sv = sig[c];
        int rk = 0;
        for (int f = 0; f < k; ++f) rk += (sig[f] > sv) || (sig[f] == sv && f < c);
        rnk[c] = rk;
    }
    __syncthreads();
    for (int c = warp; c < k; c += nwarp) {
        const int rk = rnk[c];
        const double* Gc = G + (size_t)c * k;
        const double* Vc = V + (size_t)c * k;
        const double sv = sig[c];
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
        for (int i = lane; i < k; i += 32) {
            a.U[(size_t)i * a.ldu + rk] = sv > 0.0 ? sg * Gc[i] / sv : 0.0;
            a.V[(size_t)i * a.ldv + rk] = sg * Vc[i];
        }
        if (lane == 0) a.S[rk] = sv;
    }
    if (threadIdx.x == 0 && a.sweeps_out) *a.sweeps_out = s_sweeps;
}

__host__ __device__ inline size_t jacobi_cta_smem_bytes(int k) {
    return (2 * (size_t)k * k + 2 * (size_t)k) * sizeof(double);
}

}  // namespace sorsvd_dev


namespace sorsvd_dev {

// Point-to-point variant of jacobi_cluster_kernel (same ring, same rotations,
// same output contract). A cluster barrier per round costs a release fence
// (the DSMEM stores must land) plus the barrier itself; in the Brent-Luk ring
// a slot only ever receives from its two ring neighbours, and only sends to
// them, so the rounds need no cluster-wide synchronisation at all:
//  * columns travel by st.async (16-byte DSMEM stores that count their bytes
//    on the RECEIVER's mbarrier, one mbarrier per slot per buffer parity);
//  * a slot arms its barrier for the next round (expect_tx) and waits for the
//    current one (try_wait.parity), so it starts as soon as its two inputs land;
//  * double buffering is safe without any barrier: a neighbour can only send
//    round r+1 data after it received ours for round r, i.e. after we finished
//    reading the buffer it writes.
// One cluster barrier per SWEEP remains (the convergence vote, 3 rotating flags).
// Lane layout: a lane holds the element pairs 2 lane + 64 h + {0, 1}
// (h < KP/2) of each column, so every store is a 16-byte st.async.
__device__ __forceinline__ uint32_t jc_mapa(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void jc_st_async(uint32_t addr, double x, double y, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
                 "d"(x), "d"(y), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void jc_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void jc_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "JC_WAIT:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra JC_WAIT;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__host__ __device__ inline size_t jacobi_p2p_smem_bytes(int KP, int ppc) {
    const size_t slot = 4 * (size_t)(32 * KP);
    return (2 * (size_t)ppc * slot + 2 * 2 * (size_t)ppc + 4 * (size_t)ppc + 64) * sizeof(double);
}

template <int KP>
__global__ void jacobi_p2p_kernel(JacobiArgs a) {
    if (pred_off(a.pred, a.pred_skip)) return;  // uniform over the cluster
    static_assert(KP == 2 || KP == 4, "pairs of elements per lane; selected for k <= 128");
    constexpr int KPAD = 32 * KP;
    constexpr int H = KP / 2;
    cgj::cluster_group cl = cgj::this_cluster();
    const int C = (int)cl.num_blocks();
    const int r = (int)cl.block_rank();
    const int k = a.k, ppc = a.ppc;
    const int kk = (k + 1) & ~1;
    const int P = kk / 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = r * ppc + warp;
    const bool active = warp < ppc && slot < P;

    extern __shared__ __align__(16) double sm[];
    constexpr size_t SLOT = 4 * (size_t)KPAD;  // [top G | top V | bot G | bot V]
    double* buf0 = sm;
    double* buf1 = sm + (size_t)ppc * SLOT;
    int* ids = reinterpret_cast<int*>(sm + 2 * (size_t)ppc * SLOT);  // [2][ppc][2]
    double* sig = sm + 2 * (size_t)ppc * SLOT + 2 * (size_t)ppc;     // [ppc][2]
    int* rnk = reinterpret_cast<int*>(sig + 2 * ppc);                 // [ppc][2]
    __shared__ __align__(8) unsigned long long mbar[2][32];
    __shared__ int flag[3];
    __shared__ int s_sweeps;
    // de Rijk-style start: the columns enter the ring sorted by decreasing norm (ties by
    // index), which saves a sweep on graded cores (C2: 8 -> 7). perm[p] = the column of M
    // at ring position p; V's rows are mapped back through it at the end.
    __shared__ double cnorm[KPAD];
    __shared__ int perm[KPAD];
    for (int cidx = threadIdx.x; cidx < k; cidx += blockDim.x) {
        double ss = 0.0;
        for (int i = 0; i < k; ++i) ss = fma(a.M[(size_t)i * a.ldm + cidx], a.M[(size_t)i * a.ldm + cidx], ss);
        // NaN keys (non-finite M) sort last: the comparisons below then still give every
        // column a distinct rank, so perm stays a permutation (no stray row index)
        cnorm[cidx] = ss >= 0.0 ? ss : -1.0;
    }
    __syncthreads();
    for (int cidx = threadIdx.x; cidx < k; cidx += blockDim.x) {
        int rk = 0;
        for (int f = 0; f < k; ++f) rk += (cnorm[f] > cnorm[cidx]) || (cnorm[f] == cnorm[cidx] && f < cidx);
        perm[rk] = cidx;
    }
    __syncthreads();

    if (active) {
        for (int h = 0; h < 2; ++h) {
            const int col = 2 * slot + h;
            const int src = col < k ? perm[col] : 0;
            double* G = buf0 + (size_t)warp * SLOT + (size_t)h * 2 * KPAD;
            double* Vv = G + KPAD;
            for (int i = lane; i < KPAD; i += 32) {
                G[i] = (col < k && i < k) ? a.M[(size_t)i * a.ldm + src] : 0.0;
                Vv[i] = (col < k && i == col) ? 1.0 : 0.0;
            }
        }
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[0][warp])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[1][warp])));
        }
    }
    if (threadIdx.x == 0) {
        flag[0] = flag[1] = flag[2] = 0;
        s_sweeps = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    cl.sync();

    const double tol = sqrt((double)k) * 2.220446049250313e-16;
    const double tol2 = tol * tol;
    // ring destinations (as jacobi_cluster_kernel)
    int dts = 0, dth = 0, dbs = 0, dbh = 1;
    if (P > 1) {
        if (slot == 0) { dts = 0; dth = 0; }
        else if (slot < P - 1) { dts = slot + 1; dth = 0; }
        else { dts = P - 1; dth = 1; }
        if (slot == 0) { dbs = 1; dbh = 0; }
        else { dbs = slot - 1; dbh = 1; }
    }
    uint32_t sendT[2], sendB[2], barT[2], barB[2], myBar[2];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
        double* bx = x ? buf1 : buf0;
        sendT[x] = jc_mapa(smem_u32(bx + (size_t)(dts % ppc) * SLOT + (size_t)dth * 2 * KPAD + 2 * lane), dts / ppc);
        sendB[x] = jc_mapa(smem_u32(bx + (size_t)(dbs % ppc) * SLOT + (size_t)dbh * 2 * KPAD + 2 * lane), dbs / ppc);
        barT[x] = jc_mapa(smem_u32(&mbar[x][dts % ppc]), dts / ppc);
        barB[x] = jc_mapa(smem_u32(&mbar[x][dbs % ppc]), dbs / ppc);
        myBar[x] = smem_u32(&mbar[x][warp & 31]);
    }
    constexpr uint32_t kRxBytes = 4u * KPAD * 8u;  // top + bottom column, G and V each
    int R = 0;  // global round counter (buffer R & 1 holds round R's input)
    int sweep = 0;
    for (; sweep < a.max_sweeps; ++sweep) {
        if (threadIdx.x == 0) flag[(sweep + 1) % 3] = 0;  // last read two sweep barriers ago
        int rotated = 0;
        for (int rd = 0; rd < kk - 1; ++rd, ++R) {
            if (active) {
                const bool odd = R & 1;  // (selects, not indexing: keeps the addresses in registers)
                if (lane == 0) jc_expect(odd ? myBar[0] : myBar[1], kRxBytes);  // next round's inputs
                if (R > 0) jc_wait(odd ? myBar[1] : myBar[0], ((R - 1) >> 1) & 1);
                const double* base = (R & 1 ? buf1 : buf0) + (size_t)warp * SLOT + 2 * lane;
                double gt[KP], vt[KP], gb[KP], vb[KP];
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const double2 x0 = *reinterpret_cast<const double2*>(base + 64 * h);
                    const double2 x1 = *reinterpret_cast<const double2*>(base + KPAD + 64 * h);
                    const double2 x2 = *reinterpret_cast<const double2*>(base + 2 * KPAD + 64 * h);
                    const double2 x3 = *reinterpret_cast<const double2*>(base + 3 * KPAD + 64 * h);
                    gt[2 * h] = x0.x; gt[2 * h + 1] = x0.y;
                    vt[2 * h] = x1.x; vt[2 * h + 1] = x1.y;
                    gb[2 * h] = x2.x; gb[2 * h + 1] = x2.y;
                    vb[2 * h] = x3.x; vb[2 * h + 1] = x3.y;
                }
                double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
                for (int p = 0; p < KP; ++p) {
                    al = fma(gt[p], gt[p], al);
                    be = fma(gb[p], gb[p], be);
                    ga = fma(gt[p], gb[p], ga);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (ga != 0.0 && ga * ga > tol2 * al * be) {
                    rotated = 1;
                    double c, sn;
                    jac_rotation(al, be, ga, c, sn);
#pragma unroll
                    for (int p = 0; p < KP; ++p) {
                        const double x = gt[p], y = gb[p];
                        gt[p] = c * x - sn * y;
                        gb[p] = sn * x + c * y;
                        const double u = vt[p], w = vb[p];
                        vt[p] = c * u - sn * w;
                        vb[p] = sn * u + c * w;
                    }
                }
                const uint32_t sT = odd ? sendT[0] : sendT[1], bT = odd ? barT[0] : barT[1];
                const uint32_t sB = odd ? sendB[0] : sendB[1], bB = odd ? barB[0] : barB[1];
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    jc_st_async(sT + 512u * h, gt[2 * h], gt[2 * h + 1], bT);
                    jc_st_async(sT + 8u * KPAD + 512u * h, vt[2 * h], vt[2 * h + 1], bT);
                    jc_st_async(sB + 512u * h, gb[2 * h], gb[2 * h + 1], bB);
                    jc_st_async(sB + 8u * KPAD + 512u * h, vb[2 * h], vb[2 * h + 1], bB);
                }
            }
        }
        if (rotated && lane == 0) atomicOr(&flag[sweep % 3], 1);
        cl.sync();
        int any = 0;
        for (int q = 0; q < C; ++q) any |= *cl.map_shared_rank(&flag[sweep % 3], q);
        if (!any) {
            ++sweep;
            break;
        }
    }
    if (active && R > 0) jc_wait((R & 1) ? myBar[1] : myBar[0], ((R - 1) >> 1) & 1);  // the last round's columns
    const int rounds = R, cur = R & 1;
    if (threadIdx.x == 0) s_sweeps = sweep;
    // column origins after `rounds` ring shifts (as jacobi_cluster_kernel)
    if (active && lane < 2) {
        const int h = lane;
        const int Lc = 2 * P - 1;
        const int x = (h == 0) ? (slot == 0 ? -1 : slot - 1) : (2 * P - 2 - slot);
        int os = 0, oh = 0;
        if (x >= 0) {
            const int y = ((x - rounds % Lc) % Lc + Lc) % Lc;
            if (y < P - 1) { os = y + 1; oh = 0; }
            else { os = 2 * P - 2 - y; oh = 1; }
        }
        ids[(cur * ppc + warp) * 2 + h] = 2 * os + oh;
    }
    __syncthreads();
    double* src = cur ? buf1 : buf0;
    if (active) {
        for (int h = 0; h < 2; ++h) {
            const double* G = src + (size_t)warp * SLOT + (size_t)h * 2 * KPAD;
            double ss = 0.0;
            for (int i = lane; i < KPAD; i += 32) ss = fma(G[i], G[i], ss);
            ss = warp_sum(ss);
            if (lane == 0) sig[warp * 2 + h] = sqrt(ss);
        }
    }
    cl.sync();
    if (active && lane < 2) {
        const int h = lane;
        const int id = ids[(cur * ppc + warp) * 2 + h];
        const double sv = sig[warp * 2 + h];
        int rk = 0;
        for (int q = 0; q < C; ++q) {
            const double* rs = cl.map_shared_rank(sig, q);
            const int* ri = cl.map_shared_rank(ids, q);
            for (int w = 0; w < ppc; ++w) {
                if (q * ppc + w >= P) break;
                for (int hh = 0; hh < 2; ++hh) {
                    const int oid = ri[(cur * ppc + w) * 2 + hh];
                    if (oid >= k || oid == id) continue;
                    const double os = rs[w * 2 + hh];
                    rk += (os > sv) || (os == sv && oid < id);
                }
            }
        }
        rnk[warp * 2 + h] = id < k ? rk : -1;
    }
    cl.sync();  // peers done reading sig / ids
    if (active) {
        for (int h = 0; h < 2; ++h) {
            const int rk = rnk[warp * 2 + h];
            if (rk < 0) continue;
            const double* G = src + (size_t)warp * SLOT + (size_t)h * 2 * KPAD;
            const double* Vv = G + KPAD;
            const double sv = sig[warp * 2 + h];
            double best = -1.0;
            int bi = 0;
            for (int i = lane; i < k; i += 32) {
                const double av = fabs(G[i]);
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
            const double sg = G[bi] < 0.0 ? -1.0 : 1.0;
            for (int i = lane; i < k; i += 32) {
                a.U[(size_t)i * a.ldu + rk] = sv > 0.0 ? sg * G[i] / sv : 0.0;
                a.V[(size_t)perm[i] * a.ldv + rk] = sg * Vv[i];  // row i of V is ring position i
            }
            if (lane == 0) a.S[rk] = sv;
        }
    }
    if (r == 0 && threadIdx.x == 0 && a.sweeps_out) *a.sweeps_out = s_sweeps;
}

}  // namespace sorsvd_dev
