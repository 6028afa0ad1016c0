// K5: small dense SVD of the k x k core M by one-sided (Hestenes) Jacobi.
//
// Replaces truncated_svd(M, k) -> full_svd -> LAPACKE_dgesdd('S')
// (sketch.hpp:103, dense.hpp:65-110). Output contract is the reference's:
// sigma nonincreasing (stable order for ties), U and V orthonormal, each
// column of U canonicalised so its largest-magnitude entry is positive
// (dense.hpp:80-95: first maximal index wins), V flipped with it.
//
// One CTA; columns of G = M and of the accumulated rotation V live in shared
// memory (column-major). Each round of the round-robin ("circle") ordering is
// a perfect matching of the columns, processed by independent lane groups of
// SG lanes (several pairs per warp, no barrier inside a round); rounds are
// separated by one __syncthreads. Sweeps repeat until no pair exceeds the
// orthogonality threshold |g_p.g_q| <= tol*||g_p||*||g_q||, tol = sqrt(k)*eps
// (the dgesvj criterion), which gives high relative accuracy in sigma.
// For k > 112 the two k x k arrays live in a global (L2) scratch instead.
#pragma once
#include "common.cuh"

namespace sorsvd_dev {

constexpr int kJacobiThreads = 512;

struct JacobiArgs {
    const double* M;  // k x ldm row-major
    int ldm;
    int k;
    double* U;        // k x ldu row-major (first k columns written)
    int ldu;
    double* S;        // k
    double* V;        // k x ldv row-major
    int ldv;
    double* scratch;  // global fallback: 2 * ld * k doubles
    int max_sweeps;
    int* sweeps_out;  // optional
};

__device__ __forceinline__ void jacobi_pair(int r, int i, int kk, int& p, int& q) {
    // circle method: position 0 fixed, others rotate by r
    auto pos = [&](int t) { return t == 0 ? 0 : ((t - 1 + r) % (kk - 1)) + 1; };
    p = pos(i);
    q = pos(kk - 1 - i);
}

template <int SG, bool SMEM>
__global__ void __launch_bounds__(kJacobiThreads, 1) jacobi_svd_kernel(JacobiArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int s_rot;
    __shared__ int s_sweeps;
    const int k = a.k;
    const int ld = k | 1;
    double* G = SMEM ? sm : a.scratch;
    double* V = G + (size_t)ld * k;
    double* sig = SMEM ? V + (size_t)ld * k : sm;  // k
    int* rank = reinterpret_cast<int*>(sig + k);   // k
    int* imax = rank + k;                          // k

    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int i = e / k, c = e - i * k;
        G[(size_t)c * ld + i] = a.M[(size_t)i * a.ldm + c];
        V[(size_t)c * ld + i] = (i == c) ? 1.0 : 0.0;
    }
    if (threadIdx.x == 0) s_sweeps = 0;
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int lane_g = lane % SG;
    const int gpw = 32 / SG;  // lane groups per warp
    const int kk = (k & 1) ? k + 1 : k;
    const double tol = sqrt((double)k) * 2.220446049250313e-16;

    for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
        if (threadIdx.x == 0) s_rot = 0;
        __syncthreads();
        int rot = 0;
        for (int r = 0; r < kk - 1; ++r) {
            // warp-uniform trip count so the group shuffles never diverge
            for (int pb = warp * gpw; pb < kk / 2; pb += nwarp * gpw) {
                const int pi = pb + lane / SG;
                int p = 0, q = 0;
                bool valid = pi < kk / 2;
                if (valid) {
                    jacobi_pair(r, pi, kk, p, q);
                    valid = p < k && q < k;  // dummy player for odd k
                }
                double* gp = G + (size_t)p * ld;
                double* gq = G + (size_t)q * ld;
                double al = 0.0, be = 0.0, ga = 0.0;
                if (valid) {
                    for (int i = lane_g; i < k; i += SG) {
                        const double x = gp[i], y = gq[i];
                        al = fma(x, x, al);
                        be = fma(y, y, be);
                        ga = fma(x, y, ga);
                    }
                }
                al = group_sum<SG>(al);
                be = group_sum<SG>(be);
                ga = group_sum<SG>(ga);
                if (!valid || ga == 0.0 || !(fabs(ga) > tol * sqrt(al) * sqrt(be))) continue;
                ++rot;
                const double zeta = (be - al) / (2.0 * ga);
                double t;
                if (fabs(zeta) > 1e100)
                    t = 0.5 / zeta;
                else
                    t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
                const double c = 1.0 / sqrt(fma(t, t, 1.0));
                const double s = c * t;
                double* vp = V + (size_t)p * ld;
                double* vq = V + (size_t)q * ld;
                for (int i = lane_g; i < k; i += SG) {
                    const double x = gp[i], y = gq[i];
                    gp[i] = c * x - s * y;
                    gq[i] = s * x + c * y;
                    const double u = vp[i], w = vq[i];
                    vp[i] = c * u - s * w;
                    vq[i] = s * u + c * w;
                }
            }
            __syncthreads();
        }
        if (rot && (threadIdx.x % SG) == 0) atomicAdd(&s_rot, 1);
        __syncthreads();
        const int any = s_rot;
        if (threadIdx.x == 0) s_sweeps = sweep + 1;
        __syncthreads();
        if (!any) break;
    }

    // singular values = column norms
    for (int cb = warp * gpw; cb < k; cb += nwarp * gpw) {
        const int c = cb + lane / SG;
        const double* gc = G + (size_t)(c < k ? c : 0) * ld;
        double ss = 0.0;
        if (c < k)
            for (int i = lane_g; i < k; i += SG) ss = fma(gc[i], gc[i], ss);
        ss = group_sum<SG>(ss);
        if (lane_g == 0 && c < k) sig[c] = sqrt(ss);
    }
    __syncthreads();
    // stable descending order
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        const double sj = sig[j];
        int rk = 0;
        for (int i = 0; i < k; ++i) rk += (sig[i] > sj) || (sig[i] == sj && i < j);
        rank[j] = rk;
    }
    // sign canonicalisation index: first largest |u_ij| (u_j = g_j / sigma_j)
    for (int cb = warp * gpw; cb < k; cb += nwarp * gpw) {
        const int c = cb + lane / SG;
        const double* gc = G + (size_t)(c < k ? c : 0) * ld;
        double best = -1.0;
        int bi = 0;
        for (int i = lane_g; i < k && c < k; i += SG) {
            const double av = fabs(gc[i]);
            if (av > best) {
                best = av;
                bi = i;
            }
        }
#pragma unroll
        for (int o = SG / 2; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
        if (lane_g == 0 && c < k) imax[c] = bi;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int c = e / k, i = e - c * k;  // column c (source), row i
        const int rc = rank[c];
        const double sc = sig[c];
        const double sg = G[(size_t)c * ld + imax[c]] < 0.0 ? -1.0 : 1.0;
        a.U[(size_t)i * a.ldu + rc] = sc > 0.0 ? sg * G[(size_t)c * ld + i] / sc : 0.0;
        a.V[(size_t)i * a.ldv + rc] = sg * V[(size_t)c * ld + i];
    }
    for (int c = threadIdx.x; c < k; c += blockDim.x) a.S[rank[c]] = sig[c];
    if (threadIdx.x == 0 && a.sweeps_out) *a.sweeps_out = s_sweeps;
}

}  // namespace sorsvd_dev
