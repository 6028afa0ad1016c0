// K3 fast path: adaptive CholeskyQR2 for well-conditioned sketches.
//
// thin_qr (dense.hpp:114-134) is required to be Householder-accurate, which
// the cluster Householder kernel (cqr_f64.cuh) always is. When the sketch is
// well conditioned (C1, C3, C4: the sketch spectra span a few decades at
// most) the same Q and R follow from two CholeskyQR passes
//     G = T^T T = R1^T R1,  Q' = T R1^{-1},  G' = Q'^T Q' = R2^T R2,  Q = Q' R2^{-1},
// whose bulk is four skinny GEMMs over all SMs (gemm_f64.cuh) instead of 2k
// sequential reflector steps. Cholesky factors have a positive diagonal, so
// the reference sign convention diag(R) >= 0 holds by construction.
//
// The decision is taken on the device: chol_inv_kernel writes a flag (0 =
// CholeskyQR2 accepted, 1 = fall back to Householder) and every kernel of
// both paths is predicated on it (early uniform return), so the whole QR stays
// inside one CUDA graph with no host round trip. Gates: pass 1 needs positive
// pivots with min/max pivot^2 > 1e-14 (diagonal condition estimate < 1e7);
// pass 2 needs max |Q'^T Q' - I| < 1e-2 (CholeskyQR2 is then orthogonal to
// O(eps)); anything else -> Householder.
#pragma once
#include "common.cuh"

namespace sorsvd_dev {

constexpr int kCholThreads = 1024;
constexpr size_t kCholSmemBytes = 200 * 1024;  // dynamic shared memory of chol_inv_kernel

struct CholArgs {
    const double* G;   // k x ldg symmetric (upper part used)
    int ldg;
    int k;
    double* Rinv;      // k x ldr: upper-triangular R^{-1} (zeros below, padded cols untouched)
    int ldr;
    double* work;      // k x k scratch when the factor does not fit in shared memory
    int* flag;         // 0 = accept, 1 = fallback
    int pass;          // 1 or 2
    const double* R1;  // pass 2: first-pass R (k x ldr1) to form R = R2 R1 (optional)
    int ldr1;
    double* Rout;      // pass 2: R = R2 R1 (k x ldo), optional
    int ldo;
    double* Rf;        // pass 1: this pass's R (k x ldf, upper), optional
    int ldf;
    const int* outer;  // enclosing launch predicate (optional): when off, pass 1 marks *flag dead
    int outer_skip;
};

__global__ void __launch_bounds__(kCholThreads, 1) chol_inv_kernel(CholArgs a) {
    extern __shared__ __align__(16) double smc[];
    __shared__ int s_bad;
    __shared__ double s_piv[2];
    const int k = a.k, tid = threadIdx.x;
    if (pred_off(a.outer, a.outer_skip)) {  // enclosing iteration skipped: both QR paths skip too
        if (a.pass == 1 && tid == 0) *a.flag = kPredDead;
        return;
    }
    if (a.pass == 2 && *a.flag != 0) return;  // pass 1 already rejected (or the flag is dead)
    const bool in_smem = (size_t)k * k * sizeof(double) <= kCholSmemBytes;
    double* L = in_smem ? smc : a.work;  // row-major k x k, lower triangle holds R^T
    if (tid == 0) s_bad = 0;
    double dev = 0.0;
    for (int e = tid; e < k * k; e += blockDim.x) {
        const int i = e / k, j = e - i * k;
        const double g = (j <= i) ? a.G[(size_t)j * a.ldg + i] : 0.0;  // lower triangle from the upper part
        L[e] = g;
        if (a.pass == 2 && j <= i) dev = fmax(dev, fabs(g - (i == j ? 1.0 : 0.0)));
    }
    if (a.pass == 2) {
        // max |Q'^T Q' - I| gate
        for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
        if ((tid & 31) == 0 && dev > 1e-2) atomicExch(&s_bad, 1);
    }
    __syncthreads();
    // right-looking Cholesky: L L^T = G
    double pmax = 0.0, pmin = 1e300;
    for (int j = 0; j < k; ++j) {
        if (tid == 0) {
            const double d = L[(size_t)j * k + j];
            if (!(d > 0.0)) s_bad = 1;
            const double r = d > 0.0 ? sqrt(d) : 1.0;
            L[(size_t)j * k + j] = r;
            s_piv[0] = r;
            pmax = fmax(pmax, d);
            pmin = fmin(pmin, d);
            // the pass-1 pivot gate is monotone (pmin only falls, pmax only rises):
            // reject as soon as it fails instead of after the whole factorisation
            if (a.pass == 1 && !(pmin > 1e-14 * pmax)) s_bad = 1;
        }
        __syncthreads();
        if (s_bad) break;  // not positive definite: reject early (uniform: shared flag)
        const double r = s_piv[0];
        for (int i = j + 1 + tid; i < k; i += blockDim.x) L[(size_t)i * k + j] /= r;
        __syncthreads();
        // trailing rank-1 update of the lower triangle: one warp per row, lanes
        // across its columns (no per-element index division; each element still
        // sees the same fma sequence over j, so the factor is unchanged)
        {
            const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
            for (int i = j + 1 + warp; i < k; i += nw) {
                double* Li = L + (size_t)i * k;
                const double lij = Li[j];
                for (int c = j + 1 + lane; c <= i; c += 32) Li[c] = fma(-lij, L[(size_t)c * k + j], Li[c]);
            }
        }
        __syncthreads();
    }
    if (tid == 0 && a.pass == 1 && !(pmin > 1e-14 * pmax)) s_bad = 1;
    __syncthreads();
    if (s_bad) {
        if (tid == 0) *a.flag = 1;
        return;
    }
    if (tid == 0 && a.pass == 1) *a.flag = 0;
    if (a.Rf)
        for (int e = tid; e < k * k; e += blockDim.x) {
            const int i = e / k, c = e - i * k;
            a.Rf[(size_t)i * a.ldf + c] = c >= i ? L[(size_t)c * k + i] : 0.0;
        }
    // R = L^T (upper). Rinv column c solves R x = e_c by back substitution (one thread per column);
    // the partial solution stays in shared memory (xs, column-interleaved) rather than being
    // re-read from global memory, same operation order as before.
    double* xs = in_smem ? smc + (size_t)k * k : nullptr;
    const bool xs_ok = in_smem && ((size_t)k * k + (size_t)k * k) * sizeof(double) <= kCholSmemBytes;
    for (int c = tid; c < k; c += blockDim.x) {
        // x_i for i <= c, from i = c down to 0: x_i = (delta_ic - sum_{l=i+1..c} R_il x_l) / R_ii, R_il = L[l][i]
        for (int i = c; i >= 0; --i) {
            double s = (i == c) ? 1.0 : 0.0;
            if (xs_ok)
                for (int l = i + 1; l <= c; ++l) s = fma(-L[(size_t)l * k + i], xs[(size_t)l * k + c], s);
            else
                for (int l = i + 1; l <= c; ++l) s = fma(-L[(size_t)l * k + i], a.Rinv[(size_t)l * a.ldr + c], s);
            const double x = s / L[(size_t)i * k + i];
            if (xs_ok) xs[(size_t)i * k + c] = x;
            a.Rinv[(size_t)i * a.ldr + c] = x;
        }
        for (int i = c + 1; i < k; ++i) a.Rinv[(size_t)i * a.ldr + c] = 0.0;
    }
    if (a.pass == 2 && a.Rout) {
        // R = R2 R1 (both upper): R(i,c) = sum_{l=i..c} R2(i,l) R1(l,c), R2(i,l) = L[l][i]
        for (int e = tid; e < k * k; e += blockDim.x) {
            const int i = e / k, c = e - i * k;
            double s = 0.0;
            if (c >= i)
                for (int l = i; l <= c; ++l) s = fma(L[(size_t)l * k + i], a.R1[(size_t)l * a.ldr1 + c], s);
            a.Rout[(size_t)i * a.ldo + c] = s;
        }
    }
}

}  // namespace sorsvd_dev
