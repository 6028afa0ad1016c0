// K3 for 256 < k <= 512: adaptive shifted CholeskyQR building blocks.
//
// The cluster Householder TSQR (cqr_f64.cuh) keeps a 2k x k tree node in one
// cluster's shared memory, which stops at k = 256. Above that, thin_qr
// (dense.hpp:114-134) is computed by up to five CholeskyQR passes
// X_{i} = X_{i-1} R_i^{-1}, each of which decides on the device:
//   * G = X^T X is I to within 1e-13      -> X is orthonormal: stop (the
//     remaining passes are predicated off and X is carried through);
//   * plain Cholesky with pivots within 1e-12 of each other -> plain pass;
//   * otherwise the shifted pass of Fukaya et al. (shifted CholeskyQR):
//     R = chol(G + s I), s = 11 (m k + k (k+1)) eps tr(G), which cuts the
//     condition number by ~sqrt(s)/||X|| (~1e4 here) per pass.
// So well-conditioned sketches cost CholeskyQR2 plus one Gram check, and the
// power-iterated sketches of Config 5 (cond ~ 512^5 .. 512^6) take two or
// three shifted passes first. R = R_p ... R_1 is upper triangular with
// diag(R) > 0 (the reference's sign convention, dense.hpp:127-132). The skinny
// Gram / update products are DMMA GEMMs (gemm_f64.cuh); this file holds the
// k x k pieces:
//
//  * cholc_kernel: blocked (32) right-looking Cholesky distributed over a
//    thread-block cluster, CTA r owning rows [32r, 32r+32) of L in shared
//    memory (k = 512: 16 CTAs x 128 KB). Per block step: the owner factors
//    its 32 x 32 diagonal block and inverts it, the CTAs below form their
//    panel blocks from that inverse (read over DSMEM), then update their
//    trailing blocks from the peers' panel blocks. Two cluster barriers per
//    block step (2k/32 in total). Writes R = L^T (upper, row-major).
//  * trsm_rows_kernel: X R = T by 32-column blocks (the off-diagonal part of
//    each block is a DMMA GEMM, X_{<J} R_{<J,J}): no explicit R^{-1}, whose
//    rounding error would grow like cond(R)^2 in the trailing directions.
//  * trinv_kernel: R^{-1} (upper) by back substitution, one warp per column.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace sorsvd_dev {

namespace cgc = cooperative_groups;

constexpr int kCholcThreads = 512;
constexpr int kCholcB = 32;

struct CholcArgs {
    const double* G;    // k x ldg symmetric (upper part read)
    int ldg;
    int k;
    double shift_coef;  // shifted attempt: G + shift_coef * tr(G) * I
    double* R;          // k x ldr upper (lower part zeroed)
    int ldr;
    int* flag;          // set to 1 when even the shifted factorisation fails (never cleared here)
    int* done;          // sticky: set to 1 when G is already I to within done_tol (X orthonormal)
    double done_tol;
    int* shifted;       // out: 1 when this pass used the shift (diagnostics)
    // mode 0: the adaptive pass above. Modes 1 / 2: a CholeskyQR2 factorisation for
    // k where chol_inv_kernel's factor no longer fits one CTA's shared memory (k > 160),
    // same gates as chol_inv_kernel (cholqr_f64.cuh): `flag` is the CholeskyQR2 flag
    // (0 accept, 1 fall back to Householder); pass 1 rejects on a pivot ratio below
    // 1e-14, pass 2 (skipped once pass 1 rejected) on max |G - I| > 1e-2.
    int mode;
    const int* outer;   // enclosing launch predicate (modes 1/2): pass 1 marks flag dead when off
    int outer_skip;
};

__host__ __device__ inline size_t cholc_smem_bytes(int k) {
    const int kp = ((k + kCholcB - 1) / kCholcB) * kCholcB;
    return ((size_t)kCholcB * kp + 3 * (size_t)kCholcB * kCholcB) * sizeof(double);
}

// One adaptive CholeskyQR pass decision + factor (see the file comment):
//   max |G - I| < done_tol          -> *done = 1, nothing else (X is orthonormal)
//   plain Cholesky, pivots in ratio -> R = chol(G)
//   otherwise                       -> R = chol(G + s I)   (shifted pass)
__global__ void __launch_bounds__(kCholcThreads, 1) cholc_kernel(CholcArgs a) {
    cgc::cluster_group cl = cgc::this_cluster();
    const int C = (int)cl.num_blocks(), r = (int)cl.block_rank();
    if (a.mode == 0) {
        if (*a.done) return;  // uniform over the cluster
    } else {
        if (pred_off(a.outer, a.outer_skip)) {  // enclosing iteration skipped: both QR paths skip
            if (a.mode == 1 && r == 0 && threadIdx.x == 0) *a.flag = kPredDead;
            return;
        }
        if (a.mode == 2 && *a.flag != 0) return;  // pass 1 rejected (or dead)
    }
    const int k = a.k, kp = C * kCholcB, tid = threadIdx.x;
    constexpr int B = kCholcB;
    extern __shared__ __align__(16) double sh[];
    double* Ls = sh;                      // [B][kp]: rows 32r.. of L (lower part meaningful)
    double* Dinv = Ls + (size_t)B * kp;   // [B][B] inverse of own diagonal block (lower)
    double* Pb = Dinv + B * B;            // [B][B] fetched remote block
    double* Tb = Pb + B * B;              // [B][B] temporary
    __shared__ int s_bad;
    __shared__ double s_piv, s_shift, s_dev, s_pmin, s_pmax;
    const int row0 = r * B;
    // gate: max |G - I| over this CTA's rows, reduced over the cluster
    if (a.mode != 1) {
        double dev = 0.0;
        for (int e = tid; e < B * k; e += blockDim.x) {
            const int i = e / k, j = e - i * k, gi = row0 + i;
            if (gi < k) {
                const double g = j >= gi ? a.G[(size_t)gi * a.ldg + j] : a.G[(size_t)j * a.ldg + gi];
                dev = fmax(dev, fabs(g - (j == gi ? 1.0 : 0.0)));
            }
        }
        for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
        if (tid == 0) s_dev = 0.0;
        __syncthreads();
        if ((tid & 31) == 0) {
            // non-negative doubles order like their bit patterns
            atomicMax(reinterpret_cast<unsigned long long*>(&s_dev), (unsigned long long)__double_as_longlong(dev));
        }
        cl.sync();
        double dmax = 0.0;
        for (int q = 0; q < C; ++q) dmax = fmax(dmax, *cl.map_shared_rank(&s_dev, q));
        cl.sync();
        if (a.mode == 0 && dmax < a.done_tol) {
            if (r == 0 && tid == 0) *a.done = 1;
            return;
        }
        if (a.mode == 2 && !(dmax <= 1e-2)) {  // Q' too far from orthonormal: Householder instead
            if (r == 0 && tid == 0) *a.flag = 1;
            return;
        }
    }
    int any_bad = 1;
    const int attempts = a.mode == 0 ? 2 : 1;  // CholeskyQR2 passes are never shifted
    for (int attempt = 0; attempt < attempts && any_bad; ++attempt) {
        if (tid == 0) {
            s_bad = 0;
            s_pmin = 1e300;
            s_pmax = 0.0;
            double tr = 0.0;
            if (attempt == 1)
                for (int i = 0; i < k; ++i) tr += a.G[(size_t)i * a.ldg + i];
            s_shift = attempt == 1 ? a.shift_coef * tr : 0.0;
        }
        __syncthreads();
        for (int e = tid; e < B * kp; e += blockDim.x) {
            const int i = e / kp, j = e - i * kp, gi = row0 + i;
            double v = 0.0;
            if (gi < k && j < k && j <= gi) v = a.G[(size_t)j * a.ldg + gi] + (j == gi ? s_shift : 0.0);
            if (gi >= k && j == gi) v = 1.0;  // padded rows: identity (keeps the factor nonsingular)
            Ls[e] = v;
        }
        __syncthreads();
        for (int J = 0; J < C; ++J) {
            const int c0 = J * B;
            if (r == J) {
                // unblocked Cholesky of the diagonal block D = Ls[:, c0:c0+B]
                for (int jj = 0; jj < B; ++jj) {
                    if (tid == 0) {
                        const double d = Ls[(size_t)jj * kp + c0 + jj];
                        if (!(d > 0.0) || !isfinite(d)) s_bad = 1;
                        if (c0 + jj < k) {
                            s_pmin = fmin(s_pmin, d);
                            s_pmax = fmax(s_pmax, d);
                        }
                        s_piv = d > 0.0 ? sqrt(d) : 1.0;
                        Ls[(size_t)jj * kp + c0 + jj] = s_piv;
                    }
                    __syncthreads();
                    const double pv = s_piv;
                    if (tid > jj && tid < B) Ls[(size_t)tid * kp + c0 + jj] /= pv;
                    __syncthreads();
                    for (int e = tid; e < B * B; e += blockDim.x) {
                        const int i = e / B, c = e - i * B;
                        if (c > jj && c <= i)
                            Ls[(size_t)i * kp + c0 + c] = fma(-Ls[(size_t)i * kp + c0 + jj],
                                                              Ls[(size_t)c * kp + c0 + jj], Ls[(size_t)i * kp + c0 + c]);
                    }
                    __syncthreads();
                }
                // Dinv = D^{-1} (lower): column c by forward substitution, one thread per column
                if (tid < B) {
                    const int c = tid;
                    for (int i = 0; i < B; ++i) {
                        double v = 0.0;
                        if (i == c) v = 1.0 / Ls[(size_t)i * kp + c0 + i];
                        else if (i > c) {
                            double acc = 0.0;
                            for (int l = c; l < i; ++l) acc = fma(Ls[(size_t)i * kp + c0 + l], Dinv[l * B + c], acc);
                            v = -acc / Ls[(size_t)i * kp + c0 + i];
                        }
                        Dinv[i * B + c] = v;
                    }
                }
            }
            cl.sync();
            if (*cl.map_shared_rank(&s_bad, J)) break;  // uniform: every CTA reads the owner's flag
            if (r > J) {
                // panel block L_rJ = A_rJ * Dinv^T
                const double* Dr = cl.map_shared_rank(Dinv, J);
                for (int e = tid; e < B * B; e += blockDim.x) Pb[e] = Dr[e];
                __syncthreads();
                for (int e = tid; e < B * B; e += blockDim.x) {
                    const int i = e / B, j = e - i * B;
                    double acc = 0.0;
                    for (int l = 0; l <= j; ++l) acc = fma(Ls[(size_t)i * kp + c0 + l], Pb[j * B + l], acc);
                    Tb[e] = acc;
                }
                __syncthreads();
                for (int e = tid; e < B * B; e += blockDim.x) {
                    const int i = e / B, j = e - i * B;
                    Ls[(size_t)i * kp + c0 + j] = Tb[e];
                }
            }
            cl.sync();
            if (r > J) {
                // trailing update A_rc -= L_rJ L_cJ^T for J < c <= r
                for (int cb = J + 1; cb <= r; ++cb) {
                    const double* Lc = cl.map_shared_rank(Ls, cb);
                    for (int e = tid; e < B * B; e += blockDim.x) {
                        const int i = e / B, j = e - i * B;
                        Pb[e] = Lc[(size_t)i * kp + c0 + j];  // L_cJ[i][j]
                    }
                    __syncthreads();
                    for (int e = tid; e < B * B; e += blockDim.x) {
                        const int i = e / B, j = e - i * B;
                        if (cb == r && j > i) continue;
                        double acc = Ls[(size_t)i * kp + cb * B + j];
#pragma unroll 8
                        for (int l = 0; l < B; ++l) acc = fma(-Ls[(size_t)i * kp + c0 + l], Pb[j * B + l], acc);
                        Ls[(size_t)i * kp + cb * B + j] = acc;
                    }
                    __syncthreads();
                }
            }
        }
        cl.sync();
        any_bad = 0;
        double pmin = 1e300, pmax = 0.0;
        for (int q = 0; q < C; ++q) {
            any_bad |= *cl.map_shared_rank(&s_bad, q);
            pmin = fmin(pmin, *cl.map_shared_rank(&s_pmin, q));
            pmax = fmax(pmax, *cl.map_shared_rank(&s_pmax, q));
        }
        // the plain pass is only trusted when cond(X) < ~1e6 (pivot ratio ~ 1/cond^2)
        const double piv_gate = a.mode == 0 ? 1e-12 : a.mode == 1 ? 1e-14 : 0.0;
        if (attempt == 0 && !(pmin > piv_gate * pmax)) any_bad = 1;
        cl.sync();  // peers done reading the flags before the next attempt resets them
        if (!any_bad && r == 0 && tid == 0 && a.shifted) *a.shifted = attempt;
    }
    // R = L^T: R[i][j] = L[j][i], j in this CTA's rows
    if (any_bad) {
        if (r == 0 && tid == 0) *a.flag = 1;
    } else {
        for (int e = tid; e < B * k; e += blockDim.x) {
            const int jl = e / k, i = e - jl * k, j = row0 + jl;
            if (j < k) a.R[(size_t)i * a.ldr + j] = (i <= j) ? Ls[(size_t)jl * kp + i] : 0.0;
        }
        if (a.mode == 1 && r == 0 && tid == 0) *a.flag = 0;
    }
}

// Block column of X R = T for upper-triangular R (the backward-stable
// replacement of X = T R^{-1} with an explicit inverse): rows are independent;
// each thread owns one row, forms y = T_J - W_J (W_J = X_{<J} R_{<J,J}, the
// DMMA GEMM part, or nothing for J = 0) and forward-substitutes
// x_c = (y_c - sum_{l<c} x_l R_lc) / R_cc over the 32 columns of the block.
__global__ void __launch_bounds__(256) trsm_rows_kernel(const double* __restrict__ T, int64_t ldt,
                                                        const double* __restrict__ W, int64_t ldw,
                                                        const double* __restrict__ Rjj, int ldr, int nb,
                                                        double* __restrict__ X, int64_t ldx, int64_t rows,
                                                        const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    __shared__ double Rs[kCholcB][kCholcB + 1];
    for (int e = threadIdx.x; e < kCholcB * kCholcB; e += blockDim.x) {
        const int i = e / kCholcB, j = e - i * kCholcB;
        Rs[i][j] = (i < nb && j < nb) ? Rjj[(size_t)i * ldr + j] : (i == j ? 1.0 : 0.0);
    }
    __syncthreads();
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= rows) return;
    double x[kCholcB];
    const double* tr = T + row * ldt;
#pragma unroll
    for (int c = 0; c < kCholcB; ++c) x[c] = c < nb ? tr[c] : 0.0;
    if (W) {
        const double* wr = W + row * ldw;
#pragma unroll
        for (int c = 0; c < kCholcB; ++c)
            if (c < nb) x[c] -= wr[c];
    }
#pragma unroll
    for (int c = 0; c < kCholcB; ++c) {
        double acc = x[c];
#pragma unroll
        for (int l = 0; l < c; ++l) acc = fma(-x[l], Rs[l][c], acc);
        x[c] = acc / Rs[c][c];
    }
    double* xr = X + row * ldx;
#pragma unroll
    for (int c = 0; c < kCholcB; ++c)
        if (c < nb) xr[c] = x[c];
}

__global__ void set_identity_kernel(double* __restrict__ R, int ldr, int k) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * ldr; e += gridDim.x * blockDim.x) {
        const int i = e / ldr, j = e - i * ldr;
        R[e] = (i == j) ? 1.0 : 0.0;
    }
}

// Big-QR flags at the start of a call: [0] breakdown = 0, [1] done = 0, or
// done = kPredDead when the enclosing launch predicate is off (every pass of
// the QR then skips, including the carry-through copies).
__global__ void qr_flags_init_kernel(int* flags, const int* outer, int outer_skip) {
    if (threadIdx.x == 0) {
        flags[0] = 0;
        flags[1] = pred_off(outer, outer_skip) ? kPredDead : 0;
    }
}

// dst = src (rows x cols, pitches in doubles) when *pred != pred_skip.
__global__ void copy_rows_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd,
                                 int64_t rows, int cols, const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    const int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / cols, j = e - i * cols;
        dst[i * ldd + j] = src[i * lds + j];
    }
}

// Rout = R2 R1 for upper-triangular k x k factors (CholeskyQR2's R), one thread
// per upper element: Rout_ij = sum_{l=i..j} R2_il R1_lj.
__global__ void triu_mul_kernel(const double* __restrict__ R2, int ld2, const double* __restrict__ R1, int ld1,
                                double* __restrict__ Ro, int ldo, int k, const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
        const int i = e / k, j = e - i * k;
        double acc = 0.0;
        for (int l = i; l <= j; ++l) acc = fma(R2[(size_t)i * ld2 + l], R1[(size_t)l * ld1 + j], acc);
        Ro[(size_t)i * ldo + j] = j >= i ? acc : 0.0;
    }
}

// Rinv = R^{-1} for upper-triangular R (k x ldr), one warp per column:
// x_c = 1/R_cc, x_i = -(sum_{l=i+1..c} R_il x_l) / R_ii for i = c-1 .. 0.
// Lower part of Rinv zeroed; Rinv padded columns are left untouched.
__global__ void trinv_kernel(const double* __restrict__ R, int ldr, int k, double* __restrict__ Ri, int ldi,
                             const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    extern __shared__ double xs[];  // [warps][k]
    const int wpb = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * wpb + warp;
    if (c >= k) return;
    double* x = xs + (size_t)warp * k;
    for (int i = lane; i < k; i += 32) x[i] = 0.0;
    __syncwarp();
    if (lane == 0) x[c] = 1.0 / R[(size_t)c * ldr + c];
    __syncwarp();
    for (int i = c - 1; i >= 0; --i) {
        const double* Rr = R + (size_t)i * ldr;
        double acc = 0.0;
        for (int l = i + 1 + lane; l <= c; l += 32) acc = fma(Rr[l], x[l], acc);
        acc = warp_sum(acc);
        if (lane == 0) x[i] = -acc / Rr[i];
        __syncwarp();
    }
    for (int i = lane; i < k; i += 32) Ri[(size_t)i * ldi + c] = x[i];
}

}  // namespace sorsvd_dev
