// K3: communication-avoiding tall-skinny QR (TSQR) in FP64.
//
// Replaces thin_qr (dense.hpp:114-134: LAPACKE_dgeqrf + LAPACKE_dorgqr + the
// diag(R) >= 0 sign fix at :127-132) for T1 (m x k) and T2 (n x k)
// (sketch.hpp:98-99).
//
//  * leaf kernel   : one CTA per row block; Householder QR (dgeqr2/dlarfg
//                    semantics) of the block held column-major in shared
//                    memory, then the explicit block Q formed in place
//                    (dorg2r semantics). R goes up the tree.
//  * node kernel   : one CTA per tree node; QR of the stacked [R_a; R_b]
//                    (2k x k), explicit node Q (2k x k). The root applies the
//                    reference sign convention diag(R) >= 0 by scaling its Q
//                    columns, so the final Q needs no separate pass.
//  * top-down      : the k x k "path" factors C are pushed down the tree with
//                    the segmented DMMA GEMM (gemm_f64.cuh), and the final
//                    Q rows = Q_leaf * C_leaf (one m x k x k segmented GEMM).
//
// Inside a CTA the k sequential reflector steps are the latency chain, so
// columns are owned by warps, each step costs exactly one __syncthreads, the
// owner of column j+1 builds reflector j+1 as soon as its own column is
// updated (look-ahead), and every warp reduces the dot products of several
// columns at once so their shuffle chains overlap.
//
// Blocks live in shared memory when 2k*k*8 bytes fit (k <= 112); otherwise the
// same code runs on a per-block column-major scratch region in global memory
// (L2-resident; slower, used for k = 256).
#pragma once
#include "common.cuh"

namespace sorsvd_dev {

constexpr int kQrThreads = 512;
constexpr int kQrSmemBudget = 200 * 1024;  // bytes of dynamic smem for one block

// Householder reflector for column j, rows [j, R) of a column-major block
// (dlarfg): x -> beta e_j, v = [1; x(j+1:)/(alpha-beta)], tau = (beta-alpha)/beta.
__device__ __forceinline__ void qr_make_reflector(double* A, int ld, int R, int j, double* tau, int lane) {
    double* x = A + (size_t)j * ld;
    const double alpha = x[j];
    double ss = 0.0;
    for (int i = j + 1 + lane; i < R; i += 32) ss = fma(x[i], x[i], ss);
    ss = warp_sum(ss);
    if (ss == 0.0) {
        if (lane == 0) tau[j] = 0.0;
        __syncwarp();
        return;
    }
    const double beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
    const double scal = 1.0 / (alpha - beta);
    for (int i = j + 1 + lane; i < R; i += 32) x[i] *= scal;
    __syncwarp();
    if (lane == 0) {
        x[j] = beta;
        tau[j] = (beta - alpha) / beta;
    }
    __syncwarp();
}

// Apply H = I - t v v^T (v = column j below the diagonal, v_j = 1) to up to NC
// columns c0, c0+cs, ... (< Cn) over rows [j, R). Dots reduced together.
template <int NC>
__device__ __forceinline__ void qr_apply_cols(double* A, int ld, int R, int j, double t, int c0, int cs,
                                              int Cn, int lane) {
    const double* v = A + (size_t)j * ld;
    double* y[NC];
    bool on[NC];
    double d[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        const int c = c0 + q * cs;
        on[q] = c < Cn;
        y[q] = A + (size_t)(on[q] ? c : c0) * ld;
        d[q] = (lane == 0 && on[q]) ? y[q][j] : 0.0;
    }
    for (int i = j + 1 + lane; i < R; i += 32) {
        const double vi = v[i];
#pragma unroll
        for (int q = 0; q < NC; ++q)
            if (on[q]) d[q] = fma(vi, y[q][i], d[q]);
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) d[q] = warp_sum(d[q]) * t;
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < NC; ++q)
            if (on[q]) y[q][j] -= d[q];
    }
    for (int i = j + 1 + lane; i < R; i += 32) {
        const double vi = v[i];
#pragma unroll
        for (int q = 0; q < NC; ++q)
            if (on[q]) y[q][i] = fma(-d[q], vi, y[q][i]);
    }
}

// First column index >= lo owned by warp w (columns are dealt round-robin).
__device__ __forceinline__ int qr_first_owned(int lo, int w, int nw) {
    return lo + ((w - lo) % nw + nw) % nw;
}

// In-place Householder QR (dgeqr2) of an R x Cn column-major block, R >= Cn.
// On return the upper triangle holds R (LAPACK signs), the strict lower part
// the reflector vectors, tau[0..Cn) the scalars. Ends with __syncthreads.
__device__ void qr_block_factor(double* A, int ld, int R, int Cn, double* tau) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (warp == 0) qr_make_reflector(A, ld, R, 0, tau, lane);
    for (int j = 0; j < Cn; ++j) {
        __syncthreads();
        const double tj = tau[j];
        int c = qr_first_owned(j + 1, warp, nw);
        if (c == j + 1 && c < Cn) {  // look-ahead: finish column j+1, build reflector j+1
            if (tj != 0.0) qr_apply_cols<1>(A, ld, R, j, tj, c, nw, Cn, lane);
            __syncwarp();
            qr_make_reflector(A, ld, R, j + 1, tau, lane);
            c += nw;
        }
        if (tj != 0.0) {
            for (; c < Cn; c += 4 * nw) qr_apply_cols<4>(A, ld, R, j, tj, c, nw, Cn, lane);
        }
    }
    __syncthreads();
}

// Column c of the explicit Q from its reflector (dorg2r's per-column step).
__device__ __forceinline__ void qr_finalize_col(double* A, int ld, int R, int c, double t, int lane) {
    double* x = A + (size_t)c * ld;
    for (int i = lane; i < c; i += 32) x[i] = 0.0;
    for (int i = c + 1 + lane; i < R; i += 32) x[i] *= -t;
    if (lane == 0) x[c] = 1.0 - t;
    __syncwarp();
}

// In-place explicit Q (dorg2r): A holds reflectors from qr_block_factor.
// Q = H_0 H_1 ... H_{Cn-1} [I; 0]. One __syncthreads per step; finalising
// column j+1 is folded into step j (its owner does it just before applying
// H_j to it). Ends with __syncthreads.
__device__ void qr_block_form_q(double* A, int ld, int R, int Cn, const double* tau) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int j = Cn - 1; j >= 0; --j) {
        __syncthreads();
        const double tj = tau[j];
        int c = qr_first_owned(j + 1, warp, nw);
        if (c == j + 1 && c < Cn) {
            qr_finalize_col(A, ld, R, c, tau[c], lane);
            if (tj != 0.0) qr_apply_cols<1>(A, ld, R, j, tj, c, nw, Cn, lane);
            c += nw;
        }
        if (tj != 0.0) {
            for (; c < Cn; c += 4 * nw) qr_apply_cols<4>(A, ld, R, j, tj, c, nw, Cn, lane);
        }
    }
    __syncthreads();
    if (warp == 0) qr_finalize_col(A, ld, R, 0, tau[0], lane);
    __syncthreads();
}

// Reference sign convention (dense.hpp:127-132): flip row j of R and column j
// of Q when R(j,j) < 0. Applied at the root only; here d_j in {+1,-1}.
__device__ __forceinline__ double qr_sign(double rjj) { return rjj < 0.0 ? -1.0 : 1.0; }

struct LeafArgs {
    const double* T;   // m x ldt row-major input sketch
    int64_t ldt;
    double* Qout;      // explicit leaf Q rows (row-major, ldq); may alias T
    int64_t ldq;
    const int64_t* row0;  // leaf row offsets
    const int* rows;      // leaf row counts
    int k;
    double* R;         // P x (k x ldr) row-major R factors
    int ldr;
    double* scratch;   // global fallback: per-leaf column-major block (row0[i]*k offset)
    int is_root;       // P == 1: this leaf is the tree root (apply signs)
};

// One CTA per leaf.
template <bool SMEM>
__global__ void __launch_bounds__(kQrThreads, 1) tsqr_leaf_kernel(LeafArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int leaf = blockIdx.x;
    const int R = a.rows[leaf], k = a.k;
    const int64_t r0 = a.row0[leaf];
    const int ld = R | 1;
    double* tau = sm;  // k (+pad)
    double* sgn = sm + ((k + 1) & ~1);
    double* A = SMEM ? sgn + ((k + 1) & ~1) : a.scratch + (r0 + leaf) * k;  // ld <= R+1 per leaf
    // load (row-major global -> column-major block)
    for (int e = threadIdx.x; e < R * k; e += blockDim.x) {
        const int i = e / k, c = e - i * k;
        A[(size_t)c * ld + i] = a.T[(r0 + i) * a.ldt + c];
    }
    __syncthreads();
    qr_block_factor(A, ld, R, k, tau);
    // R out (row-major k x k, zeros below the diagonal), sign-fixed at the root
    for (int c = threadIdx.x; c < k; c += blockDim.x) sgn[c] = a.is_root ? qr_sign(A[(size_t)c * ld + c]) : 1.0;
    __syncthreads();
    double* Rl = a.R + (int64_t)leaf * k * a.ldr;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int i = e / k, c = e % k;
        Rl[(int64_t)i * a.ldr + c] = c >= i ? sgn[i] * A[(size_t)c * ld + i] : 0.0;
    }
    qr_block_form_q(A, ld, R, k, tau);
    for (int e = threadIdx.x; e < R * k; e += blockDim.x) {
        const int i = e / k, c = e - i * k;
        a.Qout[(r0 + i) * a.ldq + c] = sgn[c] * A[(size_t)c * ld + i];
    }
}

struct NodeArgs {
    const double* Rin;  // nin x (k x ldr)
    int nin;
    double* Rout;       // nout x (k x ldr)
    double* Qnode;      // nout x (2k x ldq) explicit node Q (pass-through nodes: [I; 0])
    int ldq;
    int k;
    int ldr;
    double* scratch;    // global fallback: nout x (2k x k) column-major
    int is_root;
};

// One CTA per output node: QR of [R_{2i}; R_{2i+1}].
template <bool SMEM>
__global__ void __launch_bounds__(kQrThreads, 1) tsqr_node_kernel(NodeArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int node = blockIdx.x, k = a.k, R = 2 * k;
    const int ld = R | 1;
    double* tau = sm;
    double* sgn = sm + ((k + 1) & ~1);
    double* A = SMEM ? sgn + ((k + 1) & ~1) : a.scratch + (int64_t)node * (ld * k + 1);
    const double* Ra = a.Rin + (int64_t)(2 * node) * k * a.ldr;
    double* Qn = a.Qnode + (int64_t)node * R * a.ldq;
    double* Ro = a.Rout + (int64_t)node * k * a.ldr;
    if (2 * node + 1 >= a.nin) {  // pass-through: R up, Q = [I; 0]
        for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
            const int i = e / k, c = e % k;
            Ro[(int64_t)i * a.ldr + c] = Ra[(int64_t)i * a.ldr + c];
        }
        for (int e = threadIdx.x; e < R * k; e += blockDim.x) {
            const int i = e / k, c = e % k;
            Qn[(int64_t)i * a.ldq + c] = (i == c) ? 1.0 : 0.0;
        }
        return;
    }
    const double* Rb = Ra + (int64_t)k * a.ldr;
    for (int e = threadIdx.x; e < R * k; e += blockDim.x) {
        const int i = e / k, c = e % k;
        const double* src = i < k ? Ra + (int64_t)i * a.ldr : Rb + (int64_t)(i - k) * a.ldr;
        const int ii = i < k ? i : i - k;
        A[(size_t)c * ld + i] = c >= ii ? src[c] : 0.0;
    }
    __syncthreads();
    qr_block_factor(A, ld, R, k, tau);
    for (int c = threadIdx.x; c < k; c += blockDim.x) sgn[c] = a.is_root ? qr_sign(A[(size_t)c * ld + c]) : 1.0;
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int i = e / k, c = e % k;
        Ro[(int64_t)i * a.ldr + c] = c >= i ? sgn[i] * A[(size_t)c * ld + i] : 0.0;
    }
    qr_block_form_q(A, ld, R, k, tau);
    for (int e = threadIdx.x; e < R * k; e += blockDim.x) {
        const int i = e / k, c = e % k;
        Qn[(int64_t)i * a.ldq + c] = sgn[c] * A[(size_t)c * ld + i];
    }
}

}  // namespace sorsvd_dev
