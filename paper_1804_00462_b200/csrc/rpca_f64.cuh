// K7/K8: fused inexact-ALM RPCA update.
//
// One sweep over the m x n data per ALM iteration. For every entry the
// low-rank value l_ij = sum_r U_ir * S_{1/mu}(z_r) * V_jr is produced on the
// FP64 tensor core (DMMA m8n8k4 fragments of the rank-ell outer product, the
// factors read straight from L2) and consumed in registers, so L is never
// materialised:
//     s'  = S_{lambda/mu}(d - l + y/mu)
//     y'  = y + mu (d - l - s')
//     w'  = d - s' + y'/mu'   (next iteration's SOR-SVD input)
//     res += (d - l - s')^2   (stopping test)
// Traffic: read D, Y; write S, Y, W (40 B/entry). D and Y are loaded before the
// rank-ell product so their latency hides behind it. The residual is reduced
// deterministically (per-block partials, fixed-order final sum).
#pragma once
#include "common.cuh"

namespace sorsvd_dev {

constexpr int kRpcaThreads = 256;  // 8 warps -> 64 x 64 tile (warps 4 x 2, 16 x 32 each)

struct RpcaArgs {
    const double* D;
    int64_t ldd;
    double* S;       // m x ldx
    double* Y;
    double* W;       // next SOR-SVD input (may be null in the final L pass)
    double* L;       // final pass only: dense L output (ldl)
    int64_t ldx;
    int64_t ldl;
    const double* U; // m x ldu (left factors from SOR-SVD)
    int64_t ldu;
    const double* V; // n x ldv
    int64_t ldv;
    const double* sig;  // ell singular values (unshrunk)
    int64_t m, n;
    int k;
    double mu, mu_next, eps;  // eps = lambda / mu
    double* partial;          // per-block residual^2 partials
    unsigned int* nnz_partial;  // per-block count of nonzeros of the new S (telemetry), or null
    int mode;                 // 0 = ALM update, 1 = write L only
    const int* pred;          // optional: no-op when *pred == pred_skip (iteration after convergence)
    int pred_skip;
};

__global__ void __launch_bounds__(kRpcaThreads, 2) rpca_update_kernel(RpcaArgs a) {
    if (pred_off(a.pred, a.pred_skip)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t i0 = (int64_t)blockIdx.y * 64 + (warp >> 1) * 16;
    const int64_t j0 = (int64_t)blockIdx.x * 64 + (warp & 1) * 32;
    const double inv = 1.0 / a.mu;
    double acc[2][4][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    // each lane's two columns are adjacent: 16-byte loads / stores of D, Y, S, W when the
    // rows are 16-byte aligned (same arithmetic as the element path)
    const bool vec = a.mode == 0 && ((a.ldd | a.ldx) & 1) == 0 &&
                     ((reinterpret_cast<uintptr_t>(a.D) | reinterpret_cast<uintptr_t>(a.S) |
                       reinterpret_cast<uintptr_t>(a.Y) | reinterpret_cast<uintptr_t>(a.W)) & 15) == 0;
    // D (into registers) and Y (cp.async into this thread's shared-memory slots) are
    // issued before the factor loop, so their DRAM latency overlaps the L2-resident U/V
    // fragment loads and the DMMA chain instead of following it. Registers for both
    // would cost occupancy (142 regs -> 1 block per SM); this split keeps 2.
    double2 dpre[2][4];
    __shared__ double2 ysm[8][kRpcaThreads];
    if (vec) {
#pragma unroll
        for (int fm = 0; fm < 2; ++fm) {
            const int64_t i = i0 + fm * 8 + g;
#pragma unroll
            for (int fn = 0; fn < 4; ++fn) {
                const int64_t j = j0 + fn * 8 + 2 * t4;
                const bool ok = i < a.m && j + 1 < a.n;
                dpre[fm][fn] = ok ? __ldcs(reinterpret_cast<const double2*>(a.D + i * a.ldd + j))
                                  : make_double2(0.0, 0.0);
                cp_async16(&ysm[fm * 4 + fn][threadIdx.x], ok ? a.Y + i * a.ldx + j : a.Y, ok ? 16 : 0);
            }
        }
        cp_async_commit();
    }
    for (int kk0 = 0; kk0 < a.k; kk0 += 4) {
        const int kk = kk0 + t4;
        const double z = kk < a.k ? fmax(a.sig[kk] - inv, 0.0) : 0.0;
        double af[2], bf[4];
#pragma unroll
        for (int fm = 0; fm < 2; ++fm) {
            const int64_t i = i0 + fm * 8 + g;
            af[fm] = (kk < a.k && i < a.m) ? a.U[i * a.ldu + kk] * z : 0.0;
        }
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
            const int64_t j = j0 + fn * 8 + g;
            bf[fn] = (kk < a.k && j < a.n) ? a.V[j * a.ldv + kk] : 0.0;
        }
#pragma unroll
        for (int fm = 0; fm < 2; ++fm)
#pragma unroll
            for (int fn = 0; fn < 4; ++fn) dmma884(acc[fm][fn][0], acc[fm][fn][1], af[fm], bf[fn]);
    }
    double res = 0.0;
    unsigned int cnt = 0;  // nonzeros of the new S in this thread's entries
    if (vec) {
        cp_async_wait<0>();  // own slots only: no block barrier needed
#pragma unroll
        for (int fm = 0; fm < 2; ++fm) {
            const int64_t i = i0 + fm * 8 + g;
            if (i >= a.m) continue;
#pragma unroll
            for (int fn = 0; fn < 4; ++fn) {
                const int64_t j = j0 + fn * 8 + 2 * t4;
                if (j + 1 >= a.n) {  // ragged right edge: the element path
                    for (int h = 0; h < 2 && j + h < a.n; ++h) {
                        const double l = acc[fm][fn][h];
                        const double d = a.D[i * a.ldd + j + h];
                        const double y = a.Y[i * a.ldx + j + h];
                        const double t = d - l + y / a.mu;
                        const double sh = fabs(t) - a.eps;
                        const double sv = sh > 0.0 ? (t > 0.0 ? sh : -sh) : 0.0;
                        const double r = d - l - sv;
                        const double yn = y + a.mu * r;
                        a.S[i * a.ldx + j + h] = sv;
                        a.Y[i * a.ldx + j + h] = yn;
                        if (a.W) a.W[i * a.ldx + j + h] = d - sv + yn / a.mu_next;
                        res = fma(r, r, res);
                        cnt += sv != 0.0;
                    }
                    continue;
                }
                const double2 d2 = dpre[fm][fn];
                const double2 y2 = ysm[fm * 4 + fn][threadIdx.x];
                double sv[2], yn[2], wv[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double l = acc[fm][fn][h];
                    const double d = h ? d2.y : d2.x;
                    const double y = h ? y2.y : y2.x;
                    const double t = d - l + y / a.mu;
                    const double sh = fabs(t) - a.eps;
                    sv[h] = sh > 0.0 ? (t > 0.0 ? sh : -sh) : 0.0;
                    const double r = d - l - sv[h];
                    yn[h] = y + a.mu * r;
                    wv[h] = d - sv[h] + yn[h] / a.mu_next;
                    res = fma(r, r, res);
                    cnt += sv[h] != 0.0;
                }
                __stcs(reinterpret_cast<double2*>(a.S + i * a.ldx + j), make_double2(sv[0], sv[1]));
                __stcs(reinterpret_cast<double2*>(a.Y + i * a.ldx + j), make_double2(yn[0], yn[1]));
                // W is the next iteration's SOR-SVD input, read by its 2q+3 passes: a normal
                // store (L2-resident when it fits); D, Y, S are streamed
                if (a.W) *reinterpret_cast<double2*>(a.W + i * a.ldx + j) = make_double2(wv[0], wv[1]);
            }
        }
    }
#pragma unroll
    for (int fm = 0; fm < 2; ++fm) {
        if (vec) break;
        const int64_t i = i0 + fm * 8 + g;
        if (i >= a.m) continue;
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t j = j0 + fn * 8 + 2 * t4 + h;
                if (j >= a.n) continue;
                const double l = acc[fm][fn][h];
                if (a.mode == 1) {
                    a.L[i * a.ldl + j] = l;
                    continue;
                }
                const double d = a.D[i * a.ldd + j];
                const double y = a.Y[i * a.ldx + j];
                const double t = d - l + y / a.mu;
                const double sh = fabs(t) - a.eps;
                const double s = sh > 0.0 ? (t > 0.0 ? sh : -sh) : 0.0;
                const double r = d - l - s;
                const double yn = y + a.mu * r;
                a.S[i * a.ldx + j] = s;
                a.Y[i * a.ldx + j] = yn;
                if (a.W) a.W[i * a.ldx + j] = d - s + yn / a.mu_next;
                res = fma(r, r, res);
                cnt += s != 0.0;
            }
        }
    }
    if (a.mode == 1) return;
    __shared__ double red[kRpcaThreads / 32];
    __shared__ unsigned int redc[kRpcaThreads / 32];
    res = warp_sum(res);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) {
        red[warp] = res;
        redc[warp] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        unsigned int tc = 0;
        for (int w = 0; w < kRpcaThreads / 32; ++w) {
            t += red[w];
            tc += redc[w];
        }
        a.partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
        if (a.nnz_partial) a.nnz_partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = tc;
    }
}

// Deterministic single-block reduction of partials: out[0] = sum, (sqrt into out[1]);
// with integer count partials c: out[2] = their sum (exact in a double below 2^53).
__global__ void sum_partials_kernel(const double* __restrict__ p, int64_t n, double* out, const int* pred = nullptr,
                                    int pred_skip = 0, const unsigned int* __restrict__ c = nullptr) {
    if (pred_off(pred, pred_skip)) return;
    __shared__ double red[32];
    __shared__ unsigned long long redc[32];
    double t = 0.0;
    unsigned long long tc = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        t += p[i];
        if (c) tc += c[i];
    }
    t = warp_sum(t);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tc += __shfl_xor_sync(0xffffffffu, tc, o);
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5] = t;
        redc[threadIdx.x >> 5] = tc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        unsigned long long sc = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            s += red[w];
            sc += redc[w];
        }
        out[0] = s;
        out[1] = sqrt(s);
        if (c) out[2] = (double)sc;
    }
}

// Stopping test of iteration `it` on the device, so that the
// host can enqueue several iterations ahead: st[0] = done flag (sticky), st[1]
// = iterations executed, st[2] = error flag; rel[0] = this iteration's
// ||D - L - S||_F / ||D||_F. Predicated like the iteration itself.
// tele (4 doubles, may be null) = this iteration's telemetry row: mu, rel_error,
// rank_l (shrunk sigma > 1e-8 of the largest) and nnz_s (tot[2]).
__global__ void rpca_check_kernel(const double* __restrict__ tot, double dnorm, double tol, int it, int* st,
                                  double* rel, const int* pred, int pred_skip, double* tele = nullptr,
                                  const double* __restrict__ sig = nullptr, int ell = 0, double mu = 0.0) {
    if (pred_off(pred, pred_skip)) return;
    const double r = sqrt(tot[0]) / dnorm;
    rel[0] = r;
    st[1] = it + 1;
    if (tele) {
        const double z0 = fmax(sig[0] - 1.0 / mu, 0.0);
        int rank = 0;
        for (int j = 0; j < ell; ++j) rank += fmax(sig[j] - 1.0 / mu, 0.0) > 1e-8 * z0;
        tele[0] = mu;
        tele[1] = r;
        tele[2] = (double)rank;
        tele[3] = tot[2];
    }
    if (!isfinite(r)) {
        st[2] = 1;
        st[0] = 1;
    } else if (r < tol) {
        st[0] = 1;
    }
}

// Per-block partial sums of squares of a row-major m x n matrix (||D||_F).
__global__ void sumsq_partials_kernel(const double* __restrict__ x, int64_t m, int64_t n, int64_t ld,
                                      double* partial) {
    double t = 0.0;
    const int64_t total = m * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e - i * n;
        const double v = x[i * ld + j];
        t = fma(v, v, t);
    }
    __shared__ double red[32];
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        partial[blockIdx.x] = s;
    }
}

// Per-block nonzero counts (||S||_0).
__global__ void nnz_partials_kernel(const double* __restrict__ x, int64_t m, int64_t n, int64_t ld,
                                    unsigned long long* partial) {
    unsigned long long c = 0;
    const int64_t total = m * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e - i * n;
        c += x[i * ld + j] != 0.0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ unsigned long long red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        partial[blockIdx.x] = s;
    }
}

// ---- sigma_1 by repeated squaring of the small Gram matrix (mu0 estimate) ----
// *mx = max |X| over rows x cols (non-negative doubles order like their bits);
// *mx must be 0 on entry. Grid-stride, one atomic per warp.
__global__ void maxabs_kernel(const double* __restrict__ X, int rows, int cols, int ld,
                              unsigned long long* __restrict__ mx) {
    double m = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
        const int i = e / cols, j = e - i * cols;
        m = fmax(m, fabs(X[(size_t)i * ld + j]));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(mx, (unsigned long long)__double_as_longlong(m));
}

// X *= 1 / *mx, then *mx = 0 for the next use (the last block to finish resets it
// is not needed: each use gets its own slot).
__global__ void scale_by_kernel(double* __restrict__ X, int rows, int cols, int ld,
                                const unsigned long long* __restrict__ mx) {
    const double m = __longlong_as_double((long long)*mx);
    const double s = m > 0.0 ? 1.0 / m : 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
        const int i = e / cols, j = e - i * cols;
        X[(size_t)i * ld + j] *= s;
    }
}

// At[j][i] = A[i][j] for i < m, j < n (At row pitch ldt).
__global__ void transpose_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                 double* __restrict__ At, int64_t ldt) {
    __shared__ double tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + r, j = j0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < m && j < n) ? A[i * lda + j] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t j = j0 + r, i = i0 + threadIdx.x;
        if (j < n && i < m) At[j * ldt + i] = tile[threadIdx.x][r];
    }
}

}  // namespace sorsvd_dev

namespace sorsvd_dev {

// approx_error(a, x, frobenius) (sketch.hpp:168-172): ||A - U diag(sigma) V^T||_F
// in ONE pass over A, without forming the m x n reconstruction (the reference
// materialises reconstruct(x) with a dgemm and then takes norm()). Each 64 x 64
// tile of U diag(sigma) V^T is built on DMMA fragments (same layout as
// rpca_update_kernel), subtracted from A in registers and squared; per-block
// partial sums, reduced in fixed order. A may be FP32-stored (widened).
template <typename AT>
__global__ void __launch_bounds__(kRpcaThreads) approx_err_kernel(const AT* __restrict__ A, int64_t lda,
                                                                 const double* __restrict__ U, int64_t ldu,
                                                                 const double* __restrict__ sig,
                                                                 const double* __restrict__ V, int64_t ldv,
                                                                 int64_t m, int64_t n, int k, double* partial) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t i0 = (int64_t)blockIdx.y * 64 + (warp >> 1) * 16;
    const int64_t j0 = (int64_t)blockIdx.x * 64 + (warp & 1) * 32;
    double acc[2][4][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    for (int kk0 = 0; kk0 < k; kk0 += 4) {
        const int kk = kk0 + t4;
        const double z = kk < k ? sig[kk] : 0.0;
        double af[2], bf[4];
#pragma unroll
        for (int fm = 0; fm < 2; ++fm) {
            const int64_t i = i0 + fm * 8 + g;
            af[fm] = (kk < k && i < m) ? U[i * ldu + kk] * z : 0.0;
        }
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
            const int64_t j = j0 + fn * 8 + g;
            bf[fn] = (kk < k && j < n) ? V[j * ldv + kk] : 0.0;
        }
#pragma unroll
        for (int fm = 0; fm < 2; ++fm)
#pragma unroll
            for (int fn = 0; fn < 4; ++fn) dmma884(acc[fm][fn][0], acc[fm][fn][1], af[fm], bf[fn]);
    }
    double res = 0.0;
#pragma unroll
    for (int fm = 0; fm < 2; ++fm) {
        const int64_t i = i0 + fm * 8 + g;
        if (i >= m) continue;
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t j = j0 + fn * 8 + 2 * t4 + h;
                if (j >= n) continue;
                const double r = (double)A[i * lda + j] - acc[fm][fn][h];
                res = fma(r, r, res);
            }
        }
    }
    __shared__ double red[kRpcaThreads / 32];
    res = warp_sum(res);
    if (lane == 0) red[warp] = res;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kRpcaThreads / 32; ++w) t += red[w];
        partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

// E = A - U diag(sigma) V^T as a dense m x n matrix (reconstruct + subtract, sketch.hpp:163-172):
// the analysis side's spectral-norm error needs the matrix itself. 16 x 16 outputs per block,
// the factor rows staged through shared memory in 16-deep slices.
template <typename AT>
__global__ void __launch_bounds__(256) residual_kernel(const AT* __restrict__ A, int64_t lda, const double* __restrict__ U,
                                                       int64_t ldu, const double* __restrict__ sg,
                                                       const double* __restrict__ V, int64_t ldv, int64_t m, int64_t n,
                                                       int k, double* __restrict__ E, int64_t lde) {
    __shared__ double su[16][17], sv[16][17];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i = (int64_t)blockIdx.y * 16 + ty, j = (int64_t)blockIdx.x * 16 + tx;
    double acc = 0.0;
    for (int t0 = 0; t0 < k; t0 += 16) {
        const int64_t iu = (int64_t)blockIdx.y * 16 + ty, jv = (int64_t)blockIdx.x * 16 + ty;
        const int t = t0 + tx;
        su[ty][tx] = (iu < m && t < k) ? U[iu * ldu + t] * sg[t] : 0.0;
        sv[ty][tx] = (jv < n && t < k) ? V[jv * ldv + t] : 0.0;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 16; ++q) acc = fma(su[ty][q], sv[tx][q], acc);
        __syncthreads();
    }
    if (i < m && j < n) E[i * lde + j] = (double)A[i * lda + j] - acc;
}

}  // namespace sorsvd_dev
