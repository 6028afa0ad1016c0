// K3 (v2): cluster-distributed Householder QR of one tall block per cluster.
//
// Replaces the LAPACK pair behind thin_qr (dense.hpp:114-134: dgeqrf + dorgqr
// + diag(R) >= 0 at :127-132) for the sketches T1 (m x k) and T2 (n x k)
// (sketch.hpp:98-99), and serves as the leaf / node kernel of the TSQR tree
// when a sketch is larger than one cluster can hold.
//
// A block of `rows` x k is spread by rows over the C CTAs of a thread-block
// cluster (C <= 16, non-portable size), each CTA keeping its rows
// column-major in shared memory (<= ~210 KB). Reflector j needs, over all
// rows, ||x_{j+1:}||^2, alpha = x_j, the row-j entries and the dots
// s_c = sum_{i>j} x_i A(i,c); with v = [1; x/(alpha-beta)] every
// d_c = A(j,c) + s_c/(alpha-beta), so ONE cluster reduction per reflector
// (partials in shared memory, double-buffered, summed in fixed CTA order over
// DSMEM -> identical on every CTA, deterministic) gives beta, tau and all
// d_c. The explicit Q is then formed in place (dorg2r order, one reduction
// per reflector), the root applies the reference sign convention, and the
// rows go back to global memory. No tree at all when the whole sketch fits in
// one cluster (C1, C2, C4: up to 16 x 210 KB).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace sorsvd_dev {

namespace cg = cooperative_groups;

constexpr int kCqrThreads = 512;
// trailing columns a warp updates per sweep of its rows in the factor's fused pass: the
// reflector x and the next column xn are read once per group (shared-memory traffic)
constexpr int kCqrNG = 4;
constexpr int kCqrSmemBudget = 212 * 1024;

struct CqrArgs {
    const double* in;     // row-major input, block b starts at in + row0[b]*ldi
    int64_t ldi;
    double* qout;         // explicit Q rows (row-major), same row indexing; may alias in
    int64_t ldq;
    const int64_t* row0;  // per block
    const int* rows;      // per block
    int k;
    double* R;            // per block k x ldr (row-major), zeros below the diagonal
    int ldr;
    int root_sign;        // apply diag(R) >= 0 (dense.hpp:127-132)
    const int* pred;      // optional: no-op when *pred == pred_skip (CholeskyQR2 accepted)
    int pred_skip;
    // compact-WY mode (cqr_kernel only): skip the in-kernel form-Q; write the
    // unit-lower Householder vectors V into qout, tau and the root signs out.
    // Q is then formed by wy_tfactor_kernel + two DMMA GEMMs (sorsvd.cu).
    int wy;
    double* tau_out;
    double* sgn_out;
    long long* prof;  // optional (tools): per-step clock64 stamps of CTA 0 / warp 0 / lane 0
};

// shared-memory layout (doubles): A[ld*k] | red[2*RW] | S[RW] | tau[k] | sgn[k]
__host__ __device__ inline int cqr_rw(int k) { return 2 * k + 4; }
__host__ __device__ inline size_t cqr_smem_bytes(int Rb, int k) {
    const int ld = Rb | 1;
    return ((size_t)ld * k + 3 * (size_t)cqr_rw(k) + 2 * (size_t)k + 8) * sizeof(double);
}

// Process up to 4 owned columns c0, c0+cs, ... of a warp together: the
// per-column shuffle reductions overlap and x / v are read once per row.
template <int NC>
struct ColGroup {
    double* y[NC];
    bool on[NC];
    __device__ ColGroup(double* A, int ld, int c0, int cs, int cend) {
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const int c = c0 + q * cs;
            on[q] = c < cend;
            y[q] = A + (size_t)(on[q] ? c : c0) * ld;
        }
    }
};

__global__ void __launch_bounds__(kCqrThreads, 1) cqr_kernel(CqrArgs a) {
    if (pred_off(a.pred, a.pred_skip)) return;  // uniform over the cluster
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks();
    const int r = (int)cl.block_rank();
    const int b = blockIdx.x / C;
    const int rows = a.rows[b];
    const int64_t row0 = a.row0[b];
    const int k = a.k;
    const int Rb = (rows + C - 1) / C;
    const int lr0 = r * Rb;
    const int nr = max(0, min(Rb, rows - lr0));
    const int ld = Rb | 1;
    const int RW = cqr_rw(k);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;

    extern __shared__ __align__(16) double sm[];
    double* A = sm;
    double* red = A + (size_t)ld * k;
    double* S = red + 2 * RW;
    double* tau = S + RW;
    double* sgn = tau + k;
    __shared__ double sclA[512];   // 1/(alpha-beta) per reflector (deferred column scaling)
    __shared__ double betaA[512];  // R(j,j) per reflector
    __shared__ double* peers[16];

    for (int e = tid; e < nr * k; e += blockDim.x) {
        const int i = e / k, c = e - i * k;
        A[(size_t)c * ld + i] = a.in[(row0 + lr0 + i) * a.ldi + c];
    }
    if (tid < C) peers[tid] = cl.map_shared_rank(red, tid);
    __syncthreads();

    // fixed-order cluster sum of red[off + idx] over the C CTAs (loads issued back to back)
    auto csum = [&](int off, int idx) {
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = q < C ? peers[q][off + idx] : 0.0;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) s += v[q];
        return s;
    };
    auto first_owned = [&](int lo) { return lo + ((warp - lo) % nw + nw) % nw; };

    // ------------------------------------------------------------ factor --
    // Partial payload for reflector j (nt = k-j-1 trailing columns):
    //   P[0] = sum_{i>j} x_i^2, P[1] = A(j,j), P[2+t] = sum_{i>j} x_i A(i,j+1+t),
    //   P[2+nt+t] = A(j, j+1+t)   (row j entries come from its owner CTA, 0 elsewhere)
    // Step j's fused pass updates the trailing columns with H_j and at the same
    // time accumulates step j+1's payload against the (already updated) column j+1.
    {
        double* P = red;  // prologue: payload of reflector 0
        const int nt = k - 1;
        const int i0 = max(0, 1 - lr0);
        const int jo = -lr0;
        const bool owner = jo >= 0 && jo < nr;
        const double* x = A;
        for (int vc = warp; vc <= nt; vc += nw) {
            const double* y = A + (size_t)vc * ld;
            double s = 0.0;
            for (int i = i0 + lane; i < nr; i += 32) s = fma(x[i], y[i], s);
            s = warp_sum(s);
            if (lane == 0) P[vc == 0 ? 0 : 1 + vc] = s;
        }
        for (int c = tid; c <= nt; c += blockDim.x) {
            const double v = owner ? A[(size_t)c * ld + jo] : 0.0;
            if (c == 0) P[1] = v;
            else P[1 + nt + c] = v;
        }
    }
    for (int j = 0; j < k; ++j) {
        double* P = red + (j & 1) * RW;
        double* Pn = red + ((j + 1) & 1) * RW;
        const int nt = k - j - 1;
        const int i0 = max(0, j + 1 - lr0);  // local rows with global index > j
        const int jo = j - lr0;
        const bool owner = jo >= 0 && jo < nr;
        const bool prof = a.prof && r == 0 && tid == 0 && b == 0;
        if (prof) a.prof[j * 6 + 0] = clock64();
        cl.sync();
        if (prof) a.prof[j * 6 + 1] = clock64();
        for (int idx = tid; idx < 2 + 2 * nt; idx += blockDim.x) S[idx] = csum((int)(P - red), idx);
        __syncthreads();
        if (prof) a.prof[j * 6 + 2] = clock64();
        const double ss = S[0], alpha = S[1];
        double t = 0.0, beta = alpha, scal = 0.0;
        if (ss != 0.0) {
            beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
            t = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        if (tid == 0) {
            tau[j] = t;
            sgn[j] = (a.root_sign && beta < 0.0) ? -1.0 : 1.0;
            sclA[j] = scal;
            betaA[j] = beta;
        }
        const double* x = A + (size_t)j * ld;  // reflector j, still unscaled (v_i = scal * x_i)
        // deferred: finish column j-1 (scale into v, diagonal <- beta); nobody reads it this step
        if (j >= 1 && warp == (j - 1) % nw) {
            double* xm = A + (size_t)(j - 1) * ld;
            const double sm1 = sclA[j - 1];
            for (int i = max(0, j - lr0) + lane; i < nr; i += 32) xm[i] *= sm1;
            const int jm = j - 1 - lr0;
            if (lane == 0 && jm >= 0 && jm < nr) xm[jm] = betaA[j - 1];
        }
        // column j+1 first (its owner): apply H_j, then the next reflector's norm and alpha
        const int i0n = max(0, j + 2 - lr0);
        const int jon = j + 1 - lr0;
        const bool ownern = jon >= 0 && jon < nr;
        if (nt > 0 && warp == (j + 1) % nw) {
            double* y = A + (size_t)(j + 1) * ld;
            const double d = (S[2 + nt] + scal * S[2]) * t;
            if (t != 0.0) {
                for (int i = i0 + lane; i < nr; i += 32) y[i] = fma(-d * scal, x[i], y[i]);
                if (owner && lane == 0) y[jo] -= d;
            }
            __syncwarp();
            double s = 0.0;
            for (int i = i0n + lane; i < nr; i += 32) s = fma(y[i], y[i], s);
            s = warp_sum(s);
            if (lane == 0) {
                Pn[0] = s;
                Pn[1] = ownern ? y[jon] : 0.0;
            }
        }
        __syncthreads();
        if (prof) a.prof[j * 6 + 3] = clock64();
        // fused pass over the remaining trailing columns c > j+1
        if (nt > 1) {
            const double* xn = A + (size_t)(j + 1) * ld;  // next reflector (updated, unscaled)
            const int ntn = nt - 1;
            for (int c0 = first_owned(j + 2); c0 < k; c0 += kCqrNG * nw) {
                ColGroup<kCqrNG> g(A, ld, c0, nw, k);
                double dd[kCqrNG], sn[kCqrNG];
#pragma unroll
                for (int q = 0; q < kCqrNG; ++q) {
                    const int c = c0 + q * nw;
                    dd[q] = g.on[q] ? (S[2 + nt + (c - j - 1)] + scal * S[2 + (c - j - 1)]) * t : 0.0;
                    sn[q] = 0.0;
                }
                if (owner && lane == 0) {
#pragma unroll
                    for (int q = 0; q < kCqrNG; ++q)
                        if (g.on[q]) g.y[q][jo] -= dd[q];
                }
                // all loads of a row before any store: the four column pointers
                // may alias as far as the compiler knows, and a load->FMA->store
                // chain per column serialises on the shared-memory latency
#pragma unroll 2
                for (int i = i0 + lane; i < nr; i += 32) {
                    const double vi = scal * x[i];
                    const double xi = (i >= i0n) ? xn[i] : 0.0;
                    double yv[kCqrNG];
#pragma unroll
                    for (int q = 0; q < kCqrNG; ++q) yv[q] = g.y[q][i];  // off columns alias column c0 (readable)
#pragma unroll
                    for (int q = 0; q < kCqrNG; ++q) {
                        yv[q] = fma(-dd[q], vi, yv[q]);
                        sn[q] = fma(xi, yv[q], sn[q]);
                    }
#pragma unroll
                    for (int q = 0; q < kCqrNG; ++q)
                        if (g.on[q]) g.y[q][i] = yv[q];
                }
#pragma unroll
                for (int q = 0; q < kCqrNG; ++q) sn[q] = warp_sum(sn[q]);
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int q = 0; q < kCqrNG; ++q) {
                        if (g.on[q]) {
                            const int c = c0 + q * nw;
                            Pn[2 + (c - j - 2)] = sn[q];
                            Pn[2 + ntn + (c - j - 2)] = ownern ? g.y[q][jon] : 0.0;
                        }
                    }
                }
            }
        }
        if (prof) a.prof[j * 6 + 4] = clock64();
        // (no barrier here: the next step starts with cl.sync)
    }
    __syncthreads();
    if (warp == (k - 1) % nw) {  // deferred finish of the last reflector column
        double* xm = A + (size_t)(k - 1) * ld;
        const double sm1 = sclA[k - 1];
        for (int i = max(0, k - lr0) + lane; i < nr; i += 32) xm[i] *= sm1;
        const int jm = k - 1 - lr0;
        if (lane == 0 && jm >= 0 && jm < nr) xm[jm] = betaA[k - 1];
    }
    __syncthreads();

    // R (owners of rows < k), sign-fixed at the root
    double* Rb_out = a.R + (int64_t)b * k * a.ldr;
    for (int e = tid; e < nr * k; e += blockDim.x) {
        const int i = e / k, c = e - i * k;
        const int gi = lr0 + i;
        if (gi < k) Rb_out[(int64_t)gi * a.ldr + c] = c >= gi ? sgn[gi] * A[(size_t)c * ld + i] : 0.0;
    }
    __syncthreads();  // R is read from A before form-Q overwrites it

    if (a.wy) {
        // V[gi][c] = 1 on the diagonal, v_c below it, 0 above
        // (a reflector with tau = 0 is the identity: its column is written as 0 so
        //  that I - V T V^T needs no entry for it)
        for (int e = tid; e < nr * k; e += blockDim.x) {
            const int i = e / k, c = e - i * k;
            const int gi = lr0 + i;
            const double v = gi > c ? A[(size_t)c * ld + i] : (gi == c ? 1.0 : 0.0);
            a.qout[(row0 + lr0 + i) * a.ldq + c] = tau[c] != 0.0 ? v : 0.0;
        }
        if (r == 0)
            for (int c = tid; c < k; c += blockDim.x) {
                a.tau_out[c] = tau[c];
                a.sgn_out[c] = sgn[c];
            }
        cl.sync();  // peers are done reading this CTA's reduction buffers
        return;
    }

    // ------------------------------------------------------------ form Q --
    // Q = H_0 ... H_{k-1} [I; 0] in place (dorg2r order). Step j applies H_j to
    // the columns c > j, and in the same pass accumulates step j-1's dots
    // v_{j-1}^T Q(:, c >= j). Column j keeps its reflector v_j during step j
    // (everyone reads it); its owner finishes it at the start of step j-1,
    // and its step-(j-1) dot uses the closed form of the finished column:
    // Q(:,j) = [0; 1 - t_j; -t_j v_j(j+1:)].
    cl.sync();  // peers are done with the factor's reduction buffers
    int par = 0;
    auto finish_col = [&](int c) {
        double* x = A + (size_t)c * ld;
        const double tc = tau[c];
        for (int i = lane; i < nr; i += 32) {
            const int gi = lr0 + i;
            x[i] = gi > c ? -tc * x[i] : (gi == c ? 1.0 - tc : 0.0);
        }
        __syncwarp();
    };
    for (int j = k - 1; j >= 0; --j) {
        const int nt = k - j - 1;
        const int jo = j - lr0;
        const bool owner = jo >= 0 && jo < nr;
        const double tj = tau[j];
        const double* v = A + (size_t)j * ld;
        const bool reduce = nt > 0 && tj != 0.0;  // identical on every CTA
        if (reduce) {
            double* P = red + (par & 1) * RW;
            cl.sync();
            for (int idx = tid; idx < nt; idx += blockDim.x) S[idx] = csum((int)(P - red), idx);
            ++par;
        }
        __syncthreads();
        double* Pn = red + (par & 1) * RW;  // payload of step j-1
        const bool next = j >= 1 && tau[j - 1] != 0.0;
        const double* vn = A + (size_t)(j >= 1 ? j - 1 : 0) * ld;
        const int jon = j - 1 - lr0;
        const bool ownern = jon >= 0 && jon < nr;
        const int i0n = max(0, j - lr0);      // rows > j-1
        const int i0 = max(0, j + 1 - lr0);   // rows > j
        // column j (still v_j): its step-(j-1) dot in closed form
        if (next && warp == j % nw) {
            double s = 0.0;
            for (int i = i0 + lane; i < nr; i += 32) s = fma(vn[i], -tj * v[i], s);
            s = warp_sum(s);
            if (lane == 0) Pn[0] = s + (owner ? vn[jo] * (1.0 - tj) : 0.0);
        }
        // columns c > j: finish column j+1 (first use as a Q column), apply H_j, dots with v_{j-1}
        for (int c0 = first_owned(j + 1); c0 < k; c0 += 4 * nw) {
            if (c0 == j + 1) finish_col(j + 1);
            ColGroup<4> g(A, ld, c0, nw, k);
            double dd[4], sn[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                dd[q] = (reduce && g.on[q]) ? S[c0 + q * nw - j - 1] * tj : 0.0;
                sn[q] = 0.0;
            }
            if (owner && lane == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (g.on[q]) g.y[q][jo] -= dd[q];
            }
            __syncwarp();  // row j is read by another lane in the dot below
            if (next) {
#pragma unroll 2
                for (int i = i0n + lane; i < nr; i += 32) {
                    const double vi = (lr0 + i > j) ? v[i] : 0.0;
                    const double wn = vn[i];
                    double yv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) yv[q] = g.y[q][i];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        yv[q] = fma(-dd[q], vi, yv[q]);
                        sn[q] = fma(wn, yv[q], sn[q]);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (g.on[q]) g.y[q][i] = yv[q];
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) sn[q] = warp_sum(sn[q]);
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (g.on[q]) Pn[c0 + q * nw - j] = sn[q] + (ownern ? g.y[q][jon] : 0.0);
                }
            } else if (reduce) {
#pragma unroll 2
                for (int i = i0 + lane; i < nr; i += 32) {
                    const double vi = v[i];
                    double yv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) yv[q] = g.y[q][i];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (g.on[q]) g.y[q][i] = fma(-dd[q], vi, yv[q]);
                }
            }
        }
    }
    __syncthreads();
    if (warp == 0) finish_col(0);
    // every CTA must be done reading its peers' reduction buffers before exit
    cl.sync();
    for (int e = tid; e < nr * k; e += blockDim.x) {
        const int i = e / k, c = e - i * k;
        a.qout[(row0 + lr0 + i) * a.ldq + c] = sgn[c] * A[(size_t)c * ld + i];
    }
}

// Compact WY for the explicit Q of a single-block QR (LAPACK dlarft + dorgqr
// as GEMMs). With V the unit-lower Householder vectors (zero columns where
// tau = 0), H_0 ... H_{k-1} = I - V T V^T with T upper triangular and
//   T^{-1} = diag(1/tau) + strictly_upper(V^T V)
// (1 on the diagonal where tau = 0), so T comes from one triangular inverse
// (trinv_kernel) instead of dlarft's k-step recurrence, and
//   Q = (I - V T V^T)[:, :k] diag(sgn) = E diag(sgn) - V X,  X = T V1^T diag(sgn)
// (V1 = top k x k block of V): two DMMA GEMMs plus a diagonal fix-up.
// wy_prep_kernel forms U = T^{-1} and B = V1^T diag(sgn) (both k x ld, zero padded).
__global__ void wy_prep_kernel(const double* __restrict__ G, int ldg, const double* __restrict__ tau,
                               const double* __restrict__ sgn, const double* __restrict__ V, int64_t ldv, int k,
                               double* __restrict__ U, double* __restrict__ B, int ld, const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
        const int i = e / k, j = e - i * k;
        double u = 0.0;
        if (j > i) u = G[(size_t)i * ldg + j];
        else if (j == i) u = tau[i] != 0.0 ? 1.0 / tau[i] : 1.0;
        U[(size_t)i * ld + j] = u;
        // B[l][c] = V[c][l] sgn[c] for l <= c  (V1 is unit lower triangular)
        const int l = i, c = j;
        B[(size_t)l * ld + c] = l <= c ? V[(size_t)c * ldv + l] * sgn[c] : 0.0;
    }
}

// Q(c, c) += sgn[c] for c < k (the E diag(sgn) term of the compact-WY Q).
__global__ void wy_diag_kernel(double* __restrict__ Q, int64_t ldq, const double* __restrict__ sgn, int k,
                               const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    for (int c = threadIdx.x; c < k; c += blockDim.x) Q[(size_t)c * ldq + c] += sgn[c];
}

// Register-resident variant: thread t owns column c = t % k over a chunk of
// CH consecutive local rows (chunk = t / k), so the block's rows live in
// registers and every per-reflector sweep is a register FMA stream with the
// current reflector column broadcast from shared memory (all lanes of a warp
// read the same x_i). Per reflector: owners publish x / row j -> barrier ->
// per-(column, chunk) dots -> barrier -> per-column chunk sums (fixed order)
// into the cluster payload -> cluster reduction -> register update. Same
// math and payload as cqr_kernel; used when k * ceil(rows_per_cta / CH)
// threads fit one CTA.
// max threads per CTA for a CH-double register stream (64K registers / (2 CH + ~30))
__host__ __device__ constexpr int cqr_reg_maxt(int CH) {
    return CH <= 32 ? 512 : 256;
}

template <int CH>
__global__ void __launch_bounds__(cqr_reg_maxt(CH), 1) cqr_reg_kernel(CqrArgs a) {
    if (pred_off(a.pred, a.pred_skip)) return;
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks();
    const int r = (int)cl.block_rank();
    const int b = blockIdx.x / C;
    const int rows = a.rows[b];
    const int64_t row0 = a.row0[b];
    const int k = a.k;
    const int Rb = (rows + C - 1) / C;
    const int lr0 = r * Rb;
    const int nr = max(0, min(Rb, rows - lr0));
    const int nch = (Rb + CH - 1) / CH;
    const int RW = cqr_rw(k);
    const int tid = threadIdx.x;
    const int col = tid % k, chunk = tid / k;
    const bool own = chunk < nch;
    const int i0 = chunk * CH;  // first local row of this thread's chunk

    extern __shared__ __align__(16) double sm[];
    double* xb = sm;                          // [nch*CH] current reflector column (rows > j), 0 elsewhere
    double* rowj = xb + (size_t)nch * CH;     // [k]  row j of the block
    double* part = rowj + k;                  // [nch][k] per-chunk partial dots
    double* red = part + (size_t)nch * k;     // [2][RW] cluster payload
    double* S = red + 2 * RW;                 // [RW]
    double* tau = S + RW;                     // [k]
    double* sgn = tau + k;                    // [k]
    __shared__ double* peers[16];

    double v[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const int li = i0 + q;
        v[q] = (own && li < nr) ? a.in[(row0 + lr0 + li) * a.ldi + col] : 0.0;
    }
    if (tid < C) peers[tid] = cl.map_shared_rank(red, tid);
    __syncthreads();
    auto csum = [&](int off, int idx) {  // fixed-order sum, 8 remote loads in flight at a time
        double s = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double t[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) t[q] = 8 * h + q < C ? peers[8 * h + q][off + idx] : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) s += t[q];
        }
        return s;
    };

    // ------------------------------------------------------------ factor --
    int par = 0;
    for (int j = 0; j < k; ++j) {
        const int nt = k - j - 1;
        const int jl = j - lr0;  // local index of global row j (owner iff 0 <= jl < nr)
        double* P = red + (par & 1) * RW;
        ++par;
        // publish x_j (rows > j) and row j
        if (own && col == j) {
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int li = i0 + q;
                xb[li] = (li < nr && lr0 + li > j) ? v[q] : 0.0;
            }
        }
        if (own && jl >= i0 && jl < i0 + CH && jl < nr && col >= j) {
#pragma unroll
            for (int q = 0; q < CH; ++q)
                if (i0 + q == jl) rowj[col] = v[q];
        }
        __syncthreads();
        if (own && col >= j) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int q = 0; q < CH; q += 2) {
                s0 = fma(xb[i0 + q], v[q], s0);
                s1 = fma(xb[i0 + q + 1], v[q + 1], s1);
            }
            part[chunk * k + col] = s0 + s1;
        }
        __syncthreads();
        const bool ownerj = jl >= 0 && jl < nr;
        for (int vc = tid; vc <= nt; vc += blockDim.x) {
            const int c = j + vc;
            double s = 0.0;
            for (int h = 0; h < nch; ++h) s += part[h * k + c];
            const double rv = ownerj ? rowj[c] : 0.0;
            if (vc == 0) {
                P[0] = s;
                P[1] = rv;
            } else {
                P[1 + vc] = s;
                P[1 + nt + vc] = rv;
            }
        }
        cl.sync();
        for (int idx = tid; idx < 2 + 2 * nt; idx += blockDim.x) S[idx] = csum((int)(P - red), idx);
        __syncthreads();
        const double ss = S[0], alpha = S[1];
        double t = 0.0, beta = alpha, scal = 0.0;
        if (ss != 0.0) {
            beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
            t = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        if (tid == 0) {
            tau[j] = t;
            sgn[j] = (a.root_sign && beta < 0.0) ? -1.0 : 1.0;
        }
        if (own && col > j && t != 0.0) {
            const double d = (S[2 + nt + (col - j - 1)] + scal * S[2 + (col - j - 1)]) * t;
            const double ds = d * scal;
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int li = i0 + q;
                v[q] = fma(-ds, xb[li], v[q]);  // xb is 0 for rows <= j and padding rows
                if (li == jl && li < nr) v[q] -= d;  // v_j = 1 at row j
            }
        } else if (own && col == j) {
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int li = i0 + q;
                if (li < nr && lr0 + li > j) v[q] *= scal;
                if (li == jl) v[q] = beta;
            }
        }
        __syncthreads();
    }
    // R rows (< k) from their owners, sign-fixed at the root
    double* Ro = a.R + (int64_t)b * k * a.ldr;
    if (own) {
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const int li = i0 + q, gi = lr0 + li;
            if (li < nr && gi < k) Ro[(int64_t)gi * a.ldr + col] = col >= gi ? sgn[gi] * v[q] : 0.0;
        }
    }

    // ------------------------------------------------------------ form Q --
    cl.sync();  // peers are done with the factor's payload buffers
    for (int j = k - 1; j >= 0; --j) {
        const int nt = k - j - 1;
        const int jl = j - lr0;
        const double tj = tau[j];
        // publish v_j (1 at row j, reflector below, 0 above)
        if (own && col == j) {
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int li = i0 + q;
                const int gi = lr0 + li;
                xb[li] = (li < nr && gi > j) ? v[q] : (li == jl && li < nr ? 1.0 : 0.0);
            }
        }
        __syncthreads();
        if (nt > 0 && tj != 0.0) {
            double* P = red + (par & 1) * RW;
            ++par;
            if (own && col > j) {
                double s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int q = 0; q < CH; q += 2) {
                    s0 = fma(xb[i0 + q], v[q], s0);
                    s1 = fma(xb[i0 + q + 1], v[q + 1], s1);
                }
                part[chunk * k + col] = s0 + s1;
            }
            __syncthreads();
            for (int vc = tid; vc < nt; vc += blockDim.x) {
                double s = 0.0;
                for (int h = 0; h < nch; ++h) s += part[h * k + j + 1 + vc];
                P[vc] = s;
            }
            cl.sync();
            for (int idx = tid; idx < nt; idx += blockDim.x) S[idx] = csum((int)(P - red), idx);
            __syncthreads();
            if (own && col > j) {
                const double d = S[col - j - 1] * tj;
#pragma unroll
                for (int q = 0; q < CH; ++q) v[q] = fma(-d, xb[i0 + q], v[q]);
            }
        }
        if (own && col == j) {  // finish column j (dorg2r)
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int gi = lr0 + i0 + q;
                v[q] = gi > j ? -tj * v[q] : (gi == j ? 1.0 - tj : 0.0);
            }
        }
        __syncthreads();
    }
    cl.sync();  // every CTA done reading its peers' payload buffers
    if (own) {
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const int li = i0 + q;
            if (li < nr) a.qout[(row0 + lr0 + li) * a.ldq + col] = sgn[col] * v[q];
        }
    }
}

__host__ __device__ inline size_t cqr_reg_smem_bytes(int Rb, int k, int CH) {
    const int nch = (Rb + CH - 1) / CH;
    return ((size_t)nch * CH + k + (size_t)nch * k + 3 * (size_t)cqr_rw(k) + 2 * (size_t)k + 8) * sizeof(double);
}

// Stack pairs of k x k R factors into 2k x k row-major node inputs
// (pass-through nodes copy their single R and mark nothing: the node kernel
// runs on k rows and yields Q = I up to signs, which is what we want).
__global__ void stack_r_kernel(const double* __restrict__ Rin, int nin, int k, int ldr, double* __restrict__ out,
                               int ldo, const int* pred, int pred_skip) {
    if (pred_off(pred, pred_skip)) return;
    const int node = blockIdx.x;
    const int a = 2 * node, bq = 2 * node + 1;
    for (int e = threadIdx.x; e < 2 * k * k; e += blockDim.x) {
        const int i = e / k, c = e - i * k;
        const int src = i < k ? a : bq;
        const int ii = i < k ? i : i - k;
        double v = 0.0;
        if (src < nin) v = Rin[((int64_t)src * k + ii) * ldr + c];
        out[((int64_t)node * 2 * k + i) * ldo + c] = v;
    }
}

}  // namespace sorsvd_dev
