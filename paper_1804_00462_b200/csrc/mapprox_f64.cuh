// Single-pass core (sketch.hpp:54-58, dense.hpp:138-157):
//     M_approx = (Q1^T T1) * pinv(Q2^T W),  pinv(X) = V diag(w) U^T,
//     w_l = 1/sigma_l if sigma_l > tol*sigma_1 else 0,  tol = ell * eps.
// Q1^T T1 and Q2^T W are skinny TN GEMMs on the DMMA engine and the SVD of
// the ell x ell core is the Jacobi kernel; what is left is two ell^3 products
// on ell x ell operands (<= 256), far too small to be worth tensor-core
// tiling: one thread per output element, ell-long FMA chain, fixed order.
#pragma once
#include "common.cuh"

namespace sorsvd_dev {

// C[i][j] = sum_l A[i][l] * w_l * (BT ? B[j][l] : B[l][j]),  i, j < ell.
// w_l = 1 when S == nullptr, else the pseudo-inverse weight of S[l].
__global__ void small_gemm_kernel(const double* __restrict__ A, int lda, const double* __restrict__ B, int ldb,
                                  bool bt, const double* __restrict__ S, double tol, double* __restrict__ C, int ldc,
                                  int ell) {
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ell) return;
    const double cut = S ? tol * S[0] : 0.0;
    double acc = 0.0;
    for (int l = 0; l < ell; ++l) {
        double w = 1.0;
        if (S) w = S[l] > cut ? 1.0 / S[l] : 0.0;
        const double b = bt ? B[(size_t)j * ldb + l] : B[(size_t)l * ldb + j];
        acc = fma(A[(size_t)i * lda + l] * w, b, acc);
    }
    C[(size_t)i * ldc + j] = acc;
}

}  // namespace sorsvd_dev
