// Roofline denominators the driver does not measure for FP64: the DMMA
// (mma.sync m8n8k4 f64) issue-bound throughput and a streaming HBM read.
#pragma once
#include "common.cuh"

namespace sorsvd_dev {

__global__ void peak_dmma_kernel(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[4][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma884(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void peak_read_kernel(const double2* __restrict__ p, size_t n, double* out) {
    double s = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride * 4) {
        double2 v0 = p[i];
        double2 v1 = (i + stride < n) ? p[i + stride] : make_double2(0, 0);
        double2 v2 = (i + 2 * stride < n) ? p[i + 2 * stride] : make_double2(0, 0);
        double2 v3 = (i + 3 * stride < n) ? p[i + 3 * stride] : make_double2(0, 0);
        s += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
    }
    if (s == 12345.0) out[0] = s;
}

}  // namespace sorsvd_dev
