// Peak microbenchmarks for the roofline denominators the driver does not
// measure: FP64 DFMA, FP64 DMMA (mma.sync f64), FP32 FFMA, HBM read.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.0) out[0] = s;
}
template <int CH>
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-9f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.0f) out[0] = s;
}
// m8n8k4 f64: A 1 dbl, B 1 dbl, C 2 dbl per thread
template <int CH>
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
// m16n8k4 f64: A 2 dbl, B 1 dbl, C 4 dbl
template <int CH>
__global__ void dmma1684_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}
// m16n8k16 f64: A 8 dbl, B 4 dbl, C 4 dbl
template <int CH>
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = 1.0 + threadIdx.x * 1e-4 + j;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}
__global__ void read_kernel(const double2* __restrict__ p, size_t n, double* out) {
  double s = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride * 4) {
    double2 v0 = p[i];
    double2 v1 = (i + stride < n) ? p[i + stride] : make_double2(0, 0);
    double2 v2 = (i + 2 * stride < n) ? p[i + 2 * stride] : make_double2(0, 0);
    double2 v3 = (i + 3 * stride < n) ? p[i + 3 * stride] : make_double2(0, 0);
    s += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
  }
  if (s == 12345.0) out[0] = s;
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* dout; CK(cudaMalloc(&dout, 64));
  const int iters = 20000;
  for (int tpb : {256, 512, 1024}) {
    int grid = sms * (2048 / tpb);
    float ms = timeit([&] { dfma_kernel<8><<<grid, tpb>>>(dout, iters, 1.0000001, 1e-9); }, 3);
    double fl = 2.0 * grid * tpb * 8.0 * iters;
    printf("DFMA tpb=%d: %.2f TFLOP/s\n", tpb, fl / ms / 1e9);
  }
  {
    int tpb = 512, grid = sms * 4;
    float ms = timeit([&] { ffma_kernel<8><<<grid, tpb>>>((float*)dout, iters, 1.0000001f, 1e-9f); }, 3);
    double fl = 2.0 * grid * tpb * 8.0 * iters;
    printf("FFMA: %.2f TFLOP/s\n", fl / ms / 1e9);
  }
  for (int tpb : {128, 256, 512}) {
    int grid = sms * (1024 / tpb);
    int it2 = 4000;
    float ms = timeit([&] { dmma884_kernel<4><<<grid, tpb>>>(dout, it2); }, 3);
    double fl = 2.0 * 8 * 8 * 4 * 4.0 * it2 * (grid * tpb / 32);
    printf("DMMA m8n8k4 tpb=%d: %.2f TFLOP/s\n", tpb, fl / ms / 1e9);
    ms = timeit([&] { dmma1684_kernel<4><<<grid, tpb>>>(dout, it2); }, 3);
    fl = 2.0 * 16 * 8 * 4 * 4.0 * it2 * (grid * tpb / 32);
    printf("DMMA m16n8k4 tpb=%d: %.2f TFLOP/s\n", tpb, fl / ms / 1e9);
    ms = timeit([&] { dmma16816_kernel<4><<<grid, tpb>>>(dout, it2); }, 3);
    fl = 2.0 * 16 * 8 * 16 * 4.0 * it2 * (grid * tpb / 32);
    printf("DMMA m16n8k16 tpb=%d: %.2f TFLOP/s\n", tpb, fl / ms / 1e9);
  }
  {
    size_t bytes = (size_t)8 << 30;
    double2* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 0, bytes));
    size_t n = bytes / 16;
    for (int occ : {4, 8}) {
      int grid = sms * occ, tpb = 256;
      float ms = timeit([&] { read_kernel<<<grid, tpb>>>(p, n, dout); }, 5);
      printf("HBM read occ=%d: %.1f GB/s\n", occ, bytes / ms / 1e6);
    }
    CK(cudaFree(p));
  }
  return 0;
}
