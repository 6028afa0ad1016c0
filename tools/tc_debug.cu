// Standalone check of the tcgen05 TF32 tile kernel (one 128 x BN tile).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#define TC_DEBUG
#include "../paper_1804_00462_b200/csrc/tc_gemm_f32.cuh"
using namespace sorsvd_dev;
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap mk(EncodeTiledFn f, const float* base, long rows, long cols, long ld, int bx, int by, bool mn) {
    CUtensorMap m; cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}; cuuint64_t st[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by}; cuuint32_t es[2] = {1, 1};
    CUresult r = f(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode failed %d\n", (int)r);
    return m;
}
int main(int argc, char** argv) {
    const int M = 128, K = argc > 1 ? atoi(argv[1]) : 32, N = 32;
    const bool ta = argc > 2 && atoi(argv[2]);
    std::vector<float> A((size_t)M * K), B((size_t)K * N), C((size_t)M * N);
    for (size_t i = 0; i < A.size(); ++i) A[i] = (float)((long)(i * 37 % 11) - 5) * 0.25f;
    for (size_t i = 0; i < B.size(); ++i) B[i] = (float)((long)(i * 13 % 7) - 3) * 0.5f;
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
    std::vector<float> At(A.size());  // for TA: store A^T as K x M
    for (int i = 0; i < M; ++i) for (int k = 0; k < K; ++k) At[(size_t)k * M + i] = A[(size_t)i * K + k];
    cudaMemcpy(dA, ta ? At.data() : A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dC, 0xff, C.size() * 4);
    void* fp; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeTiledFn f = (EncodeTiledFn)fp;
    CUtensorMap ma = ta ? mk(f, dA, K, M, M, 32, 32, true) : mk(f, dA, M, K, K, 32, 128, false);
    CUtensorMap mb = mk(f, dB, K, N, N, 32, 32, true);
    float* ddbg; cudaMalloc(&ddbg, 64 * 4); cudaMemset(ddbg, 0, 256);
    cudaMemcpyToSymbol(tc_dbg, &ddbg, sizeof(ddbg));
    TcArgs a{}; a.C = dC; a.ldc = N; a.M = M; a.K = K; a.k_chunk = K;
    size_t sm = TcShape<32>::SMEM;
    if (ta) {
        cudaFuncSetAttribute(tc_gemm_tf32_kernel<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        tc_gemm_tf32_kernel<32, true><<<1, 256, sm>>>(ma, mb, a);
    } else {
        cudaFuncSetAttribute(tc_gemm_tf32_kernel<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        tc_gemm_tf32_kernel<32, false><<<1, 256, sm>>>(ma, mb, a);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, nrm = 0;
    for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
        double r = 0; for (int k = 0; k < K; ++k) r += (double)A[(size_t)i * K + k] * B[(size_t)k * N + j];
        err = fmax(err, fabs(r - C[(size_t)i * N + j])); nrm = fmax(nrm, fabs(r));
        if (i < 2 && j < 4) printf("C[%d][%d] = %g ref %g\n", i, j, C[(size_t)i * N + j], r);
    }
    printf("max err %g (max |ref| %g)\n", err, nrm);
    float hd[64]; cudaMemcpy(hd, ddbg, 256, cudaMemcpyDeviceToHost);
    printf("tmem %g a_s %g\nA smem:", hd[0], hd[1]); for (int q = 2; q < 10; ++q) printf(" %g", hd[q]);
    printf("\nB smem:"); for (int q = 10; q < 18; ++q) printf(" %g", hd[q]);
    printf("\nA[0][0..7]:"); for (int q = 0; q < 8; ++q) printf(" %g", A[q]);
    printf("\nB[0][0..7]:"); for (int q = 0; q < 8; ++q) printf(" %g", B[q]); printf("\n");
    // find a permutation hint: which ref entry matches C[0][0..3]
    return 0;
}
