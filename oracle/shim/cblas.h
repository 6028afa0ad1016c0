/* TEST INFRASTRUCTURE (oracle only). Minimal CBLAS declarations so the
 * reference headers (/root/reference/proj/include/sorsvd/dense.hpp:4) compile
 * against the OpenBLAS 0.3.15 that ships in this image's opencv wheel. The
 * reference expects these from an un-vendored vendor/ dir
 * (/root/reference/proj/CMakeLists.txt:5). Standard CBLAS enum values. */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
typedef enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 } CBLAS_ORDER;
typedef enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 } CBLAS_TRANSPOSE;
void cblas_dgemm(CBLAS_ORDER order, CBLAS_TRANSPOSE ta, CBLAS_TRANSPOSE tb, int m, int n, int k,
                 double alpha, const double* a, int lda, const double* b, int ldb, double beta,
                 double* c, int ldc);
void openblas_set_num_threads(int n);
char* openblas_get_config(void);
#ifdef __cplusplus
}
#endif
