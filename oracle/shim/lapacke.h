/* TEST INFRASTRUCTURE (oracle only). Minimal LAPACKE declarations for the
 * three routines the reference calls (dense.hpp:48,73 dgesdd; :119 dgeqrf;
 * :124 dorgqr). Standard LAPACKE layout constants, 32-bit lapack_int. */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
typedef int lapack_int;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102
lapack_int LAPACKE_dgesdd(int layout, char jobz, lapack_int m, lapack_int n, double* a,
                          lapack_int lda, double* s, double* u, lapack_int ldu, double* vt,
                          lapack_int ldvt);
lapack_int LAPACKE_dgeqrf(int layout, lapack_int m, lapack_int n, double* a, lapack_int lda,
                          double* tau);
lapack_int LAPACKE_dorgqr(int layout, lapack_int m, lapack_int n, lapack_int k, double* a,
                          lapack_int lda, const double* tau);
#ifdef __cplusplus
}
#endif
