// Builder-written LAPACKE shim for oracle/_ref: forwards LAPACKE_dsyev to
// scipy's bundled OpenBLAS (32-bit integer interface).
#pragma once
typedef int lapack_int;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102
extern "C" lapack_int scipy_LAPACKE_dsyev(int, char, char, lapack_int, double*, lapack_int, double*);
inline lapack_int LAPACKE_dsyev(int layout, char jobz, char uplo, lapack_int n, double* a, lapack_int lda,
                                double* w) {
  return scipy_LAPACKE_dsyev(layout, jobz, uplo, n, a, lda, w);
}
