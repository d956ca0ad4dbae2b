/* Prototype-only LAPACKE shim for the reference oracle (test infrastructure
 * only). linalg.hpp:17 defines LAPACK_COMPLEX_CPP before including this, and
 * calls LAPACKE_zgesdd (linalg.hpp:417) / LAPACKE_zgesvd (linalg.hpp:427). */
#pragma once
#include <complex>
typedef int lapack_int;
typedef std::complex<double> lapack_complex_double;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102
#define LAPACKE_zgesdd scipy_LAPACKE_zgesdd
#define LAPACKE_zgesvd scipy_LAPACKE_zgesvd
extern "C" {
lapack_int scipy_LAPACKE_zgesdd(int layout, char jobz, lapack_int m, lapack_int n,
                                lapack_complex_double* a, lapack_int lda, double* s,
                                lapack_complex_double* u, lapack_int ldu,
                                lapack_complex_double* vt, lapack_int ldvt);
lapack_int scipy_LAPACKE_zgesvd(int layout, char jobu, char jobvt, lapack_int m, lapack_int n,
                                lapack_complex_double* a, lapack_int lda, double* s,
                                lapack_complex_double* u, lapack_int ldu,
                                lapack_complex_double* vt, lapack_int ldvt, double* superb);
}
