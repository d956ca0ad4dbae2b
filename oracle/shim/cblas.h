/* Prototype-only CBLAS shim for building the reference oracle (test
 * infrastructure only). The reference includes <cblas.h> at
 * /root/reference/proj/include/qtnh/linalg.hpp:18 and calls cblas_zgemm at
 * linalg.hpp:391. The implementation is the OpenBLAS build bundled with scipy
 * (scipy.libs/libscipy_openblas-*.so), whose symbols carry a "scipy_" prefix. */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
#define cblas_zgemm scipy_cblas_zgemm
void scipy_cblas_zgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb,
                       int m, int n, int k, const void* alpha, const void* a, int lda,
                       const void* b, int ldb, const void* beta, void* c, int ldc);
#ifdef __cplusplus
}
#endif
