/* Minimal LAPACKE prototype header -- TEST INFRASTRUCTURE ONLY.
 * The image has LAPACKE symbols (OpenBLAS 0.3.15 / LAPACK 3.9.0 bundled with
 * opencv-python-headless) but no lapacke.h.  The reference's lapack.cpp
 * (/root/reference/proj/src/lapack.cpp:9-15) defines lapack_complex_double
 * before including this header; these are the four routines it calls
 * (:41, :65, :82, :109). */
#ifndef EBEM_ORACLE_LAPACKE_SHIM_H
#define EBEM_ORACLE_LAPACKE_SHIM_H
#ifndef lapack_int
#define lapack_int int
#endif
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102
#ifdef __cplusplus
extern "C" {
#endif
lapack_int LAPACKE_zgetrf(int matrix_layout, lapack_int m, lapack_int n,
                          lapack_complex_double* a, lapack_int lda,
                          lapack_int* ipiv);
lapack_int LAPACKE_zgetrs(int matrix_layout, char trans, lapack_int n,
                          lapack_int nrhs, const lapack_complex_double* a,
                          lapack_int lda, const lapack_int* ipiv,
                          lapack_complex_double* b, lapack_int ldb);
lapack_int LAPACKE_zgecon(int matrix_layout, char norm, lapack_int n,
                          const lapack_complex_double* a, lapack_int lda,
                          double anorm, double* rcond);
lapack_int LAPACKE_zgeqp3(int matrix_layout, lapack_int m, lapack_int n,
                          lapack_complex_double* a, lapack_int lda,
                          lapack_int* jpvt, lapack_complex_double* tau);
#ifdef __cplusplus
}
#endif
#endif
