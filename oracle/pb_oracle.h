/* TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into, or called by,
 * the product library (paper_1902_08115_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.
 *
 * A plain-C restatement of the reference's hot path (the header-only
 * panelblas library under /root/reference/proj/include/panelblas).  Every
 * routine restates the reference's arithmetic ORDER (l-ascending tile
 * accumulation with separate multiply and add, reciprocal scaling in the
 * edges, the left-looking band schedule of potrf, the nr=4 blocked
 * right-looking getrf), so on any input it reproduces the reference bit for
 * bit; tests/test_oracle.py pins that against oracle/_ref (the reference
 * compiled from its own headers) and against the reference's exact fixtures.
 *
 * Return values follow the reference: BLAS routines return the positive
 * 1-based Fortran index of the first bad argument (blas.hpp:27-31), LAPACK
 * routines -index, numerical failures +p, panel routines the engine Status
 * codes (level3.hpp:360-575), kInfoUnsupported = -1000 (gemm.hpp:183).
 */
#ifndef PB_ORACLE_H
#define PB_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_dmat { double* data; int ps, m, n, pm, cn; } orc_dmat;

int orc_dgemm(char transa, char transb, int m, int n, int k, double alpha, const double* a, int lda,
              const double* b, int ldb, double beta, double* c, int ldc);
int orc_dsyrk(char uplo, char trans, int n, int k, double alpha, const double* a, int lda,
              double beta, double* c, int ldc);
int orc_dtrsm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
              const double* a, int lda, double* b, int ldb);
int orc_dtrmm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
              const double* a, int lda, double* b, int ldb);
int orc_dpotrf(char uplo, int n, double* a, int lda);
int orc_dgetrf(int m, int n, double* a, int lda, int* ipiv);

int orc_gemm_nd(char transa, char transb, int m, int n, int k, double alpha, orc_dmat a, orc_dmat b,
                double beta, orc_dmat c, orc_dmat d);
int orc_syrk_nd(int n, int k, double alpha, orc_dmat a, double beta, orc_dmat c, orc_dmat d);
int orc_trsm_rltn_nd(int m, int n, double alpha, orc_dmat a, orc_dmat b, orc_dmat d);
int orc_syrk_potrf_nd(int n, int k, orc_dmat a, orc_dmat b, orc_dmat c, orc_dmat d);
int orc_trmm_rlnn_nd(int m, int n, double alpha, orc_dmat a, orc_dmat b, orc_dmat d);

/* Threaded batch loops (contiguous split) — the "port" CPU baseline. */
void orc_dgemm_batch(char ta, char tb, int m, int n, int k, double alpha, const double* a, int lda,
                     long long sa, const double* b, int ldb, long long sb, double beta, double* c,
                     int ldc, long long sc, long long batch, int threads);
void orc_dpotrf_batch(char uplo, int n, double* a, int lda, long long sa, int* info,
                      long long batch, int threads);
void orc_dgetrf_batch(int m, int n, double* a, int lda, long long sa, int* ipiv, long long sipiv,
                      int* info, long long batch, int threads);
void orc_gemm_nd_batch(char ta, char tb, int m, int n, int k, double alpha, orc_dmat a, long long sa,
                       orc_dmat b, long long sb, double beta, orc_dmat c, long long sc, orc_dmat d,
                       long long sd, long long batch, int threads);
/* config-5 chain, pm = 0 column-major / 1 panel-major, offsets in doubles */
void orc_chain_batch(int pm, const int* nvec, const long long* off, double* A, double* C, double* B,
                     int* info, long long batch, int threads);

#ifdef __cplusplus
}
#endif
#endif
