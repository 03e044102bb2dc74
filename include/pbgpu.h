/* pbgpu — B200-native batched FP64 small-matrix BLAS/LAPACK.
 *
 * C ABI (extern "C", plain pointers and sizes) that replaces the reference
 * library's hot-path entry points (panelblas, /root/reference/proj/include/
 * panelblas/).  Each declaration cites the reference interface it replaces.
 *
 * Pointer kinds.  Every matrix/ipiv/info pointer of one call must be of one
 * kind: CUDA device (or managed) memory, or host memory (pageable or
 * pinned).  Device calls are asynchronous on `stream`; host calls stage
 * through the GPU (chunked, copies overlapped with compute) and return when
 * the results are back in host memory.  There is no CPU compute path: with
 * no usable GPU every call fails with PB_INFO_NO_DEVICE.
 *
 * Return value / pb_result.info follow the reference exactly:
 *   BLAS routines (dgemm, dsyrk, dtrsm): a bad argument returns its positive
 *     1-based Fortran position (blas.hpp:27-31, 77-79);
 *   LAPACK routines (dpotrf, dgetrf): -position for a bad argument, +p for a
 *     numerical failure (blas.hpp:190-215, mat_view.hpp:78-90);
 *   panel routines (*_nd): the engine Status codes (level3.hpp:360-575),
 *     PB_INFO_UNSUPPORTED = kInfoUnsupported (gemm.hpp:183).
 * Batched factorizations/solves report per-problem numerical failures in the
 * caller's info[batch] array (same memory kind as the matrices) and return 0
 * from the call itself unless an argument is invalid.  Arguments the
 * reference signature has keep the reference's position in error reports;
 * the batched extensions (strides, batch, info, ipiv) report positions
 * after them.  info (and ipiv) of the batched factorizations must not be NULL.
 */
#ifndef PBGPU_H
#define PBGPU_H

#ifdef __cplusplus
extern "C" {
#endif

#define PB_INFO_UNSUPPORTED (-1000) /* gemm.hpp:183 kInfoUnsupported */
#define PB_INFO_CUDA_ERROR (-2000)  /* a CUDA call failed; see pb_result.message */
#define PB_INFO_NO_DEVICE (-2001)   /* no usable CUDA device: no CPU fallback exists */

/* Panel-major descriptor, byte-compatible with panelblas::PanelRef
 * (panel_mat.hpp:51-81): element (i, j) at data[(i/ps)*ps*cn + j*ps + i%ps],
 * pm = ceil(m/ps)*ps, cn = ceil(n/ps)*ps.  ps must be 4 (KernelConfig::ps). */
typedef struct pb_dmat {
  double* data;
  int ps, m, n, pm, cn;
} pb_dmat;

/* Outcome of one call — panelblas::BlasResult (blas.hpp:32-40) flattened:
 * info, the BlasCallError {routine, index, message} of an invalid call, and
 * the textbook flop count of the whole call (bench.hpp:119-138). */
typedef struct pb_result {
  int info;
  int error_index;
  const char* routine;
  const char* message;
  long long flops;
} pb_result;

typedef void* pb_stream; /* cudaStream_t; NULL = the calling thread's default stream */

int pb_version(void);
/* Number of visible CUDA devices (0 when none).  Selecting a device is the
 * caller's job (cudaSetDevice / torch.cuda.set_device), one process per GPU. */
int pb_device_count(void);
/* Measured-FP64 helpers used by the bench: DMMA / DFMA peak probes (TFLOP/s). */
double pb_probe_dmma_tflops(void);

/* ---------------- single-call, netlib-shaped (drop-in for blas.hpp) ---------------- */
/* replaces panelblas::dgemm  (blas.hpp:73-102) */
int pb_dgemm(char transa, char transb, int m, int n, int k, double alpha, const double* a, int lda,
             const double* b, int ldb, double beta, double* c, int ldc, pb_result* res);
/* replaces panelblas::dsyrk  (blas.hpp:104-128) */
int pb_dsyrk(char uplo, char trans, int n, int k, double alpha, const double* a, int lda,
             double beta, double* c, int ldc, pb_result* res);
/* replaces panelblas::dtrsm  (blas.hpp:178-188) */
int pb_dtrsm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
             const double* a, int lda, double* b, int ldb, pb_result* res);
/* replaces panelblas::dpotrf (blas.hpp:190-202) */
int pb_dpotrf(char uplo, int n, double* a, int lda, pb_result* res);
/* replaces panelblas::dgetrf (blas.hpp:204-215); ipiv has min(m, n) entries, 1-based */
int pb_dgetrf(int m, int n, double* a, int lda, int* ipiv, pb_result* res);

/* ---------------- single-call, panel-major (drop-in for level3.hpp native API) ---------------- */
/* replaces panelblas::gemm_nd (level3.hpp:360-403); transa must be 'N' */
int pb_gemm_nd(char transa, char transb, int m, int n, int k, double alpha, pb_dmat a, pb_dmat b,
               double beta, pb_dmat c, pb_dmat d, pb_result* res);
/* replaces panelblas::syrk_nd (level3.hpp:407-441) */
int pb_syrk_nd(int n, int k, double alpha, pb_dmat a, double beta, pb_dmat c, pb_dmat d,
               pb_result* res);
/* replaces panelblas::trsm_rltn_nd (level3.hpp:484-526) */
int pb_trsm_rltn_nd(int m, int n, double alpha, pb_dmat a, pb_dmat b, pb_dmat d, pb_result* res);
/* replaces panelblas::syrk_potrf_nd (level3.hpp:533-575) */
int pb_syrk_potrf_nd(int n, int k, pb_dmat a, pb_dmat b, pb_dmat c, pb_dmat d, pb_result* res);

/* ---------------- strided batched (problem p at base + p*stride elements) ---------------- */
int pb_dgemm_batched(char transa, char transb, int m, int n, int k, double alpha, const double* a,
                     int lda, long long stride_a, const double* b, int ldb, long long stride_b,
                     double beta, double* c, int ldc, long long stride_c, int batch,
                     pb_stream stream, pb_result* res);
int pb_dsyrk_batched(char uplo, char trans, int n, int k, double alpha, const double* a, int lda,
                     long long stride_a, double beta, double* c, int ldc, long long stride_c,
                     int batch, pb_stream stream, pb_result* res);
int pb_dtrsm_batched(char side, char uplo, char transa, char diag, int m, int n, double alpha,
                     const double* a, int lda, long long stride_a, double* b, int ldb,
                     long long stride_b, int* info, int batch, pb_stream stream, pb_result* res);
int pb_dpotrf_batched(char uplo, int n, double* a, int lda, long long stride_a, int* info,
                      int batch, pb_stream stream, pb_result* res);
int pb_dgetrf_batched(int m, int n, double* a, int lda, long long stride_a, int* ipiv,
                      long long stride_ipiv, int* info, int batch, pb_stream stream,
                      pb_result* res);
/* panel-major: the descriptors give the shape of problem 0, *.data its base */
int pb_gemm_nd_batched(char transa, char transb, int m, int n, int k, double alpha, pb_dmat a,
                       long long stride_a, pb_dmat b, long long stride_b, double beta, pb_dmat c,
                       long long stride_c, pb_dmat d, long long stride_d, int batch,
                       pb_stream stream, pb_result* res);
int pb_syrk_nd_batched(int n, int k, double alpha, pb_dmat a, long long stride_a, double beta,
                       pb_dmat c, long long stride_c, pb_dmat d, long long stride_d, int batch,
                       pb_stream stream, pb_result* res);
int pb_trsm_rltn_nd_batched(int m, int n, double alpha, pb_dmat a, long long stride_a, pb_dmat b,
                            long long stride_b, pb_dmat d, long long stride_d, int* info,
                            int batch, pb_stream stream, pb_result* res);
int pb_syrk_potrf_nd_batched(int n, int k, pb_dmat a, long long stride_a, pb_dmat b,
                             long long stride_b, pb_dmat c, long long stride_c, pb_dmat d,
                             long long stride_d, int* info, int batch, pb_stream stream,
                             pb_result* res);

/* ---------------- variable-size chain (Riccati-like stage, config 5) ----------------
 * Per problem p of order n[p] (square, ld = n[p], problem storage at
 * base + offset[p] elements; pm layout uses ps = 4 and n[p] % 4 == 0):
 *   layout 'C' (column-major):  dsyrk('l','n') C += A A^T; dpotrf('l') C;
 *                               dtrsm('r','l','t','n') X L^T = B  (X over B)
 *   layout 'P' (panel-major):   syrk_potrf_nd(n, n, A, A, C, C);
 *                               trsm_rltn_nd(n, n, 1, C, B, B)
 * info[p] = 0, or the failing pivot of the Cholesky step; max_n bounds n[p].
 * Memory kinds: A, C, B and info all on the device (asynchronous on `stream`;
 * with device n / offset the split by order costs one device -> host copy and
 * a stream synchronisation), n / offset on the HOST with device matrices
 * (asynchronous, no synchronisation), or everything on the host (staged
 * through the device, returns when done; the caller's riccati-style buffers). */
int pb_chain_vbatched(char layout, const int* n, const long long* offset, double* A, double* C,
                      double* B, int* info, int batch, int max_n, pb_stream stream,
                      pb_result* res);

/* ---------------- triangular multiply (completes the six-routine surface) ---------------- */
/* replaces panelblas::dtrmm (blas.hpp:166-176 -> level3.hpp:250-275): B <- alpha op(A) B
 * (side 'l') or alpha B op(A) (side 'r'); validation shared with dtrsm (blas.hpp:132-162) */
int pb_dtrmm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
             const double* a, int lda, double* b, int ldb, pb_result* res);
int pb_dtrmm_batched(char side, char uplo, char transa, char diag, int m, int n, double alpha,
                     const double* a, int lda, long long stride_a, double* b, int ldb,
                     long long stride_b, int batch, pb_stream stream, pb_result* res);
/* replaces panelblas::trmm_rlnn_nd (level3.hpp:446-479): d <- alpha b a, a lower non-unit;
 * b may alias d exactly */
int pb_trmm_rlnn_nd(int m, int n, double alpha, pb_dmat a, pb_dmat b, pb_dmat d, pb_result* res);
int pb_trmm_rlnn_nd_batched(int m, int n, double alpha, pb_dmat a, long long stride_a, pb_dmat b,
                            long long stride_b, pb_dmat d, long long stride_d, int batch,
                            pb_stream stream, pb_result* res);

/* ---------------- layout conversion on the device (panel_mat.hpp:45-48, 141-171) ---------------- */
/* replaces panelblas::memsize (panel_mat.hpp:45-48): bytes of an m x n matrix packed with height ps */
long long pb_memsize(int m, int n, int ps);
/* replaces pack_from_colmajor (panel_mat.hpp:141-160): d <- packed op(a), op(a) is d.m x d.n,
 * any panel height d.ps; pad lanes of d are never written */
int pb_pack(char trans, const double* a, int lda, pb_dmat d, pb_result* res);
int pb_pack_batched(char trans, const double* a, int lda, long long stride_a, pb_dmat d,
                    long long stride_d, int batch, pb_stream stream, pb_result* res);
/* replaces unpack_to_colmajor (panel_mat.hpp:164-171): a (s.m x s.n, ld lda) <- s */
int pb_unpack(pb_dmat s, double* a, int lda, pb_result* res);
int pb_unpack_batched(pb_dmat s, long long stride_s, double* a, int lda, long long stride_a,
                      int batch, pb_stream stream, pb_result* res);

/* ---------------- batched factorized Riccati recursion (the paper's application) ----------------
 * replaces, for a batch of independent OCPs with equal (nx, nu, N), RiccatiFusedWork's stage loop
 * as riccati_run's FusedNative path drives it (riccati.hpp:257-373, 402-512).  Panel-major, ps = 4:
 *   m0 (nt x nt, nt = nx + nu): bordered stage matrix [[R, S], [S^T, Q]], packed fully symmetric;
 *   q (nx x nx): Q;  g (nt x nx): G = [B^T; A^T].
 * calL_N = chol(Q); for s = N-1 .. 0: C = G calL_{s+1} (trmm_rlnn_nd),
 * F_s = chol(m0 + C C^T) (syrk_potrf_nd), calL_s = trailing nx x nx block of F_s.
 * f receives the N stage factors F_s of problem p at f.data + p*stride_f + s*f.pm*f.cn (lower,
 * crossing tiles zero-filled, strictly-upper tiles zero: [[Lambda, 0], [L, calL]]);
 * lterm (optional, data may be NULL) receives calL_N.  info[p] = 0 or the failing pivot's
 * 1-based bordered index (riccati.hpp:234-278); stage[p] (optional) = the failing stage, N for
 * the terminal factor, -1 when none failed.  Stages below a failed one are unspecified. */
int pb_riccati_nd_batched(int nx, int nu, int N, pb_dmat m0, long long stride_m0, pb_dmat q,
                          long long stride_q, pb_dmat g, long long stride_g, pb_dmat f,
                          long long stride_f, pb_dmat lterm, long long stride_lterm, int* info,
                          int* stage, int batch, pb_stream stream, pb_result* res);

/* Fault injection: with the environment variable PBGPU_MUTATE=eps set when the library is
 * loaded, every routine adds eps to element (0, 0) of each problem's result (the analogue of
 * PANELBLAS_MUTATE, gemm.hpp:126-127, micro_kernel.hpp:424-426) — a negative control that
 * must turn the parity harness red. */

#ifdef __cplusplus
}
#endif
#endif /* PBGPU_H */
