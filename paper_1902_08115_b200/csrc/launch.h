// Internal launcher interface between the host boundary (pbgpu_api.cpp) and
// the sm_100a kernels.  Plain structs of device pointers and sizes; every
// launcher is asynchronous on the given stream and returns the launch error.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pbg {

// Operand storage kinds for the tiled DMMA engine (gemm.cu).  x is the
// operand's row index in the product (i of op(A), j of op(B)^T), l the
// contraction index.
enum Lay : int {
  L_MNC = 0,  // column-major, x contiguous: (x, l) at x + l*ld
  L_KC = 1,   // column-major, l contiguous: (x, l) at l + x*ld
  L_PMX = 2,  // panel-major (ps = 4), panels over x: (x/4)*4*cn + l*4 + x%4
  L_PML = 3,  // panel-major (ps = 4), panels over l: (l/4)*4*cn + x*4 + l%4
};

struct OpDesc {
  const double* base = nullptr;  // problem 0
  long long stride = 0;          // elements between consecutive problems
  int ld = 0;                    // leading dimension (cm) or panel width cn (pm)
  int bulk = 0;                  // 1 when every bulk copy is 16-byte aligned
  const long long* offs = nullptr;  // optional per-problem element offsets (replace p * stride; no TMA)
};

struct OutDesc {
  const double* c = nullptr;  // source of beta*C (may equal d)
  double* d = nullptr;
  long long sc = 0, sd = 0;
  int ldc = 0, ldd = 0;  // ld (cm) or cn (pm)
  int vec = 0;           // 1 when 16-byte paired accesses are aligned
  const long long* offs = nullptr;    // optional per-problem element offsets of d (and c, unless offs_c)
  const long long* offs_c = nullptr;  // optional per-problem element offsets of c alone
};

struct GemmLaunch {
  int lay_a = L_MNC, lay_b = L_KC;  // M side (op(A)) and N side (op(B)^T)
  int out_pm = 0;                   // 0: C/D column-major, 1: panel-major
  OpDesc a, b;
  OutDesc o;
  int m = 0, n = 0, k = 0;
  double alpha = 1.0, beta = 0.0;
  int uplo = 0;  // 0 full, 1 lower (i >= j), 2 upper (i <= j)
  const int* skip = nullptr;  // optional: skip problems with skip[p] != 0
  int batch = 0;
};
cudaError_t gemm_launch(const GemmLaunch& g, cudaStream_t s);
// d <- beta*c on the (uplo-masked) m x n result; beta == 0 writes +0 without reading c.
cudaError_t scale_launch(int out_pm, const OutDesc& o, int m, int n, double beta, int uplo,
                         int batch, cudaStream_t s);

// Per-device runtime state (runtime.cpp, thread-safe): SM count, and the
// >48 KB dynamic shared-memory opt-in of a kernel on the current device.
int num_sms();
cudaError_t smem_attr(const void* fn, int bytes, bool max_carveout = false);

// small-size panel-major NT gemm (s <= 32, packed problems): gemm_small.cu
bool gemm_small_ok(int s, const double* a, const double* b, const double* c, const double* d, long long sa,
                   long long sb, long long sc, long long sd, int cna, int cnb, int cnc, int cnd);
cudaError_t gemm_small_launch(int s, double alpha, const double* a, const double* b, double beta,
                              const double* c, double* d, long long batch, cudaStream_t st);
// column-major NN square packed problems, 32 <= s <= 64, s % 8 == 0 (gemm_small.cu)
bool gemm_cm_ok(int s, const double* a, const double* b, const double* c, long long sa, long long sb,
                long long sc, int lda, int ldb, int ldc);
cudaError_t gemm_cm_launch(int s, double alpha, const double* a, const double* b, double beta, double* c,
                           long long batch, cudaStream_t st);
// column-major small problems, m, n <= 32, any k / trans / leading dimensions: warp per problem
// (gemm_cmsmall.cu) — the small-n branch of the size switch (variant D, gemm.hpp:190-204)
bool gemm_cmsmall_ok(int m, int n);
// uplo: 0 full, 1 lower, 2 upper — the opposite triangle is neither read nor written (dsyrk)
cudaError_t gemm_cmsmall_launch(int ta, int tb, int m, int n, int k, double alpha, const double* a, int lda,
                                long long sa, const double* b, int ldb, long long sb, double beta, double* c,
                                int ldc, long long sc, int uplo, long long batch, cudaStream_t s);

}  // namespace pbg

namespace pbg {

// Cholesky (dpotrf, in place).  upper = 1 runs the lower algorithm on the
// transposed storage (factor.hpp:45-99 twin windows).  info[p] receives 0 or
// the failing column; on failure only the tiles the reference's band
// schedule would have stored are written (see potrf.cu).
struct PotrfLaunch {
  double* a = nullptr;
  long long stride = 0;
  int lda = 0, n = 0, upper = 0;  // lda: leading dimension (cm) or panel width cn (pm)
  int pm = 0, zero_fill = 0;      // panel-major (lower only); LowerZero band zeros (syrk_potrf_nd)
  const long long* offs = nullptr;  // optional per-problem element offsets (replace p * stride)
  int offs_even = 0;                // caller's promise: every offset is even (16-byte bulk copies)
  int* info = nullptr;
  int batch = 0;
};
cudaError_t potrf_launch(const PotrfLaunch& L, cudaStream_t s);
// pipelined left-looking CTA-per-problem Cholesky, n <= 160 (potrf_cta.cu)
cudaError_t potrf_cta_launch(double* a, long long stride, const long long* offs, const int* nvec, int lda,
                             int n, int upper, int pm, int zero_fill, int* info, int info_offset,
                             int skip_nonzero, int batch, cudaStream_t s);
// register-resident segment-per-problem Cholesky, n <= 32 (potrf_reg.cu); same
// contract as potrf_cta_launch, which forwards orders <= 32 here
cudaError_t potrf_reg_launch(double* a, long long stride, const long long* offs, const int* nvec, int lda, int nmax,
                             int upper, int pm, int zero_fill, int* info, int info_offset, int skip_nonzero,
                             int batch, cudaStream_t s);
// same kernel with the prologue S = C + A B^T (A, B n x k, same storage kind as C)
// (D may differ from C: the kernel stages from c and writes d)
cudaError_t syrk_potrf_cta_launch(double* d, long long stride_d, const long long* offs, const int* nvec, int ldd,
                                  const double* c, long long stride_c, int ldc,
                                  const double* A, const double* B, long long stride_ab, int k, int ldab,
                                  int n, int pm, int zero_fill, int* info, int batch, cudaStream_t s);
// variable batch (offs/nvec required): lower C <- C + A A^T only (the chain's dsyrk
// step), A n x n in the same storage kind, n <= 160
cudaError_t syrk_lower_cta_launch(double* c, const long long* offs, const int* nvec, const double* A, int nmax,
                                  int pm, int* info, int batch, cudaStream_t s);

// LU with partial pivoting (dgetrf, in place).
struct GetrfLaunch {
  double* a = nullptr;
  long long stride = 0;
  int lda = 0, m = 0, n = 0;
  int* ipiv = nullptr;
  long long stride_ipiv = 0;
  int* info = nullptr;
  int batch = 0;
};
cudaError_t getrf_launch(const GetrfLaunch& L, cudaStream_t s);
// pipelined CTA-per-problem LU for shared-memory-resident problems (getrf_cta.cu)
cudaError_t getrf_cta_launch(double* a, long long stride, int lda, int m, int n, int* ipiv, long long sp,
                             int* info, int piv_offset, int keep_info, int batch, cudaStream_t s);

// square n = 40..96 (multiples of 8), compile-time shapes (getrf_sq.cu)
bool getrf_sq_ok(const double* a, long long stride, int lda, int m, int n);
// piv_offset / keep_info / left_cols: the trailing square block of the blocked path
// (its interchanges are also applied to the left_cols columns left of it)
cudaError_t getrf_sq_launch(double* a, long long stride, int lda, int n, int* ipiv, long long sp, int* info,
                            int piv_offset, int keep_info, int left_cols, int batch, cudaStream_t s);

// register-resident warp-per-problem LU, m, n <= 32 (getrf_reg.cu)
bool getrf_reg_ok(int m, int n);
cudaError_t getrf_reg_launch(double* a, long long stride, int lda, int m, int n, int* ipiv, long long sp, int* info,
                             int batch, cudaStream_t s);

// row-resident CTA-per-problem LU, m <= 224 and n <= 64 (n <= 96 for m <= 96)
// (getrf_rows.cu); piv_offset / keep_info serve the tall panels of the blocked path
bool getrf_rows_ok(int m, int n);
// col0/ncols: the panel is columns [col0, col0 + n) of an ncols-column matrix and its
// interchanges are applied to every other column (ncols <= n: panel only)
cudaError_t getrf_rows_launch(double* a, long long stride, int lda, int m, int n, int* ipiv, long long sp, int* info,
                              int piv_offset, int keep_info, int batch, int col0, int ncols, cudaStream_t s);

// Triangular solve.  Column-major dtrsm (in place on b) or the panel-major
// trsm_rltn_nd (b -> d, d may alias b).  The effective problem is always a
// right-side solve X * op(A) = alpha * B over rows of X (Left runs on the
// transposed B through 'twin' addressing, level3.hpp:300-303).
struct TrsmLaunch {
  int pm = 0;                // 0: column-major, 1: panel-major (right/lower/trans/non-unit only)
  int twin = 0;              // Left side: rows of the effective problem are columns of B
  int lower = 1, trans = 0;  // flags of the effective (right-side) problem
  int unit = 0;
  int mm = 0, nn = 0;  // effective rows (independent) and triangle order
  double alpha = 1.0;
  const double* a = nullptr;
  long long sa = 0;
  int lda = 0;  // ld (cm) or cn (pm)
  const double* b = nullptr;
  long long sb = 0;
  int ldb = 0;
  double* d = nullptr;
  long long sd = 0;
  int ldd = 0;
  int* info = nullptr;  // per-problem zero-diagonal report (written before any store)
  int skip_nonzero = 0; // skip problems whose info is already nonzero (blocked callers)
  int batch = 0;
  // variable batches (chain): per-problem order (mm = nn = nvec[p], ld = n or
  // round_up(n, 4)) and element offsets shared by a, b and d
  const int* nvec = nullptr;
  const long long* offs = nullptr;
  // optional per-problem element offsets of a (offs_a) and of b / d (offs_b)
  // with a uniform order (the chain's large orders and the blocked potrf over them)
  const long long* offs_a = nullptr;
  const long long* offs_b = nullptr;
};
cudaError_t trsm_launch(const TrsmLaunch& L, cudaStream_t s);
// Triangular multiply D = alpha * X * op(A) over the same effective right-side
// problem as TrsmLaunch (info / skip / nvec / offs ignored): dtrmm (all flag
// sets, Left as twin) and the panel-major trmm_rlnn_nd; D may alias B (trmm.cu)
cudaError_t trmm_launch(const TrsmLaunch& L, cudaStream_t s);
// panel-major trsm_rltn_nd with alpha == 0: zero-diagonal report, then D = +0 (trsm.cu)
cudaError_t trsm_nd_zero_launch(const TrsmLaunch& L, cudaStream_t s);
// warp-per-8-rows left-looking DMMA solve for X * A^T = alpha B, A lower (trsm_rlt.cu);
// trsm_launch forwards these flag sets
bool trsm_rlt_ok(const TrsmLaunch& L);
// keep the default stream-ordered memory pool's memory between calls (scratch reuse;
// once per device, runtime.cpp)
void mempool_keep();
cudaError_t trsm_rlt_launch(const TrsmLaunch& L, cudaStream_t s);

// Fused panel-major lower chol(C + A B^T) (syrk_potrf_nd).
struct SyrkPotrfLaunch {
  const double *a = nullptr, *b = nullptr, *c = nullptr;
  double* d = nullptr;
  long long sa = 0, sb = 0, sc = 0, sd = 0;
  const long long* offs = nullptr;  // optional per-problem offsets of a, b, c and d (replace the strides)
  int offs_even = 0;                // caller's promise: every offset is even
  int cna = 0, cnb = 0, cnc = 0, cnd = 0;
  int n = 0, k = 0;
  int* info = nullptr;
  int batch = 0;
};
cudaError_t syrk_potrf_launch(const SyrkPotrfLaunch& L, cudaStream_t s);

// Variable-size chain (config 5).  layout 0 = column-major, 1 = panel-major.
struct ChainLaunch {
  int pm = 0;
  const int* n = nullptr;               // device arrays (always)
  const long long* offset = nullptr;
  const int* n_host = nullptr;          // optional host copies: the split is planned
  const long long* offset_host = nullptr;  // without a device -> host round trip
  double *A = nullptr, *C = nullptr, *B = nullptr;
  int* info = nullptr;
  int batch = 0, max_n = 0;
};
cudaError_t chain_launch(const ChainLaunch& L, cudaStream_t s);

// Batched factorized Riccati recursion (riccati.cu): panel-major (ps = 4)
// operands, uniform dims; f holds N stage factors per OCP (stage s at
// f + p*sf + s*cnf*cnf), lterm (optional) the terminal factor chol(Q).
struct RiccatiLaunch {
  int nx = 0, nu = 0, N = 0;
  const double* m0 = nullptr; long long sm0 = 0; int cnm0 = 0;  // nt x nt bordered matrix
  const double* q = nullptr; long long sq = 0; int cnq = 0;     // nx x nx
  const double* g = nullptr; long long sg = 0; int cng = 0;     // nt x nx, [B^T; A^T]
  double* f = nullptr; long long sf = 0; int cnf = 0;           // N x (nt x nt)
  double* lterm = nullptr; long long sl = 0; int cnl = 0;       // nx x nx
  int* info = nullptr;
  int* stage = nullptr;
  int batch = 0;
};
cudaError_t riccati_launch(const RiccatiLaunch& R, cudaStream_t s);

// Layout kernels (layout.cu): batched pack (column-major op(A) -> panel-major,
// any ps, pad lanes untouched) and unpack (panel-major -> column-major).
cudaError_t pack_launch(int trans, int m, int n, const double* a, int lda, long long sa, double* d, int ps,
                        int cn, long long sd, int batch, cudaStream_t s);
cudaError_t unpack_launch(int m, int n, const double* src, int ps, int cn, long long ss, double* a, int lda,
                          long long sa, int batch, cudaStream_t s);
// Fault injection (PBGPU_MUTATE, the analogue of PANELBLAS_MUTATE, gemm.hpp:126-127 /
// micro_kernel.hpp:424-426): adds eps to element (0, 0) of each problem's result.
double mutation_epsilon();
cudaError_t mutate_launch(double* d, long long sd, const long long* offs, int batch, double eps, cudaStream_t s);

double probe_dmma_tflops();

}  // namespace pbg
