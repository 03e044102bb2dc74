// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" wrapper around the reference's own header-only C++20 library
// (/root/reference/proj/include/panelblas/*.hpp), compiled by oracle/Makefile
// straight from those sources into oracle/_ref/libpanelblas_ref.so.  No
// reference source is copied: the headers are included in place via -I.
//
// It exposes (a) the reference's BLAS-shaped adapters and native panel
// routines (blas.hpp:73-215, level3.hpp:360-575), (b) its naive oracles
// (reference.hpp:23-199), (c) its seeded generator (matgen.hpp:14-57) and
// (d) multithreaded batch loops over (a) used as the CPU baseline arm of
// bench.py (one std::thread per core, contiguous problem split, as
// SURVEY.md §8(d) prescribes).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "panelblas/blas.hpp"
#include "panelblas/matgen.hpp"
#include "panelblas/reference.hpp"
#include "panelblas/riccati.hpp"

using namespace panelblas;

template <typename F>
static void parallel_for(long long batch, int threads, F&& f) {
  if (threads <= 1) { for (long long p = 0; p < batch; ++p) f(p); return; }
  std::vector<std::thread> pool;
  long long per = (batch + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    long long lo = t * per, hi = std::min(batch, lo + per);
    if (lo >= hi) break;
    pool.emplace_back([=, &f] { for (long long p = lo; p < hi; ++p) f(p); });
  }
  for (auto& th : pool) th.join();
}


extern "C" {

// Same byte layout as pb_dmat in include/pbgpu.h and panelblas::PanelRef.
struct ref_dmat {
  double* data;
  int ps, m, n, pm, cn;
};

static int g_err_index = 0;
int ref_last_error_index() { return g_err_index; }

static int blas_ret(const BlasResult& r) {
  g_err_index = r.error ? r.error->index : 0;
  return r.info;
}

static TransOp tr(char c) { return *parse_trans(c); }
static PanelRef pr(const ref_dmat& d) { return PanelRef{d.data, d.ps, d.m, d.n, d.pm, d.cn}; }
static ConstPanelRef cpr(const ref_dmat& d) { return ConstPanelRef(pr(d)); }

// ---- (a) the reference path through the boundary being replaced ----
int ref_dgemm(char ta, char tb, int m, int n, int k, double alpha, const double* a, int lda,
              const double* b, int ldb, double beta, double* c, int ldc) {
  BlasConfig cfg;
  return blas_ret(dgemm(cfg, ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc));
}
int ref_dsyrk(char uplo, char trans, int n, int k, double alpha, const double* a, int lda,
              double beta, double* c, int ldc) {
  BlasConfig cfg;
  return blas_ret(dsyrk(cfg, uplo, trans, n, k, alpha, a, lda, beta, c, ldc));
}
int ref_dtrsm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
              const double* a, int lda, double* b, int ldb) {
  BlasConfig cfg;
  return blas_ret(dtrsm(cfg, side, uplo, transa, diag, m, n, alpha, a, lda, b, ldb));
}
int ref_dtrmm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
              const double* a, int lda, double* b, int ldb) {
  BlasConfig cfg;
  return blas_ret(dtrmm(cfg, side, uplo, transa, diag, m, n, alpha, a, lda, b, ldb));
}
int ref_dpotrf(char uplo, int n, double* a, int lda) {
  BlasConfig cfg;
  return blas_ret(dpotrf(cfg, uplo, n, a, lda));
}
int ref_dgetrf(int m, int n, double* a, int lda, int* ipiv) {
  BlasConfig cfg;
  std::vector<int> piv;
  int info = blas_ret(dgetrf(cfg, m, n, a, lda, piv));
  for (size_t i = 0; i < piv.size(); ++i) ipiv[i] = piv[i];
  return info;
}
int ref_gemm_nd(char ta, char tb, int m, int n, int k, double alpha, ref_dmat a, ref_dmat b,
                double beta, ref_dmat c, ref_dmat d) {
  EngineConfig cfg;
  g_err_index = 0;
  return gemm_nd(cfg, tr(ta), tr(tb), m, n, k, alpha, cpr(a), cpr(b), beta, cpr(c), pr(d)).status.info;
}
int ref_syrk_nd(int n, int k, double alpha, ref_dmat a, double beta, ref_dmat c, ref_dmat d) {
  EngineConfig cfg;
  g_err_index = 0;
  return syrk_nd(cfg, n, k, alpha, cpr(a), beta, cpr(c), pr(d)).status.info;
}
int ref_trsm_rltn_nd(int m, int n, double alpha, ref_dmat a, ref_dmat b, ref_dmat d) {
  EngineConfig cfg;
  g_err_index = 0;
  return trsm_rltn_nd(cfg, m, n, alpha, cpr(a), cpr(b), pr(d)).status.info;
}
int ref_syrk_potrf_nd(int n, int k, ref_dmat a, ref_dmat b, ref_dmat c, ref_dmat d) {
  EngineConfig cfg;
  g_err_index = 0;
  return syrk_potrf_nd(cfg, n, k, cpr(a), cpr(b), cpr(c), pr(d)).status.info;
}

// ---- (b) naive oracles (second opinion) ----
void ref_naive_gemm(char ta, char tb, int m, int n, int k, double alpha, const double* a, int lda,
                    const double* b, int ldb, double beta, double* c, int ldc) {
  ConstMatView av{a, tr(ta) == TransOp::NoTrans ? m : k, tr(ta) == TransOp::NoTrans ? k : m, lda};
  ConstMatView bv{b, tr(tb) == TransOp::NoTrans ? k : n, tr(tb) == TransOp::NoTrans ? n : k, ldb};
  ref::naive_gemm(tr(ta), tr(tb), m, n, k, alpha, av, bv, beta, MatView{c, m, n, ldc});
}
int ref_naive_potrf(char uplo, int n, double* a, int lda) {
  return ref::naive_potrf(*parse_uplo(uplo), n, MatView{a, n, n, lda}).info;
}
int ref_naive_getrf(int m, int n, double* a, int lda, int* ipiv) {
  std::vector<int> piv;
  int info = ref::naive_getrf(m, n, MatView{a, m, n, lda}, piv).info;
  for (size_t i = 0; i < piv.size(); ++i) ipiv[i] = piv[i];
  return info;
}
int ref_naive_trsm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
                   const double* a, int lda, double* b, int ldb) {
  int t = *parse_side(side) == Side::Left ? m : n;
  return ref::naive_trsm(*parse_side(side), *parse_uplo(uplo), tr(transa), *parse_diag(diag), m, n,
                         alpha, ConstMatView{a, t, t, lda}, MatView{b, m, n, ldb}).info;
}
void ref_naive_trmm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
                    const double* a, int lda, double* b, int ldb) {
  int t = *parse_side(side) == Side::Left ? m : n;
  ref::naive_trmm(*parse_side(side), *parse_uplo(uplo), tr(transa), *parse_diag(diag), m, n, alpha,
                  ConstMatView{a, t, t, lda}, MatView{b, m, n, ldb});
}

// ---- (c) seeded generators (matgen.hpp) ----
void ref_rng_uniform(uint64_t seed, long long count, double lo, double hi, double* out) {
  Rng rng(seed);
  for (long long i = 0; i < count; ++i) out[i] = rng.uniform(lo, hi);
}
void ref_make_spd(int n, uint64_t seed, double* out) {
  Rng rng(seed);
  Matrix a = make_spd(n, rng);
  std::memcpy(out, a.data(), sizeof(double) * n * n);
}

// ---- (d) multithreaded batch loops: the CPU baseline ----
int ref_hw_threads() { return (int)std::thread::hardware_concurrency(); }

void ref_dgemm_batch(char ta, char tb, int m, int n, int k, double alpha, const double* a, int lda,
                     long long sa, const double* b, int ldb, long long sb, double beta, double* c,
                     int ldc, long long sc, long long batch, int threads) {
  parallel_for(batch, threads, [&](long long p) {
    BlasConfig cfg;
    dgemm(cfg, ta, tb, m, n, k, alpha, a + p * sa, lda, b + p * sb, ldb, beta, c + p * sc, ldc);
  });
}
void ref_dpotrf_batch(char uplo, int n, double* a, int lda, long long sa, int* info,
                      long long batch, int threads) {
  parallel_for(batch, threads, [&](long long p) {
    BlasConfig cfg;
    info[p] = dpotrf(cfg, uplo, n, a + p * sa, lda).info;
  });
}
void ref_dgetrf_batch(int m, int n, double* a, int lda, long long sa, int* ipiv, long long sipiv,
                      int* info, long long batch, int threads) {
  parallel_for(batch, threads, [&](long long p) {
    BlasConfig cfg;
    std::vector<int> piv;
    info[p] = dgetrf(cfg, m, n, a + p * sa, lda, piv).info;
    for (size_t i = 0; i < piv.size(); ++i) ipiv[p * sipiv + i] = piv[i];
  });
}
void ref_gemm_nd_batch(char ta, char tb, int m, int n, int k, double alpha, ref_dmat a, long long sa,
                       ref_dmat b, long long sb, double beta, ref_dmat c, long long sc, ref_dmat d,
                       long long sd, long long batch, int threads) {
  parallel_for(batch, threads, [&](long long p) {
    EngineConfig cfg;
    ref_dmat ap = a, bp = b, cp = c, dp = d;
    ap.data += p * sa; bp.data += p * sb; cp.data += p * sc; dp.data += p * sd;
    gemm_nd(cfg, tr(ta), tr(tb), m, n, k, alpha, cpr(ap), cpr(bp), beta, cpr(cp), pr(dp));
  });
}
// cfg5 column-major chain per problem: dsyrk('l','n') C += A A^T; dpotrf('l') C;
// dtrsm('r','l','t','n') X L^T = B.  Variable n per problem, offsets in doubles.
void ref_chain_cm_batch(const int* nvec, const long long* off_nn, double* A, double* C, double* B,
                        int* info, long long batch, int threads) {
  parallel_for(batch, threads, [&](long long p) {
    BlasConfig cfg;
    int n = nvec[p];
    double* a = A + off_nn[p]; double* c = C + off_nn[p]; double* b = B + off_nn[p];
    dsyrk(cfg, 'l', 'n', n, n, 1.0, a, n, 1.0, c, n);
    int inf = dpotrf(cfg, 'l', n, c, n).info;
    if (inf == 0) inf = dtrsm(cfg, 'r', 'l', 't', 'n', n, n, 1.0, c, n, b, n).info;
    info[p] = inf;
  });
}
// cfg5 panel-major chain: syrk_potrf_nd(n, n, A, A, C, C) then trsm_rltn_nd(n, n, 1, L, B, B).
void ref_chain_pm_batch(const int* nvec, const long long* off_nn, double* A, double* C, double* B,
                        int* info, long long batch, int threads) {
  parallel_for(batch, threads, [&](long long p) {
    EngineConfig cfg;
    int n = nvec[p];
    PanelRef a = PanelRef::over(A + off_nn[p], n, n, 4);
    PanelRef c = PanelRef::over(C + off_nn[p], n, n, 4);
    PanelRef b = PanelRef::over(B + off_nn[p], n, n, 4);
    int inf = syrk_potrf_nd(cfg, n, n, a, a, c, c).status.info;
    if (inf == 0) inf = trsm_rltn_nd(cfg, n, n, 1.0, c, b, b).status.info;
    info[p] = inf;
  });
}


// ---- (e) trmm_rlnn_nd, pack, and the Riccati application (riccati.hpp) ----
int ref_trmm_rlnn_nd(int m, int n, double alpha, ref_dmat a, ref_dmat b, ref_dmat d) {
  EngineConfig cfg;
  g_err_index = 0;
  return trmm_rlnn_nd(cfg, m, n, alpha, cpr(a), cpr(b), pr(d)).status.info;
}
void ref_pack_from_colmajor(char trans, const double* a, int lda, int am, int an, ref_dmat d) {
  pack_from_colmajor(ConstMatView{a, am, an, lda}, pr(d), tr(trans));
}
void ref_unpack_to_colmajor(ref_dmat s, double* a, int lda) {
  unpack_to_colmajor(cpr(s), MatView{a, s.m, s.n, lda});
}
long long ref_memsize(int m, int n, int ps) { return (long long)memsize(m, n, ps); }
// make_ocp_data (riccati.hpp:65-103): column-major a (nx x nx), b (nx x nu), q, r, s (nu x nx)
void ref_make_ocp_data(int nx, int nu, uint64_t seed, double* a, double* b, double* q, double* r, double* s) {
  OcpData d = make_ocp_data(nx, nu, seed);
  std::memcpy(a, d.a.data(), sizeof(double) * nx * nx);
  if (nu) std::memcpy(b, d.b.data(), sizeof(double) * nx * nu);
  std::memcpy(q, d.q.data(), sizeof(double) * nx * nx);
  if (nu) std::memcpy(r, d.r.data(), sizeof(double) * nu * nu);
  if (nu) std::memcpy(s, d.s.data(), sizeof(double) * nu * nx);
}
// RiccatiFusedWork on make_ocp_data(seed): init_terminal, then N steps.  Stage s's bordered
// factor [[Lambda, 0], [L, calL]] lands column-major (nt x nt, zeros above) at fst + s*nt*nt,
// the terminal factor calL_N at lterm (nx x nx).  Returns status.info; *fail_stage = the
// failing stage (N for the terminal factor) or -1.
int ref_riccati_fused(int nx, int nu, int N, uint64_t seed, double* fst, double* lterm, int* fail_stage) {
  OcpData d = make_ocp_data(nx, nu, seed);
  EngineConfig cfg;
  RiccatiFusedWork w(d, cfg);
  const int nt = nx + nu;
  *fail_stage = -1;
  Status st = w.init_terminal();
  if (!st.ok()) { *fail_stage = N; return st.info; }
  Matrix c0 = w.call_cm();
  std::memcpy(lterm, c0.data(), sizeof(double) * nx * nx);
  for (int n = N - 1; n >= 0; --n) {
    RiccatiStepResult r = w.step();
    if (!r.ok()) { *fail_stage = n; return r.status.info; }
    double* out = fst + (long long)n * nt * nt;
    std::memset(out, 0, sizeof(double) * nt * nt);
    Matrix lam = w.lambda_cm(), l = w.l_cm(), cl = w.call_cm();
    for (int j = 0; j < nu; ++j)
      for (int i = j; i < nu; ++i) out[i + j * nt] = lam(i, j);
    for (int j = 0; j < nu; ++j)
      for (int i = 0; i < nx; ++i) out[nu + i + j * nt] = l(i, j);
    for (int j = 0; j < nx; ++j)
      for (int i = j; i < nx; ++i) out[nu + i + (nu + j) * nt] = cl(i, j);
  }
  return 0;
}
// riccati_run (riccati.hpp:402-512): impl 0 blas, 1 fused, 2 oracle; returns the residual.
double ref_riccati_run(int nx, int nu, int N, int impl, uint64_t seed, int* info) {
  RiccatiRunResult r = riccati_run(OcpDims{nx, nu, N}, static_cast<RiccatiImpl>(impl), seed);
  *info = r.status.info;
  return r.residual;
}
// chol_residual (riccati.hpp:124-140), column-major
double ref_chol_residual(int n, const double* l, int ldl, const double* p, int ldp) {
  return chol_residual(ConstMatView{l, n, n, ldl}, ConstMatView{p, n, n, ldp});
}
// riccati_oracle_step (riccati.hpp:145-180) on make_ocp_data(seed): p <- step(pnext), cm nx x nx
int ref_riccati_oracle_step(int nx, int nu, uint64_t seed, const double* pnext, double* p) {
  OcpData d = make_ocp_data(nx, nu, seed);
  return riccati_oracle_step(d, ConstMatView{pnext, nx, nx, nx}, MatView{p, nx, nx, nx}).info;
}
uint64_t ref_riccati_seed() { return kRiccatiSeed; }

}  // extern "C"
