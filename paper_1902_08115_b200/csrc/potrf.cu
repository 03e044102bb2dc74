// Batched Cholesky (dpotrf, lower; upper through transposed addressing) for sm_100a.
//
// Replaces potrf_core (factor.hpp:45-99).  The size switch:
//   n <= 32   potrf_reg.cu  (register-resident, a lane segment per problem);
//   n <= 160  potrf_cta.cu  (one CTA per problem, shared-memory resident,
//             pipelined left-looking panels on DMMA);
//   n > 160   right-looking blocked over 128-column panels, composed here from
//             potrf_cta (diagonal block) -> trsm_rlt (panel solve) -> the DMMA
//             gemm engine (lower syrk of the trailing matrix); column-major
//             (lower / upper) or panel-major (lower, with the LowerZero band
//             zeros of syrk_potrf_nd) in place.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace pbg {

constexpr int kPotrfSmemMax = 160;

cudaError_t potrf_launch(const PotrfLaunch& L, cudaStream_t s) {
  if (L.batch <= 0 || L.n <= 0) return cudaSuccess;
  static const int blocked_from = [] {  // PBGPU_POTRF_BLOCKED_FROM=n: blocked path from this order on (tuning)
    const char* e = getenv("PBGPU_POTRF_BLOCKED_FROM");
    return e ? atoi(e) : kPotrfSmemMax + 1;
  }();
  if (L.n <= kPotrfSmemMax && L.n < blocked_from)
    return potrf_cta_launch(L.a, L.stride, L.offs, nullptr, L.lda, L.n, L.upper, L.pm, L.zero_fill, L.info, 0, 0,
                            L.batch, s);
  if (L.pm && L.upper) return cudaErrorInvalidValue;
  // element (i, j) of the lower problem: i + j*lda (lower), j + i*lda (upper),
  // (i/4)*4*cn + 4j + i%4 (panel-major; block corners are multiples of 8, so
  // every sub-block is again a panel-major view with the same cn)
  auto at = [&](int i, int j) -> long long {
    if (L.pm) return (long long)(i >> 2) * 4 * L.lda + (long long)j * 4 + (i & 3);
    return L.upper ? (long long)j + (long long)i * L.lda : (long long)i + (long long)j * L.lda;
  };
  // Right-looking blocked over 128-column panels: potrf(A11) -> A21 = A21 L11^{-T}
  // (trsm) -> A22 -= A21 A21^T (DMMA syrk) -> recurse on A22.  Problems whose
  // info turned nonzero are skipped by every later stage.
  static const int nb_env = [] {  // PBGPU_POTRF_NB: block order of the blocked path (tuning)
    const char* e = getenv("PBGPU_POTRF_NB");
    return e ? atoi(e) : 0;
  }();
  const int nb = nb_env >= 16 && nb_env <= kPotrfSmemMax && nb_env % 8 == 0 ? nb_env : 128;
  for (int c0 = 0; c0 < L.n; c0 += nb) {
    const int w = std::min(nb, L.n - c0), rest = L.n - c0 - w;
    // element (i, j) of the lower problem lives at i + j*lda (lower) or j + i*lda (upper)
    double* a11 = L.a + at(c0, c0);
    cudaError_t e = potrf_cta_launch(a11, L.stride, L.offs, nullptr, L.lda, w, L.upper, L.pm, L.zero_fill, L.info,
                                     c0, c0 > 0, L.batch, s);
    if (e != cudaSuccess) return e;
    if (!rest) break;
    TrsmLaunch T;
    T.pm = L.pm;
    T.twin = L.upper;      // upper: rows of the effective problem are columns
    T.lower = 1;
    T.trans = 1;           // X * L11^T = A21
    T.unit = 0;
    T.mm = rest;
    T.nn = w;
    T.alpha = 1.0;
    T.a = a11; T.sa = L.stride; T.lda = L.lda;
    T.offs_a = T.offs_b = L.offs;  // (null: strided)
    // Lower: A21 rows c0+w.. at (c0+w) + c0*lda.  Upper: twin view of A12 at c0 + (c0+w)*lda.
    double* b = L.upper ? L.a + (long long)c0 + (long long)(c0 + w) * L.lda : L.a + at(c0 + w, c0);
    T.b = b; T.sb = L.stride; T.ldb = L.lda;
    T.d = b; T.sd = L.stride; T.ldd = L.lda;
    T.info = L.info;
    T.skip_nonzero = 1;
    T.batch = L.batch;
    if (L.upper) T.trans = 0, T.lower = 0;  // twin problem: X * U11 = A12^T with U11 = L11^T stored upper
    e = trsm_launch(T, s);
    if (e != cudaSuccess) return e;
    GemmLaunch g;
    double* a22 = L.a + at(c0 + w, c0 + w);
    if (L.pm) {      // A22 -= A21 A21^T, panel-major in and out
      g.lay_a = g.lay_b = L_PMX;
      g.out_pm = 1;
    } else if (!L.upper) {  // A22 -= A21 A21^T  (syrk 'l','n')
      g.lay_a = g.lay_b = L_MNC;
    } else {         // A22(upper) -= A12^T A12 (syrk 'u','t')
      g.lay_a = g.lay_b = L_KC;
    }
    g.a.base = g.b.base = b;
    g.a.stride = g.b.stride = L.stride;
    g.a.ld = g.b.ld = L.lda;
    g.a.bulk = g.b.bulk = ((reinterpret_cast<uintptr_t>(b) & 15) == 0) && L.lda % 2 == 0 &&
                          (L.offs ? L.offs_even != 0 : L.stride % 2 == 0);
    g.a.offs = g.b.offs = L.offs;
    g.o.offs = L.offs;
    g.o.c = a22;
    g.o.d = a22;
    g.o.sc = g.o.sd = L.stride;
    g.o.ldc = g.o.ldd = L.lda;
    // 16-byte pairs (i, i + 1), i even: block origins are multiples of 4 rows
    g.o.vec = ((reinterpret_cast<uintptr_t>(a22) & 15) == 0) && (L.pm || L.lda % 2 == 0) &&
              (L.offs ? L.offs_even != 0 : L.stride % 2 == 0);
    g.m = g.n = rest;
    g.k = w;
    g.alpha = -1.0;
    g.beta = 1.0;
    g.uplo = L.upper ? 2 : 1;
    g.skip = L.info;
    g.batch = L.batch;
    e = gemm_launch(g, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace pbg
