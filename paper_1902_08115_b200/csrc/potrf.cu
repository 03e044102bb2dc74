// Batched Cholesky (dpotrf, lower; upper through transposed addressing) for sm_100a.
//
// Replaces potrf_core (factor.hpp:45-99) and its tile kernels
// (kernel_potrf_sub/_diag, micro_kernel.hpp:607-636).  One CTA owns one
// problem for n <= 160: the lower triangle is loaded once into shared memory
// (column stride S = 4 mod 16 doubles, so every DMMA fragment load is
// conflict-free) and factored right-looking in 8-column blocks:
//   1. warp 0 factors the 8x8 diagonal block in registers with warp shuffles
//      (sqrt, reciprocal, rank-1 updates; the failing-pivot test is the
//      reference's `piv <= 0.0`, micro_kernel.hpp:314);
//   2. all threads solve the panel rows against it (one row per thread,
//      scaling by the reciprocal of the diagonal like edge_trsm_right);
//   3. all warps apply the trailing lower update A22 -= L21 L21^T with FP64
//      tensor-core DMMA m8n8k4 on 8x8 tiles.
// The factor is written back once.  On failure at column p (0-based) the
// write-back reproduces exactly the tiles the reference's band schedule had
// stored: all lower entries of rows < 8*floor(p/8) and, in that 8-row band,
// the columns < 4*floor(p/4) (test_factor.cpp:251-277).
//
// Larger n is blocked on the host side (pbgpu_api.cpp) over this kernel, the
// trsm kernel and the DMMA gemm engine.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace pbg {

struct PotrfArgs {
  double* a;
  long long stride;
  int lda, n, upper;
  int* info;
  int info_offset;  // added to a reported failing column (blocked callers)
  int skip_nonzero; // skip problems whose info is already nonzero
  int S, NC;        // smem column stride and allocated columns
};

__host__ __device__ inline int smem_stride(int rows8) {
  // smallest S >= rows8 with S % 16 == 4 (conflict-free DMMA fragments)
  int s = ((rows8 - 4 + 15) / 16) * 16 + 4;
  return s < rows8 ? s + 16 : s;
}

__global__ void __launch_bounds__(256) potrf_smem_kernel(const __grid_constant__ PotrfArgs P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double dinv[8];
  __shared__ int sh_fail;
  const int p = blockIdx.x;
  if (P.skip_nonzero && P.info[p] != 0) return;
  const int n = P.n, S = P.S, tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
  double* a = P.a + (long long)p * P.stride;
  auto A = [&](int i, int j) -> double& { return sm[i + j * S]; };

  // ---- load the lower triangle (upper: the transposed storage) ----
  if (!P.upper) {
    stage_cm(sm, S, a, P.lda, 0, n, n, true, tid, nthr);
    cp_async_wait_all();
  } else {
    for (int e = tid; e < n * n; e += nthr) {
      int i = e / n, j = e - i * n;  // lower-problem (i, j) = storage (j, i)
      if (i >= j) A(i, j) = a[j + (long long)i * P.lda];
    }
  }
  if (tid == 0) sh_fail = 0;
  __syncthreads();

  const int nt8 = (n + 7) >> 3;
  for (int kb = 0; kb < nt8; ++kb) {
    const int c0 = kb * 8, w = min(8, n - c0);
    // ---- 1. diagonal block in registers (warp 0) ----
    if (warp == 0) {
      const int r = lane;
      double v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = (r < w && c <= r) ? A(c0 + r, c0 + c) : 0.0;
      int fail = 0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < w && !fail) {
          const double piv = __shfl_sync(0xffffffffu, v[c], c);
          if (piv <= 0.0) {
            fail = c + 1;
          } else {
            const double s = sqrt(piv);
            const double inv = 1.0 / s;
            if (r == c) v[c] = s;
            if (r > c) v[c] *= inv;
            if (lane == c) dinv[c] = inv;
#pragma unroll
            for (int c2 = c + 1; c2 < 8; ++c2) {
              const double f = __shfl_sync(0xffffffffu, v[c], c2);
              if (c2 < w && r >= c2) v[c2] -= v[c] * f;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (r < w && c <= r) A(c0 + r, c0 + c) = v[c];
      if (lane == 0 && fail) sh_fail = c0 + fail;
    }
    __syncthreads();
    if (sh_fail) break;
    const int r0 = c0 + w;
    if (r0 >= n) break;
    // ---- 2. panel rows: L21 = A21 L11^{-T} ----
    for (int i = r0 + tid; i < n; i += nthr) {
      double x[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = A(i, c0 + c);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
#pragma unroll
        for (int l = 0; l < c; ++l) x[c] -= x[l] * A(c0 + c, c0 + l);
        x[c] *= dinv[c];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) A(i, c0 + c) = x[c];
    }
    __syncthreads();
    // ---- 3. trailing update A22 -= L21 L21^T on lower 8x8 tiles (DMMA) ----
    {
      const int g = lane >> 2, t = lane & 3;
      const int t0 = kb + 1, mt = nt8 - t0, ntiles = mt * (mt + 1) / 2;
      for (int idx = warp; idx < ntiles; idx += nwarps) {
        int I = (int)((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
        while ((I + 1) * (I + 2) / 2 <= idx) ++I;
        while (I * (I + 1) / 2 > idx) --I;
        const int J = idx - I * (I + 1) / 2;
        const int ri = (t0 + I) * 8, rj = (t0 + J) * 8;
        double d0 = 0.0, d1 = 0.0;
        dmma(d0, d1, A(ri + g, c0 + t), A(rj + g, c0 + t));
        dmma(d0, d1, A(ri + g, c0 + 4 + t), A(rj + g, c0 + 4 + t));
        A(ri + g, rj + 2 * t) -= d0;
        A(ri + g, rj + 2 * t + 1) -= d1;
      }
    }
    __syncthreads();
  }

  // ---- write back ----
  const int fail = sh_fail;
  int lim_rows = n, band_lo = n, band_cols = 0;
  if (fail) {
    const int pc = fail - 1;
    band_lo = (pc / 8) * 8;     // rows below this band were never stored
    lim_rows = min(n, band_lo + 8);
    band_cols = (pc / 4) * 4;  // stored columns inside the failing band
  }
  if (!P.upper) {
    for (int e = tid; e < n * n; e += nthr) {
      int j = e / n, i = e - j * n;
      if (i < j || i >= lim_rows) continue;
      if (i >= band_lo && j >= band_cols) continue;
      a[i + (long long)j * P.lda] = A(i, j);
    }
  } else {
    for (int e = tid; e < n * n; e += nthr) {
      int i = e / n, j = e - i * n;
      if (i < j || i >= lim_rows) continue;
      if (i >= band_lo && j >= band_cols) continue;
      a[j + (long long)i * P.lda] = A(i, j);
    }
  }
  if (tid == 0) P.info[p] = fail ? fail + P.info_offset : 0;
}

static cudaError_t potrf_smem(double* a, long long stride, int lda, int n, int upper, int* info,
                              int info_offset, int skip_nonzero, int batch, cudaStream_t s) {
  PotrfArgs P;
  P.a = a;
  P.stride = stride;
  P.lda = lda;
  P.n = n;
  P.upper = upper;
  P.info = info;
  P.info_offset = info_offset;
  P.skip_nonzero = skip_nonzero;
  const int n8 = (n + 7) & ~7;
  P.S = smem_stride(n8);
  P.NC = n8;
  size_t smem = (size_t)P.S * P.NC * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(potrf_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         220 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int threads = n <= 24 ? 64 : (n <= 64 ? 128 : 256);
  potrf_smem_kernel<<<batch, threads, smem, s>>>(P);
  return cudaGetLastError();
}

constexpr int kPotrfSmemMax = 160;

cudaError_t potrf_launch(const PotrfLaunch& L, cudaStream_t s) {
  if (L.batch <= 0 || L.n <= 0) return cudaSuccess;
  static const int kernel = [] {  // PBGPU_POTRF_KERNEL: cta (default) | warp | smem
    const char* e = getenv("PBGPU_POTRF_KERNEL");
    if (!e) return 0;
    return e[0] == 'w' ? 1 : (e[0] == 's' ? 2 : 0);
  }();
  if (kernel == 1 && L.n <= 64)
    return potrf_warp_launch(L.a, L.stride, L.lda, L.n, L.upper, L.info, 0, 0, L.batch, s);
  static const int blocked_from = [] {  // PBGPU_POTRF_BLOCKED_FROM=n: blocked path from this order on (tuning)
    const char* e = getenv("PBGPU_POTRF_BLOCKED_FROM");
    return e ? atoi(e) : kPotrfSmemMax + 1;
  }();
  if (kernel == 0 && L.n <= kPotrfSmemMax && L.n < blocked_from)
    return potrf_cta_launch(L.a, L.stride, nullptr, nullptr, L.lda, L.n, L.upper, 0, 0, L.info, 0, 0, L.batch, s);
  if (L.n <= kPotrfSmemMax && L.n < blocked_from)
    return potrf_smem(L.a, L.stride, L.lda, L.n, L.upper, L.info, 0, 0, L.batch, s);
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
    double* a11 = L.a + (long long)c0 + (long long)c0 * L.lda;
    cudaError_t e = potrf_cta_launch(a11, L.stride, nullptr, nullptr, L.lda, w, L.upper, 0, 0, L.info, c0, c0 > 0, L.batch, s);
    if (e != cudaSuccess) return e;
    if (!rest) break;
    TrsmLaunch T;
    T.pm = 0;
    T.twin = L.upper;      // upper: rows of the effective problem are columns
    T.lower = 1;
    T.trans = 1;           // X * L11^T = A21
    T.unit = 0;
    T.mm = rest;
    T.nn = w;
    T.alpha = 1.0;
    T.a = a11; T.sa = L.stride; T.lda = L.lda;
    // Lower: A21 rows c0+w.. at (c0+w) + c0*lda.  Upper: twin view of A12 at c0 + (c0+w)*lda.
    double* b = L.upper ? L.a + (long long)c0 + (long long)(c0 + w) * L.lda
                        : L.a + (long long)(c0 + w) + (long long)c0 * L.lda;
    T.b = b; T.sb = L.stride; T.ldb = L.lda;
    T.d = b; T.sd = L.stride; T.ldd = L.lda;
    T.info = L.info;
    T.skip_nonzero = 1;
    T.batch = L.batch;
    if (L.upper) T.trans = 0, T.lower = 0;  // twin problem: X * U11 = A12^T with U11 = L11^T stored upper
    e = trsm_launch(T, s);
    if (e != cudaSuccess) return e;
    GemmLaunch g;
    double* a22 = L.a + (long long)(c0 + w) + (long long)(c0 + w) * L.lda;
    if (!L.upper) {  // A22 -= A21 A21^T  (syrk 'l','n')
      g.lay_a = g.lay_b = L_MNC;
    } else {         // A22(upper) -= A12^T A12 (syrk 'u','t')
      g.lay_a = g.lay_b = L_KC;
    }
    g.a.base = g.b.base = b;
    g.a.stride = g.b.stride = L.stride;
    g.a.ld = g.b.ld = L.lda;
    g.a.bulk = g.b.bulk = ((reinterpret_cast<uintptr_t>(b) & 15) == 0) && L.lda % 2 == 0 && L.stride % 2 == 0;
    g.o.c = a22;
    g.o.d = a22;
    g.o.sc = g.o.sd = L.stride;
    g.o.ldc = g.o.ldd = L.lda;
    g.o.vec = 0;
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
