// Batched LU with partial row pivoting (dgetrf) for sm_100a.
//
// Replaces getrf (factor.hpp:105-230).  One CTA owns one problem for
// m, n <= 160: the matrix is loaded once into shared memory (column stride
// = 4 mod 16 doubles) and factored right-looking in 8-column blocks:
//   1. warp 0 factors the panel: pivot search as a warp argmax over
//      (|v|, row) with the reference's rule — strict '>' scan, ties to the
//      lowest row, a NaN diagonal keeps its row (factor.hpp:141-148); a zero
//      pivot records the first failing column and skips swap and scaling
//      (factor.hpp:151-158); scaling by the reciprocal; rank-1 updates skip
//      zero multipliers (factor.hpp:160-165);
//   2. one thread per column applies the block's row swaps outside the
//      panel in pivot order (factor.hpp:175-183) and solves its U12 column
//      against the unit-lower 8x8 block (factor.hpp:191-199);
//   3. all warps update A22 -= L21 U12 with FP64 tensor-core DMMA m8n8k4.
// Larger problems are blocked on the host side over this kernel (tall
// panels), a row-swap kernel, the trsm kernel and the DMMA gemm engine.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace pbg {

struct GetrfArgs {
  double* a;
  long long stride;
  int lda, m, n;
  int* ipiv;
  long long sp;
  int* info;
  int piv_offset;   // added to recorded pivots / failing columns (blocked callers)
  int keep_info;    // keep an earlier nonzero info (first zero pivot wins)
  int S;
};

__host__ __device__ inline int lu_stride(int rows8) {
  int s = ((rows8 - 4 + 15) / 16) * 16 + 4;
  return s < rows8 ? s + 16 : s;
}

__global__ void __launch_bounds__(256) getrf_smem_kernel(const __grid_constant__ GetrfArgs P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int piv_s[8];
  __shared__ int first_zero;
  const int p = blockIdx.x;
  const int m = P.m, n = P.n, S = P.S, tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
  const int minmn = min(m, n);
  double* a = P.a + (long long)p * P.stride;
  int* ipiv = P.ipiv + (long long)p * P.sp;
  auto A = [&](int i, int j) -> double& { return sm[i + j * S]; };

  stage_cm(sm, S, a, P.lda, 0, m, n, false, tid, nthr);
  cp_async_wait_all();
  if (tid == 0) first_zero = 0;
  __syncthreads();

  for (int c0 = 0; c0 < minmn; c0 += 8) {
    const int w = min(8, minmn - c0);
    // ---- 1. panel factorization (warp 0) ----
    if (warp == 0) {
      for (int c = 0; c < w; ++c) {
        const int col = c0 + c;
        // argmax |A(i, col)| over i >= col; strict '>' per lane keeps the lowest row
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int i = col + lane; i < m; i += 32) {
          const double v = fabs(A(i, col));
          if (v > bv) { bv = v; bi = i; }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
          if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        int piv = bi;
        const double dg = A(col, col);
        if (isnan(dg) || bi == 0x7fffffff) piv = col;  // NaN diagonal: nothing compares greater
        const double pv = A(piv, col);
        if (lane == 0) { piv_s[c] = piv; ipiv[col] = piv + 1 + P.piv_offset; }
        if (pv != 0.0) {
          if (piv != col && lane < w) {
            const double x = A(col, c0 + lane);
            A(col, c0 + lane) = A(piv, c0 + lane);
            A(piv, c0 + lane) = x;
          }
          __syncwarp();
          const double inv = 1.0 / A(col, col);
          for (int i = col + 1 + lane; i < m; i += 32) A(i, col) *= inv;
        } else if (lane == 0 && first_zero == 0) {
          first_zero = col + 1;
        }
        __syncwarp();
        for (int i = col + 1 + lane; i < m; i += 32) {
          const double f = A(i, col);
          // zero multipliers skip only the rest of the nr = 4 column block
          for (int c2 = c + 1; c2 < w; ++c2)
            if (f != 0.0 || c2 > (c | 3)) A(i, c0 + c2) -= f * A(col, c0 + c2);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // ---- 2. row swaps outside the panel + U12 solve, one thread per column ----
    for (int q = tid; q < n; q += nthr) {
      if (q >= c0 && q < c0 + w) continue;
      for (int c = 0; c < w; ++c) {
        const int pr = piv_s[c], row = c0 + c;
        if (pr != row) {
          const double x = A(row, q);
          A(row, q) = A(pr, q);
          A(pr, q) = x;
        }
      }
      if (q >= c0 + w) {
        double u[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) u[c] = c < w ? A(c0 + c, q) : 0.0;
#pragma unroll
        for (int c = 1; c < 8; ++c)
#pragma unroll
          for (int l = 0; l < c; ++l)
            if (c < w) u[c] -= u[l] * A(c0 + c, c0 + l);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < w) A(c0 + c, q) = u[c];
      }
    }
    __syncthreads();
    // ---- 3. trailing update A22 -= L21 U12 (DMMA, k = 8) ----
    const int r0 = c0 + 8;
    if (w == 8 && r0 < m && r0 < n) {
      const int g = lane >> 2, t = lane & 3;
      const int ti = (m - r0 + 7) >> 3, tj = (n - r0 + 7) >> 3;
      for (int idx = warp; idx < ti * tj; idx += nwarps) {
        const int I = idx % ti, J = idx / ti;
        const int ri = r0 + I * 8, cj = r0 + J * 8;
        double d0 = 0.0, d1 = 0.0;
        dmma(d0, d1, A(ri + g, c0 + t), A(c0 + t, cj + g));
        dmma(d0, d1, A(ri + g, c0 + 4 + t), A(c0 + 4 + t, cj + g));
        A(ri + g, cj + 2 * t) -= d0;
        A(ri + g, cj + 2 * t + 1) -= d1;
      }
    }
    __syncthreads();
  }

  for (int e = tid; e < m * n; e += nthr) {
    int j = e / m, i = e - j * m;
    a[i + (long long)j * P.lda] = A(i, j);
  }
  if (tid == 0) {
    const int fz = first_zero ? first_zero + P.piv_offset : 0;
    if (!P.keep_info || P.info[p] == 0) P.info[p] = fz;
  }
}

// Applies the row interchanges ipiv[k0 .. k1) (absolute, 1-based) to the
// columns [q0, q1) in pivot order (factor.hpp:175-183).
__global__ void laswp_kernel(double* a, long long stride, int lda, const int* ipiv, long long sp,
                             int k0, int k1, int q0, int q1) {
  const int p = blockIdx.y;
  double* ap = a + (long long)p * stride;
  const int* ip = ipiv + (long long)p * sp;
  for (int q = q0 + blockIdx.x * blockDim.x + threadIdx.x; q < q1; q += gridDim.x * blockDim.x) {
    double* col = ap + (long long)q * lda;
    for (int k = k0; k < k1; ++k) {
      const int r = ip[k] - 1;
      if (r != k) {
        const double x = col[k];
        col[k] = col[r];
        col[r] = x;
      }
    }
  }
}

static cudaError_t getrf_smem(double* a, long long stride, int lda, int m, int n, int* ipiv,
                              long long sp, int* info, int piv_offset, int keep_info, int batch,
                              cudaStream_t s) {
  GetrfArgs P;
  P.a = a;
  P.stride = stride;
  P.lda = lda;
  P.m = m;
  P.n = n;
  P.ipiv = ipiv;
  P.sp = sp;
  P.info = info;
  P.piv_offset = piv_offset;
  P.keep_info = keep_info;
  P.S = lu_stride((m + 7) & ~7);
  size_t smem = (size_t)P.S * ((n + 7) & ~7) * sizeof(double);
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  {
    cudaError_t e = smem_attr((const void*)getrf_smem_kernel, 220 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int mx = std::max(m, n);
  int threads = mx <= 32 ? 64 : (mx <= 64 ? 128 : 256);
  getrf_smem_kernel<<<batch, threads, smem, s>>>(P);
  return cudaGetLastError();
}

static bool fits_smem(int m, int n) {
  return (size_t)lu_stride((m + 7) & ~7) * ((n + 7) & ~7) * sizeof(double) <= 220 * 1024;
}

cudaError_t getrf_launch(const GetrfLaunch& L, cudaStream_t s) {
  if (L.batch <= 0 || L.m <= 0 || L.n <= 0) return cudaSuccess;
  static const bool legacy = [] {
    const char* e = getenv("PBGPU_GETRF_KERNEL");
    return e && e[0] == 's';
  }();
  if (!legacy && getrf_reg_ok(L.m, L.n))
    return getrf_reg_launch(L.a, L.stride, L.lda, L.m, L.n, L.ipiv, L.stride_ipiv, L.info, L.batch, s);
  if (!legacy && getrf_sq_ok(L.a, L.stride, L.lda, L.m, L.n))
    return getrf_sq_launch(L.a, L.stride, L.lda, L.n, L.ipiv, L.stride_ipiv, L.info, 0, 0, 0, L.batch, s);
  static const int blocked_from = [] {  // PBGPU_GETRF_BLOCKED_FROM=n: blocked path from this order on (tuning)
    const char* e = getenv("PBGPU_GETRF_BLOCKED_FROM");
    return e ? atoi(e) : 80;
  }();
  if (fits_smem(L.m, L.n) && !legacy && L.m <= 224 && std::min(L.m, L.n) < blocked_from)
    return getrf_cta_launch(L.a, L.stride, L.lda, L.m, L.n, L.ipiv, L.stride_ipiv, L.info, 0, 0, L.batch, s);
  if (fits_smem(L.m, L.n) && std::min(L.m, L.n) < blocked_from)
    return getrf_smem(L.a, L.stride, L.lda, L.m, L.n, L.ipiv, L.stride_ipiv, L.info, 0, 0, L.batch, s);
  // Blocked right-looking LU over tall panels of nb columns.
  const int minmn = std::min(L.m, L.n);
  int nb = 64;
  while (nb > 8 && !fits_smem(L.m, nb)) nb /= 2;
  if (!fits_smem(L.m, nb)) return cudaErrorInvalidValue;
  if (fits_smem(L.m, 96) && L.n <= 192) nb = 96;
  static const int nb_env = [] {  // PBGPU_GETRF_NB: tall-panel width of the row-resident path (tuning)
    const char* e = getenv("PBGPU_GETRF_NB");
    return e ? atoi(e) : 0;
  }();
  const int nbr = nb_env == 16 || nb_env == 48 || nb_env == 64 ? nb_env : 32;  // 32 measured best (n = 96, 192)
  const bool rows = !legacy && getrf_rows_ok(L.m, nbr);
  if (rows) nb = nbr;  // tall panels on the row-resident kernel
  for (int j0 = 0; j0 < minmn; j0 += nb) {
    const int jb = std::min(nb, minmn - j0);
    const int mm = L.m - j0;
    double* panel = L.a + (long long)j0 + (long long)j0 * L.lda;
    // the trailing square block, once it fits the shared-memory-resident kernel:
    // one launch, its interchanges on the columns left of it fused in
    if (j0 > 0 && L.m == L.n && !legacy && getrf_sq_ok(panel, L.stride, L.lda, mm, L.n - j0))
      return getrf_sq_launch(panel, L.stride, L.lda, mm, L.ipiv + j0, L.stride_ipiv, L.info, j0, 1, j0, L.batch, s);
    // 1. factor the tall panel rows j0.., cols j0..j0+jb (pivots offset by j0)
    cudaError_t e = rows ? getrf_rows_launch(panel, L.stride, L.lda, mm, jb, L.ipiv + j0, L.stride_ipiv, L.info, j0,
                                             j0 > 0, L.batch, j0, L.n, s)
                    : (!legacy && mm <= 224)
                        ? getrf_cta_launch(panel, L.stride, L.lda, mm, jb, L.ipiv + j0, L.stride_ipiv, L.info, j0,
                                           j0 > 0, L.batch, s)
                        : getrf_smem(panel, L.stride, L.lda, mm, jb, L.ipiv + j0, L.stride_ipiv, L.info, j0,
                                     j0 > 0, L.batch, s);
    if (e != cudaSuccess) return e;
    // 2. apply the panel's interchanges to the columns left and right of it
    //    (the row-resident panel kernel already moved whole rows)
    dim3 grid(std::max(1, (std::max(j0, L.n - j0 - jb) + 127) / 128), L.batch);
    if (j0 > 0 && !rows) {
      laswp_kernel<<<grid, 128, 0, s>>>(L.a, L.stride, L.lda, L.ipiv, L.stride_ipiv, j0, j0 + jb, 0, j0);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    const int nw = L.n - j0 - jb;
    if (nw <= 0) continue;
    if (!rows) {
      laswp_kernel<<<grid, 128, 0, s>>>(L.a, L.stride, L.lda, L.ipiv, L.stride_ipiv, j0, j0 + jb,
                                        j0 + jb, L.n);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // 3. U12 = L11^{-1} A12 (left, lower, no-trans, unit) = transposed right-side problem
    double* a12 = L.a + (long long)j0 + (long long)(j0 + jb) * L.lda;
    TrsmLaunch T;
    T.pm = 0;
    T.twin = 1;
    T.lower = 1;
    T.trans = 1;  // flip(NoTrans)
    T.unit = 1;
    T.mm = nw;
    T.nn = jb;
    T.alpha = 1.0;
    T.a = panel; T.sa = L.stride; T.lda = L.lda;
    T.b = a12; T.sb = L.stride; T.ldb = L.lda;
    T.d = a12; T.sd = L.stride; T.ldd = L.lda;
    T.info = nullptr;
    T.batch = L.batch;
    e = trsm_launch(T, s);
    if (e != cudaSuccess) return e;
    // 4. A22 -= L21 U12
    const int m2 = L.m - j0 - jb;
    if (m2 <= 0) continue;
    GemmLaunch g;
    g.lay_a = L_MNC;  // L21 (m2 x jb), column-major
    g.lay_b = L_KC;   // U12 (jb x nw), column-major: (x = q, l) at l + q*lda
    const bool al = L.lda % 2 == 0 && L.stride % 2 == 0;
    const double* l21 = panel + jb;
    g.a.base = l21; g.a.stride = L.stride; g.a.ld = L.lda;
    g.a.bulk = al && ((reinterpret_cast<uintptr_t>(l21) & 15) == 0);
    g.b.base = a12; g.b.stride = L.stride; g.b.ld = L.lda;
    g.b.bulk = al && ((reinterpret_cast<uintptr_t>(a12) & 15) == 0);
    double* a22 = a12 + jb;
    g.o.c = a22; g.o.d = a22;
    g.o.sc = g.o.sd = L.stride;
    g.o.ldc = g.o.ldd = L.lda;
    g.o.vec = al && ((reinterpret_cast<uintptr_t>(a22) & 15) == 0);
    g.m = m2; g.n = nw; g.k = jb;
    g.alpha = -1.0; g.beta = 1.0;
    g.batch = L.batch;
    e = gemm_launch(g, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace pbg
