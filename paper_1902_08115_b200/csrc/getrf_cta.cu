// Pipelined right-looking batched LU with partial pivoting, one CTA per problem
// (sm_100a).  Replaces getrf (factor.hpp:105-230) for matrices resident in
// shared memory (S * n * 8 bytes <= ~200 KB; also the tall panels of the
// blocked path).
//
// The matrix lives in shared memory, column-major, stride S = 4 mod 16 doubles
// (conflict-free DMMA fragments).  Per 8-column block k:
//   * the panel warp holds rows c0.. of the block in registers, row-per-lane
//     (R rows per lane), and factors it: pivot search as a warp argmax over
//     (|v|, row) with the reference's rule (strict '>' scan, ties to the
//     lowest row, a NaN diagonal keeps its row — factor.hpp:141-148), the row
//     exchange, reciprocal scaling, and the rank-1 update that skips zero
//     multipliers (factor.hpp:149-165); a zero pivot records the first failing
//     column, no swap, no scaling (factor.hpp:157-158);
//   * three update warps apply the block's interchanges to the columns right
//     of it, solve U12 against the unit-lower 8x8 block (factor.hpp:188-199)
//     and run the trailing update A22 -= L21 U12 on FP64 tensor cores (DMMA).
//     They finish block k+1's columns first and hand that block to the panel
//     warp (lookahead), then update the rest while panel k+1 is factored.
// Interchanges on the columns left of each block are applied once at the end
// (same order, same result as factor.hpp:175-183's eager swaps).  Loads and
// stores are per-column TMA bulk copies.
#include <cstdint>

#include "common.cuh"
#include "launch.h"

namespace pbg {

struct GetrfCtaArgs {
  double* a;
  long long stride;
  int lda, m, n;
  int* ipiv;
  long long sp;
  int* info;
  int piv_offset;
  int keep_info;
  int S;
};

__device__ __forceinline__ void gsync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// Update warps' work on columns [j0, j1) for step k: interchanges, U12 solve
// (one thread per column), then the trailing DMMA tiles of those columns.
template <int NU>
__device__ __forceinline__ void lu_update_cols(double* sm, int S, int m, int c0, int w, const int* piv,
                                               int j0, int j1, int utid, int uw, int lane) {
  constexpr int NUT = 32 * NU;
  // 1. row interchanges + unit-lower solve, one thread per column
  for (int j = j0 + utid; j < j1; j += NUT) {
    double* col = sm + (long long)j * S;
    double u[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < w) {
        const int pr = piv[c], row = c0 + c;
        if (pr != row) {
          const double x = col[row];
          col[row] = col[pr];
          col[pr] = x;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) u[c] = c < w ? col[c0 + c] : 0.0;
#pragma unroll
    for (int c = 1; c < 8; ++c)
#pragma unroll
      for (int l = 0; l < c; ++l)
        if (c < w) u[c] -= u[l] * sm[c0 + c + (long long)(c0 + l) * S];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < w) col[c0 + c] = u[c];
  }
  // the trailing tiles of these columns need the solved U12 rows of all of them
  gsync(3, NUT);
  if (w < 8) return;  // last block: nothing below/right to update
  // 2. trailing update of rows >= c0 + 8, columns [j0, j1): tiles (I, J)
  const int r0 = c0 + 8;
  if (r0 >= m) return;
  const int ti = (m - r0 + 7) >> 3, tj = (j1 - j0 + 7) >> 3;
  const int tg = (tj + 3) >> 2, nt = ti * tg;  // items: one row tile x up to 4 column tiles
  const int g = lane >> 2, t = lane & 3;
  for (int idx = uw; idx < nt; idx += NU) {  // warp-uniform loop, no predicated MMA
    const int I = idx % ti, J0 = (idx / ti) * 4;
    const int ri = r0 + I * 8;
    const double a0 = sm[ri + g + (long long)(c0 + t) * S];
    const double a1 = sm[ri + g + (long long)(c0 + 4 + t) * S];
    const int nj = min(4, tj - J0);
    // independent accumulators: the four tiles' loads, MMAs and stores overlap
    double d[4][2], b[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int cj = j0 + (J0 + u) * 8;
      d[u][0] = d[u][1] = 0.0;
      b[u][0] = u < nj ? sm[c0 + t + (long long)(cj + g) * S] : 0.0;
      b[u][1] = u < nj ? sm[c0 + 4 + t + (long long)(cj + g) * S] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      dmma(d[u][0], d[u][1], a0, b[u][0]);
      dmma(d[u][0], d[u][1], a1, b[u][1]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u < nj) {
        double* c = sm + ri + g + (long long)(j0 + (J0 + u) * 8 + 2 * t) * S;
        c[0] -= d[u][0];
        c[S] -= d[u][1];
      }
  }
}

template <int R, int NU>
__global__ void __launch_bounds__(32 * (NU + 1)) getrf_cta_kernel(const __grid_constant__ GetrfCtaArgs P) {
  constexpr int NTH = 32 * (NU + 1);
  extern __shared__ __align__(16) double sm[];
  __shared__ int piv_s[2][8];
  __shared__ int piv_all[224];  // local pivot rows (0-based) of every column
  __shared__ double scr[16];
  __shared__ int first_zero;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = P.m, n = P.n, S = P.S, minmn = min(m, n);
  const long long p = blockIdx.x;
  double* a = P.a + p * P.stride;
  int* ipiv = P.ipiv + p * P.sp;
  const bool bulk = (P.lda % 2 == 0) && (m % 2 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0);

  // ---- stage: one TMA bulk copy per column ----
  if (bulk) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(&bar, 8u * (uint32_t)m * (uint32_t)n);
      first_zero = 0;
    }
    __syncthreads();
    for (int j = tid; j < n; j += NTH) bulk_g2s(sm + (long long)j * S, a + (long long)j * P.lda, 8u * m, &bar);
    mbar_wait(&bar, 0);
  } else {
    if (tid == 0) first_zero = 0;
    stage_cm(sm, S, a, P.lda, 0, m, n, false, tid, NTH);
    cp_async_wait_all();
  }
  __syncthreads();

  const int nblk = (minmn + 7) >> 3;
  if (warp == 0) {
    // ---------------------------------------------------------------- panel warp
    for (int k = 0; k < nblk; ++k) {
      if (k > 0) gsync(2, NTH);  // block k fully updated
      const int c0 = 8 * k, w = min(8, minmn - c0), rows = m - c0;
      int* pv = piv_s[k & 1];
      double x[R][8];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int r = c0 + lane + 32 * q;
#pragma unroll
        for (int c = 0; c < 8; ++c) x[q][c] = (r < m && c < w) ? sm[r + (long long)(c0 + c) * S] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // static column index: no register-array selects
        if (c >= w) break;
        const int col = c0 + c;
        // pivot: max |v| over rows >= col, strict '>' (lowest row wins ties)
        double bv = -1.0;
        int bi = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int r = c0 + lane + 32 * q;
          const double v = fabs(x[q][c]);
          if (r >= col && r < m && v > bv) { bv = v; bi = r; }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
          if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        // col - c0 = c < 8: the diagonal row sits in slot q = 0 of lane c
        const double dg = __shfl_sync(0xffffffffu, x[0][c], c);
        int pr = bi;
        if (isnan(dg) || bi == 0x7fffffff) pr = col;
        const int lp = (pr - c0) & 31, qp = (pr - c0) >> 5;
        double pvl = 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (q == qp) pvl = x[q][c];
        const double pivv = __shfl_sync(0xffffffffu, pvl, lp);
        if (lane == 0) {
          pv[c] = pr;
          piv_all[col] = pr;
          ipiv[col] = pr + 1 + P.piv_offset;
        }
        const bool nz = pivv != 0.0;
        if (nz && pr != col) {
          // exchange panel rows col (lane c, slot 0) and pr (lane lp, slot qp)
          if (lane == c)
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) scr[cc] = x[0][cc];
#pragma unroll
          for (int q = 0; q < R; ++q)
            if (lane == lp && q == qp)
#pragma unroll
              for (int cc = 0; cc < 8; ++cc) scr[8 + cc] = x[q][cc];
          __syncwarp();
          if (lane == c)
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) x[0][cc] = scr[8 + cc];
#pragma unroll
          for (int q = 0; q < R; ++q)
            if (lane == lp && q == qp)
#pragma unroll
              for (int cc = 0; cc < 8; ++cc) x[q][cc] = scr[cc];
          __syncwarp();
        } else if (!nz && lane == 0 && first_zero == 0) {
          first_zero = col + 1;
        }
        // pivot row (after the exchange) to every lane
        double u[8];
#pragma unroll
        for (int cc = c; cc < 8; ++cc) u[cc] = __shfl_sync(0xffffffffu, x[0][cc], c);
        const double inv = nz ? 1.0 / u[c] : 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int r = c0 + lane + 32 * q;
          if (r > col && r < m) {
            if (nz) x[q][c] *= inv;
            const double f = x[q][c];
            if (f != 0.0)
#pragma unroll
              for (int c2 = c + 1; c2 < 8; ++c2)
                if (c2 < w) x[q][c2] -= f * u[c2];
          }
        }
      }
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int r = c0 + lane + 32 * q;
        if (r < m)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c < w) sm[r + (long long)(c0 + c) * S] = x[q][c];
      }
      gsync(1, NTH);  // panel k (+ its pivots) published
    }
  } else {
    // ---------------------------------------------------------------- update warps
    const int utid = tid - 32, uw = warp - 1;
    for (int k = 0; k < nblk; ++k) {
      gsync(1, NTH);  // panel k published
      const int c0 = 8 * k, w = min(8, minmn - c0);
      const int* pv = piv_s[k & 1];
      const int nb = c0 + w;  // first column right of the panel
      // lookahead: block k+1's columns first, hand it to the panel warp
      const int ahead = min(n, nb + 8);
      if (k + 1 < nblk) {
        lu_update_cols<NU>(sm, S, m, c0, w, pv, nb, ahead, utid, uw, lane);
        gsync(3, 32 * NU);
        gsync(2, NTH);  // block k+1 ready
        lu_update_cols<NU>(sm, S, m, c0, w, pv, ahead, n, utid, uw, lane);
      } else {
        lu_update_cols<NU>(sm, S, m, c0, w, pv, nb, n, utid, uw, lane);
      }
      gsync(3, 32 * NU);
    }
  }
  __syncthreads();
  // ---- deferred interchanges on the columns left of each block (pivot order) ----
  for (int j = tid; j < n; j += NTH) {
    double* col = sm + (long long)j * S;
    const int kb = j >> 3;  // block containing column j (its own swaps are done)
    for (int r = 8 * (kb + 1); r < minmn; ++r) {
      const int pr = piv_all[r];
      if (pr != r) {
        const double x = col[r];
        col[r] = col[pr];
        col[pr] = x;
      }
    }
  }
  __syncthreads();
  // ---- write back ----
  if (bulk) {
    fence_proxy_async();
    for (int j = tid; j < n; j += NTH) bulk_s2g(a + (long long)j * P.lda, smem_u32(sm + (long long)j * S), 8u * m);
    bulk_commit();
    bulk_wait_read0();
  } else {
    for (int j = 0; j < n; ++j)
      for (int i = tid; i < m; i += NTH) a[i + (long long)j * P.lda] = sm[i + (long long)j * S];
  }
  if (tid == 0) {
    const int fz = first_zero ? first_zero + P.piv_offset : 0;
    if (!P.keep_info || P.info[p] == 0) P.info[p] = fz;
  }
}

template <int R, int NU>
static cudaError_t getrf_cta_t(const GetrfCtaArgs& P, int batch, cudaStream_t s) {
  const size_t smem = (size_t)P.S * ((P.n + 7) & ~7) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(getrf_cta_kernel<R, NU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         220 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  getrf_cta_kernel<R, NU><<<(unsigned)batch, 32 * (NU + 1), smem, s>>>(P);
  return cudaGetLastError();
}

cudaError_t getrf_cta_launch(double* a, long long stride, int lda, int m, int n, int* ipiv, long long sp,
                             int* info, int piv_offset, int keep_info, int batch, cudaStream_t s) {
  GetrfCtaArgs P;
  P.a = a; P.stride = stride; P.lda = lda; P.m = m; P.n = n;
  P.ipiv = ipiv; P.sp = sp; P.info = info;
  P.piv_offset = piv_offset; P.keep_info = keep_info;
  const int m8 = (m + 7) & ~7;
  int S = ((m8 - 4 + 15) / 16) * 16 + 4;
  if (S < m8) S += 16;
  P.S = S;
  if ((size_t)S * ((n + 7) & ~7) * sizeof(double) > 220 * 1024) return cudaErrorInvalidValue;
  // update warps sized to the work: one for n <= 40, two up to 96, three above
  const int nu = n <= 40 ? 1 : (n <= 96 ? 2 : 3);
  switch ((m + 31) / 32) {
#define PB_R(RV)                                      \
  case RV:                                            \
    if (nu == 1) return getrf_cta_t<RV, 1>(P, batch, s); \
    if (nu == 2) return getrf_cta_t<RV, 2>(P, batch, s); \
    return getrf_cta_t<RV, 3>(P, batch, s);
    PB_R(1) PB_R(2) PB_R(3) PB_R(4) PB_R(5) PB_R(6) PB_R(7)
#undef PB_R
  }
  return cudaErrorInvalidValue;
}

}  // namespace pbg
