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
#include <cstdlib>

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
  __shared__ __align__(16) double scr[16];
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
    // Rows never move inside the panel: each register slot tracks its row's
    // current LAPACK position, a pivot step updates two positions, and the
    // panel is written back at the final positions (the same result as the
    // reference's sequential swaps, factor.hpp:149-156).
    const uint32_t ubuf0 = smem_u32(&scr[0]);
    for (int k = 0; k < nblk; ++k) {
      if (k > 0) gsync(2, NTH);  // block k fully updated
      const int c0 = 8 * k, w = min(8, minmn - c0);
      int* pv = piv_s[k & 1];
      double x[R][8];
      int pos[R];
      bool done[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int r = c0 + lane + 32 * q;
        pos[q] = r;
        done[q] = r >= m;
#pragma unroll
        for (int c = 0; c < 8; ++c) x[q][c] = (r < m && c < w) ? sm[r + (long long)(c0 + c) * S] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // static column index: no register-array selects
        if (c >= w) break;
        const int col = c0 + c;
        // pivot: max |v| (NaN never wins), ties to the lowest position, as
        // three reductions over the non-negative doubles' bit patterns
        unsigned long long bk = 0;
        unsigned bp = 0xffffffffu;
        bool dnan = false;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const double v = fabs(x[q][c]);
          const unsigned long long key = isnan(v) ? 0ull : (unsigned long long)__double_as_longlong(v);
          const bool better = !done[q] && (key > bk || (key == bk && (unsigned)pos[q] < bp));
          bk = better ? key : bk;
          bp = better ? (unsigned)pos[q] : bp;
          dnan |= !done[q] && pos[q] == col && isnan(v);
        }
        const bool has = bp != 0xffffffffu;
        const unsigned hi = (unsigned)(bk >> 32), lo = (unsigned)bk;
        const unsigned khi = __reduce_max_sync(0xffffffffu, has ? hi : 0u);
        const unsigned klo = __reduce_max_sync(0xffffffffu, has && hi == khi ? lo : 0u);
        const unsigned q0 = __reduce_min_sync(0xffffffffu, has && hi == khi && lo == klo ? bp : 0xffffffffu);
        const int pr = __any_sync(0xffffffffu, dnan) ? col : (int)q0;  // a NaN diagonal keeps its row
        // pivot row (from c, pairs) to every lane through shared scratch
        const uint32_t ub = ubuf0 + (c & 1) * 64;
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (!done[q] && pos[q] == pr)
#pragma unroll
            for (int cc = c & ~1; cc < 8; cc += 2) sts128(ub + 8u * cc, x[q][cc], x[q][cc + 1]);
        __syncwarp();
        double u[8];
#pragma unroll
        for (int cc = c & ~1; cc < 8; cc += 2) lds128(ub + 8u * cc, u[cc], u[cc + 1]);
        const bool nz = u[c] != 0.0;
        if (lane == 0) {
          pv[c] = pr;
          piv_all[col] = pr;
          ipiv[col] = pr + 1 + P.piv_offset;
          if (!nz && first_zero == 0) first_zero = col + 1;
        }
        const double inv = nz ? __drcp_rn(u[c]) : 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (nz && !done[q]) pos[q] = pos[q] == pr ? col : (pos[q] == col ? pr : pos[q]);
          const bool act = !done[q] && pos[q] != col;
          done[q] = done[q] || pos[q] == col;
          if (act) {
            if (nz) x[q][c] *= inv;
            const double f = x[q][c];
            // zero multipliers skip only the rest of the nr = 4 column block
            // (factor.hpp:160-165); the next block takes the plain update
#pragma unroll
            for (int c2 = c + 1; c2 < 8; ++c2)
              if (f != 0.0 || c2 > (c | 3)) x[q][c2] = fma(-f, u[c2], x[q][c2]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int r = c0 + lane + 32 * q;
        if (r < m)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c < w) sm[pos[q] + (long long)(c0 + c) * S] = x[q][c];
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
  {
    cudaError_t e = smem_attr((const void*)getrf_cta_kernel<R, NU>, 220 * 1024);
    if (e != cudaSuccess) return e;
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
  // update warps sized to the work (measured, tools/sweep_getrf_nu.sh): one up
  // to n = 48, three above (PBGPU_GETRF_NU = 1|2|3|5|7 overrides, tuning only)
  static const int nu_env = [] {
    const char* e = getenv("PBGPU_GETRF_NU");
    return e ? atoi(e) : 0;
  }();
  const int nu = nu_env ? nu_env : (n <= 48 ? 1 : 3);
  switch ((m + 31) / 32) {
#define PB_R(RV)                                      \
  case RV:                                            \
    if (nu == 1) return getrf_cta_t<RV, 1>(P, batch, s); \
    if (nu == 2) return getrf_cta_t<RV, 2>(P, batch, s); \
    if (nu == 5) return getrf_cta_t<RV, 5>(P, batch, s); \
    if (nu == 7) return getrf_cta_t<RV, 7>(P, batch, s); \
    return getrf_cta_t<RV, 3>(P, batch, s);
    PB_R(1) PB_R(2) PB_R(3) PB_R(4) PB_R(5) PB_R(6) PB_R(7)
#undef PB_R
  }
  return cudaErrorInvalidValue;
}

}  // namespace pbg
