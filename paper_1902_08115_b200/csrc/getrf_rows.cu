// Row-resident batched LU with partial pivoting for mid-size problems
// (m <= 32*NW rows, n <= N columns; sm_100a).
//
// Replaces getrf (factor.hpp:105-230) for the config-4 orders that do not fit
// one warp.  One CTA of NW warps owns one problem and every thread holds ONE
// ORIGINAL row of it in registers for the whole factorization; rows never
// move.  Interchanges are tracked as each row's current LAPACK position
// (LAPACK's swap of positions c and q is two register updates), so the only
// data that crosses threads per column is the pivot row.  Per column c:
//   * each warp reduces its candidates with the reference's rule
//     (factor.hpp:141-148: strict '>' scan from the diagonal, ties to the
//     lowest current position, a NaN diagonal keeps its row, NaN candidates
//     never win) as three redux.sync reductions over the non-negative
//     doubles' bit patterns plus a vote;
//   * every warp's winner publishes its row (columns c..) and key in shared
//     memory, and ONE CTA barrier later every thread picks the global winner
//     from the NW keys and reads that row back as broadcast loads;
//   * a nonzero pivot scales the rows below by its correctly rounded
//     reciprocal (factor.hpp:149-156; a zero pivot records the first zero
//     column and neither swaps nor scales, 157-158) and the rank-1 update
//     skips zero multipliers (160-165).
// At the end every row is stored at its final position, with ipiv (1-based)
// and info.  Tall panels of the blocked path (n > the resident orders) use
// the same kernel with pivot / info offsets.
#include <cstdint>

#include "common.cuh"
#include "launch.h"

namespace pbg {

struct GetrfRowsArgs {
  double* a;
  long long stride;
  int lda, m, n;
  int* ipiv;
  long long sp;
  int* info;
  int piv_offset;
  int keep_info;  // keep an info already set by an earlier panel
  int batch;
  // tall panels of the blocked path: the panel is columns [col0, col0 + n) of a
  // matrix with ncols columns; its interchanges are applied to all the others
  int col0, ncols;
};

template <int N, int NW>
__global__ void __launch_bounds__(32 * NW) getrf_rows_kernel(const __grid_constant__ GetrfRowsArgs P) {
  constexpr int NP = (N + 1) & ~1;
  __shared__ __align__(16) double cand[2][NW][NP];  // every warp's candidate pivot row
  __shared__ uint4 kbuf[2][NW];                     // its key: {hi, lo, position, NaN-diagonal flag}
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const long long p = blockIdx.x;
  const int m = P.m, n = P.n, minmn = min(m, n);
  double* a = P.a + p * P.stride;
  const long long lda = P.lda;
  const int r = tid;  // this thread's original row

  double x[N];
#pragma unroll
  for (int j = 0; j < N; ++j) x[j] = ldg_if(a + r + j * lda, r < m && j < n, 0.0);

  int pos = r;
  bool done = r >= m;
  int my_ipiv = 0, first_zero = 0;
#pragma unroll (N)
  for (int c = 0; c < N; ++c) {
    if (c >= minmn) continue;  // uniform (no break: the loop must stay fully unrolled)
    const int b = c & 1;
    // ---- warp-level candidate ----
    const double v = fabs(x[c]);
    const unsigned long long key = (done || isnan(v)) ? 0ull : (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned khi = __reduce_max_sync(0xffffffffu, done ? 0u : hi);
    const unsigned klo = __reduce_max_sync(0xffffffffu, !done && hi == khi ? lo : 0u);
    const unsigned wq = __reduce_min_sync(0xffffffffu, !done && hi == khi && lo == klo ? (unsigned)pos : 0xffffffffu);
    const bool is_dnan = !done && pos == c && isnan(x[c]);
    const bool wnan = __any_sync(0xffffffffu, is_dnan);
    const bool wwin = wnan ? is_dnan : (!done && (unsigned)pos == wq);
    if (wwin) {
#pragma unroll
      for (int j = c & ~1; j < N; j += 2) sts128(smem_u32(&cand[b][warp][j]), x[j], x[j + 1]);
      kbuf[b][warp] = make_uint4(wnan ? 0u : khi, wnan ? 0u : klo, wnan ? (unsigned)c : wq, wnan ? 1u : 0u);
    } else if (lane == 0 && wq == 0xffffffffu && !wnan) {
      kbuf[b][warp] = make_uint4(0u, 0u, 0xffffffffu, 0u);  // no candidate rows left in this warp
    }
    __syncthreads();
    // ---- global winner ----
    int w = 0;
    uint4 best = kbuf[b][0];
#pragma unroll
    for (int u = 1; u < NW; ++u) {
      const uint4 k = kbuf[b][u];
      const bool better = best.w == 0u && (k.w != 0u || k.x > best.x || (k.x == best.x && (k.y > best.y ||
                                                                       (k.y == best.y && k.z < best.z))));
      best = better ? k : best;
      w = better ? u : w;
    }
    const int pr = (int)best.z;
    const uint32_t urow = smem_u32(&cand[b][w][0]);
    const double upiv = lds64(urow + 8u * c);
    const bool nz = upiv != 0.0;
    if (tid == c) my_ipiv = pr + 1 + P.piv_offset;
    if (!nz && first_zero == 0) first_zero = c + 1;
    // ---- interchange (positions only) ----
    if (nz && !done) pos = pos == pr ? c : (pos == c ? pr : pos);
    const bool act = !done && pos != c;
    done = done || pos == c;
    // ---- scale and rank-1 update of the rows below ----
    if (act) {
      if (nz) x[c] *= __drcp_rn(upiv);
      const double f = x[c];
      // zero multipliers are skipped only inside the reference's nr = 4 column
      // block (factor.hpp:160-165); later blocks get the plain trailing update
      // (207-215), where 0 * Inf = NaN reaches them
      const bool fz = f == 0.0;
      // pivot row pairs loaded next to their use (volatile loads stay in
      // place): the live set is the row plus one pair, not two rows
#pragma unroll
      for (int j = (c + 1) & ~1; j < N; j += 2) {
        if (fz && j + 1 <= (c | 3)) continue;
        double u0, u1;
        lds128(urow + 8u * j, u0, u1);
        if (j >= c + 1 && !(fz && j <= (c | 3))) x[j] = fma(-f, u0, x[j]);
        x[j + 1] = fma(-f, u1, x[j + 1]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < N; ++j) stg_if(a + pos + j * lda, x[j], r < m && j < n);
  // the panel's interchanges on the other columns of the rows (LAPACK applies
  // them to the whole row; the reference, factor.hpp:175-183): every row moves
  // from its original position to its final one, 16 columns per round, reads
  // and writes separated by barriers (the moves form a permutation)
  if (P.ncols > n) {
    const bool mv = r < m && pos != r;
    const int lo = -P.col0, hi = P.ncols - P.col0;  // column range relative to the panel
    for (int q0 = lo; q0 < hi; q0 += 16) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int q = q0 + u;
        const bool ok = mv && q < hi && (q < 0 || q >= n);
        v[u] = ldg_if(a + r + (long long)q * lda, ok, 0.0);
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int q = q0 + u;
        stg_if(a + pos + (long long)q * lda, v[u], mv && q < hi && (q < 0 || q >= n));
      }
      __syncthreads();
    }
  }
  if (tid < minmn) P.ipiv[p * P.sp + tid] = my_ipiv;
  if (tid == 0) {
    const int fz = first_zero ? first_zero + P.piv_offset : 0;
    if (!P.keep_info || P.info[p] == 0) P.info[p] = fz;
  }
}

template <int N, int NW>
static cudaError_t rows_t(const GetrfRowsArgs& P, cudaStream_t s) {
  getrf_rows_kernel<N, NW><<<(unsigned)P.batch, 32 * NW, 0, s>>>(P);
  return cudaGetLastError();
}

bool getrf_rows_ok(int m, int n) { return m >= 1 && n >= 1 && m <= 224 && n <= 96 && !(n > 64 && m > 96); }

cudaError_t getrf_rows_launch(double* a, long long stride, int lda, int m, int n, int* ipiv, long long sp, int* info,
                              int piv_offset, int keep_info, int batch, int col0, int ncols, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  GetrfRowsArgs P{a, stride, lda, m, n, ipiv, sp, info, piv_offset, keep_info, batch, col0, ncols};
  const int nw = (m + 31) / 32;
  if (n <= 16) {
    switch (nw) {
      case 1: return rows_t<16, 1>(P, s);
      case 2: return rows_t<16, 2>(P, s);
      case 3: return rows_t<16, 3>(P, s);
      case 4: return rows_t<16, 4>(P, s);
      case 5: return rows_t<16, 5>(P, s);
      case 6: return rows_t<16, 6>(P, s);
      case 7: return rows_t<16, 7>(P, s);
    }
  } else if (n <= 32) {
    switch (nw) {
      case 1: return rows_t<32, 1>(P, s);
      case 2: return rows_t<32, 2>(P, s);
      case 3: return rows_t<32, 3>(P, s);
      case 4: return rows_t<32, 4>(P, s);
      case 5: return rows_t<32, 5>(P, s);
      case 6: return rows_t<32, 6>(P, s);
      case 7: return rows_t<32, 7>(P, s);
    }
  } else if (n <= 48) {
    switch (nw) {
      case 1: return rows_t<48, 1>(P, s);
      case 2: return rows_t<48, 2>(P, s);
      case 3: return rows_t<48, 3>(P, s);
      case 4: return rows_t<48, 4>(P, s);
      case 5: return rows_t<48, 5>(P, s);
      case 6: return rows_t<48, 6>(P, s);
      case 7: return rows_t<48, 7>(P, s);
    }
  } else if (n <= 64) {
    switch (nw) {
      case 1: return rows_t<64, 1>(P, s);
      case 2: return rows_t<64, 2>(P, s);
      case 3: return rows_t<64, 3>(P, s);
      case 4: return rows_t<64, 4>(P, s);
      case 5: return rows_t<64, 5>(P, s);
      case 6: return rows_t<64, 6>(P, s);
      case 7: return rows_t<64, 7>(P, s);
    }
  } else {
    switch (nw) {
      case 1: return rows_t<96, 1>(P, s);
      case 2: return rows_t<96, 2>(P, s);
      case 3: return rows_t<96, 3>(P, s);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace pbg
