// Register-resident batched LU with partial pivoting, m, n <= 32 (sm_100a).
//
// The small-n branch for getrf (factor.hpp:105-230).  One warp owns one
// problem; lane i holds ORIGINAL row i in registers and never moves: row
// interchanges are tracked as each lane's current position `pos` (LAPACK's
// physical swap of positions c and q becomes two register updates), so a
// pivot step costs no data movement.  Per column c:
//   * pivot search over the rows not yet chosen — the reference's rule
//     (factor.hpp:141-148: strict '>' scan from the diagonal, ties to the
//     lowest current position, a NaN diagonal keeps its row, NaN candidates
//     never win) as three warp reductions on the non-negative doubles' bit
//     patterns (redux.sync max of the high word, max of the low word among
//     the high-word winners, min of the position among the full winners),
//     plus a vote for the NaN-diagonal case;
//   * the pivot row is broadcast through a per-warp shared buffer;
//   * a nonzero pivot scales the rows below by its correctly rounded
//     reciprocal (factor.hpp:149-156), a zero pivot records the first zero
//     column and neither swaps nor scales (157-158);
//   * the rank-1 update skips zero multipliers (160-165).
// At the end every lane stores its row at its final position (columns stay
// coalesced: the positions are a permutation of the lanes), ipiv (1-based)
// and info (first zero pivot).
#include <cstdint>

#include "common.cuh"
#include "launch.h"

namespace pbg {

struct GetrfRegArgs {
  double* a;
  long long stride;
  int lda, m, n;
  int* ipiv;
  long long sp;
  int* info;
  int batch;
};

constexpr int kLuRegWarps = 4;

// LD != 0: compile-time leading dimension (packed square problems, lda == m == n == N)
#ifndef PB_LUREG_MINB
#define PB_LUREG_MINB 7
#endif
template <int N, int LD>
__global__ void __launch_bounds__(32 * kLuRegWarps, N <= 24 ? PB_LUREG_MINB : 4) getrf_reg_kernel(const __grid_constant__ GetrfRegArgs P) {
  __shared__ __align__(16) double rowbuf[kLuRegWarps][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p = (long long)blockIdx.x * kLuRegWarps + warp;
  if (p >= P.batch) return;  // warp-uniform
  const int m = LD ? LD : P.m, n = LD ? LD : P.n, minmn = min(m, n);
  double* a = P.a + p * P.stride;
  const long long lda = LD ? LD : P.lda;

  double x[N];
#pragma unroll
  for (int j = 0; j < N; ++j) x[j] = ldg_if(a + lane + j * lda, lane < m && j < n, 0.0);

  int pos = lane;          // current (LAPACK) position of this lane's row
  bool done = lane >= m;   // chosen as a pivot already (or not a row at all)
  int my_ipiv = 0, first_zero = 0;
  const uint32_t buf0 = smem_u32(&rowbuf[warp][0][0]);
#pragma unroll
  for (int c = 0; c < N; ++c) {
    if (c >= minmn) break;  // uniform
    // ---- pivot search ----
    const double v = fabs(x[c]);
    const unsigned long long key = (done || isnan(v)) ? 0ull : (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned khi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned klo = __reduce_max_sync(0xffffffffu, hi == khi && !done ? lo : 0u);
    const bool win = !done && hi == khi && lo == klo;
    const unsigned q0 = __reduce_min_sync(0xffffffffu, win ? (unsigned)pos : 0xffffffffu);
    const bool diag_nan = __any_sync(0xffffffffu, !done && pos == c && isnan(x[c]));
    const int q = diag_nan ? c : (int)q0;
    const bool is_piv = !done && pos == q;
    // ---- pivot row to every lane ----
    const uint32_t buf = buf0 + (c & 1) * 32 * 8;
    if (is_piv) {
#pragma unroll
      for (int j = c & ~1; j < N; j += 2) sts128(buf + 8u * j, x[j], x[j + 1]);
    }
    __syncwarp();
    const double pv = lds64(buf + 8u * c);
    const bool nz = pv != 0.0;
    if (lane == c) my_ipiv = q + 1;
    if (!nz && first_zero == 0) first_zero = c + 1;
    // ---- interchange (positions only) ----
    if (nz) {
      if (is_piv) pos = c;
      else if (!done && pos == c) pos = q;
    }
    done = done || is_piv;
    // ---- scale and rank-1 update of the rows below ----
    if (!done) {
      if (nz) x[c] *= __drcp_rn(pv);
      const double f = x[c];
      // zero multipliers skip only the rest of the reference's nr = 4 column
      // block (factor.hpp:160-165); later blocks take the plain trailing
      // update (207-215), where 0 * Inf = NaN
      // pivot row pairs loaded next to their use (volatile loads stay in place):
      // the live set is the row plus one pair, not two rows
      const bool fz = f == 0.0;
#pragma unroll
      for (int j = (c + 1) & ~1; j < N; j += 2) {
        if (fz && j + 1 <= (c | 3)) continue;
        double u0, u1;
        lds128(buf + 8u * j, u0, u1);
        if (j >= c + 1 && !(fz && j <= (c | 3))) x[j] = fma(-f, u0, x[j]);
        x[j + 1] = fma(-f, u1, x[j + 1]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < N; ++j) stg_if(a + pos + j * lda, x[j], lane < m && j < n);
  if (lane < minmn) P.ipiv[p * P.sp + lane] = my_ipiv;
  if (lane == 0) P.info[p] = first_zero;
}

template <int N>
static cudaError_t lu_reg_t(const GetrfRegArgs& P, cudaStream_t s) {
  const unsigned grid = (unsigned)((P.batch + kLuRegWarps - 1) / kLuRegWarps);
  if (P.m == N && P.n == N && P.lda == N)
    getrf_reg_kernel<N, N><<<grid, 32 * kLuRegWarps, 0, s>>>(P);
  else
    getrf_reg_kernel<N, 0><<<grid, 32 * kLuRegWarps, 0, s>>>(P);
  return cudaGetLastError();
}

bool getrf_reg_ok(int m, int n) { return m >= 1 && n >= 1 && m <= 32 && n <= 32; }

cudaError_t getrf_reg_launch(double* a, long long stride, int lda, int m, int n, int* ipiv, long long sp, int* info,
                             int batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  GetrfRegArgs P{a, stride, lda, m, n, ipiv, sp, info, batch};
  if (n <= 8) return lu_reg_t<8>(P, s);
  if (n <= 16) return lu_reg_t<16>(P, s);
  if (n <= 24) return lu_reg_t<24>(P, s);
  if (n <= 32) return lu_reg_t<32>(P, s);
  return cudaErrorInvalidValue;
}

}  // namespace pbg
