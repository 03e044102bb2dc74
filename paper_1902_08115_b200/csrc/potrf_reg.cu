// Register-resident batched Cholesky for small orders, n <= 32 (sm_100a).
//
// The small-n branch of the size switch (the paper's small-size algorithm
// family; the reference's potrf_core, factor.hpp:45-99, with its edge
// kernels edge_potrf / edge_trsm_right, micro_kernel.hpp:309-356).  A
// segment of W = 8, 16 or 32 lanes owns one problem (4, 2 or 1 problems per
// warp): lane i holds row i of the lower triangle in registers (N doubles),
// loaded column by column so every column is one coalesced access.  The
// factorization is right-looking over columns c:
//   * each lane publishes its current a(i, c) to a per-warp shared column
//     buffer (double-buffered by column parity: no write-after-read hazard);
//   * every lane reads the pivot and the column below it back as broadcast
//     loads, forms inv = rsqrt(pivot) (failure test `piv <= 0.0`,
//     micro_kernel.hpp:314), scales its own entry, and applies the rank-1
//     update a(i, c2) -= l(i, c) * a(c2, c) * inv to the columns right of c.
// No shuffles, no barriers beyond __syncwarp, no shared-memory copy of the
// matrix: occupancy is bounded by registers only.  Rows past n are identity
// padding.  On a failure at column p only the reference's write set is
// stored (rows < 8*floor((p-1)/8) + 8 of columns < 4*floor((p-1)/4); see
// potrf_cta.cu and test_factor.cpp:251-277): those entries are final when
// column p-1 fails, everything right of it is never written.
#include <cstdint>

#include "common.cuh"
#include "launch.h"

namespace pbg {

struct PotrfRegArgs {
  double* a;
  long long stride;
  const long long* offs;  // optional per-problem element offsets (variable batches)
  const int* nvec;        // optional per-problem order (variable batches)
  int lda, n, upper, batch, zero_fill;
  int* info;
  int info_offset;
  int skip_nonzero;
};

constexpr int kRegWarps = 4;

// CS != 0: compile-time column stride (packed column-major lower problems,
// lda == n == N): every access is the row pointer plus an immediate offset.
#ifndef PB_REG_LATE_FROM
#define PB_REG_LATE_FROM 32
#endif
#ifndef PB_REG_BLOCKS32
#define PB_REG_BLOCKS32 4
#endif
template <int N, int W, int PM, int CS, int RR>
__global__ void __launch_bounds__(32 * kRegWarps, (N >= 32 ? PB_REG_BLOCKS32 : 4)) potrf_reg_kernel(const __grid_constant__ PotrfRegArgs P) {
  // RR rows per lane: lane i of a W-lane segment owns rows i, i + W, ... (N <= W * RR)
  static_assert(N <= W * RR && W <= 32 && 32 % W == 0, "segment shape");
  constexpr int SEGS = 32 / W;
  __shared__ __align__(16) double colbuf[kRegWarps][2][32 * RR];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = lane % W, seg = lane / W;
  const long long p = ((long long)blockIdx.x * kRegWarps + warp) * SEGS + seg;
  const bool live = p < P.batch && !(P.skip_nonzero && P.info[p] != 0);
  const int n = live ? (P.nvec ? P.nvec[p] : P.n) : 0;
  double* a = P.a + (live ? (P.offs ? P.offs[p] : p * P.stride) : 0);
  const long long lda = CS ? CS : (P.nvec ? (PM ? ((n + 3) & ~3) : n) : P.lda);
  const long long cs = CS ? CS : (PM ? 4 : (P.upper ? 1 : lda));
  // element (r, j) of the lower problem is rowp(r)[j * cs] in all three storage kinds
  auto rowp = [&](int r) -> double* {
    return a + (PM ? (long long)(r >> 2) * 4 * lda + (r & 3) : ((!CS && P.upper) ? (long long)r * lda : r));
  };
  double x[RR][N];
#pragma unroll
  for (int q = 0; q < RR; ++q) {
    const int r = i + W * q;
    double* rp = rowp(r);
#pragma unroll
    for (int j = 0; j < N; ++j) x[q][j] = ldg_if(rp + j * cs, j <= r && r < n, r == j ? 1.0 : 0.0);
  }

  const uint32_t buf0 = smem_u32(&colbuf[warp][0][seg * W * RR]);
  unsigned bad = 0;   // bit c: column c's pivot failed the test
  unsigned infp = 0;  // bit c: column c's pivot is +Inf (L_cc = sqrt(+Inf) = +Inf, not Inf * 0)
#pragma unroll
  for (int c = 0; c < N; ++c) {
    const uint32_t buf = buf0 + (c & 1) * 32 * RR * 8;
#pragma unroll
    for (int q = 0; q < RR; ++q) sts64(buf + 8u * (i + W * q), x[q][c]);
    __syncwarp();
    // N >= 32: only the pivot now, the multipliers a(c2, c) are read pair by pair next to
    // their use — holding the whole column would cost 64 registers and a resident CTA
    constexpr bool LATE = N >= PB_REG_LATE_FROM;
    double col[N];
    if constexpr (LATE) {
      col[c] = lds64(buf + 8u * c);
    } else {
#pragma unroll
      for (int c2 = c & ~1; c2 < N; c2 += 2) lds128(buf + 8u * c2, col[c2], col[c2 + 1]);
    }
    const double piv = col[c];  // == x[.][c] on the row c
    bad |= (piv <= 0.0 ? 1u : 0u) << c;
    infp |= (piv == __longlong_as_double(0x7ff0000000000000LL) ? 1u : 0u) << c;
    double inv = rsqrt_nb(piv);
    // denormal / +inf pivots: CUDA's full rsqrt (within 1 ulp of the reference's 1 / sqrt(piv))
    if (__any_sync(0xffffffffu, rsqrt_special(piv))) inv = rsqrt_special(piv) ? rsqrt(piv) : inv;
    if constexpr (LATE) {
      static_assert(!LATE || RR == 1, "late multiplier loads are written for one row per lane");
      x[0][c] *= inv;
      const double t = x[0][c] * inv;
#pragma unroll
      for (int c2 = (c + 1) & ~1; c2 < N; c2 += 2) {
        double u0, u1;
        lds128(buf + 8u * c2, u0, u1);
        if (c2 > c) x[0][c2] = fma(-t, u0, x[0][c2]);
        x[0][c2 + 1] = fma(-t, u1, x[0][c2 + 1]);
      }
    } else {
#pragma unroll
      for (int q = 0; q < RR; ++q) {
        x[q][c] *= inv;
        const double t = x[q][c] * inv;
#pragma unroll
        for (int c2 = c + 1; c2 < N; ++c2) x[q][c2] = fma(-t, col[c2], x[q][c2]);
      }
    }
  }
  const unsigned nmask = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
  const int fail = __ffs(bad & nmask);  // first failing column, 1-based (0: none)

  // ---- write back: the reference's write set, coalesced column by column ----
  if (n > 0) {
    int band_lo = n, ncols = n;
    if (fail) {
      band_lo = ((fail - 1) / 8) * 8 + 8;
      ncols = ((fail - 1) / 4) * 4;
    }
#pragma unroll
    for (int q = 0; q < RR; ++q) {
      const int r = i + W * q;
      const bool row_ok = r < n && r < band_lo;
      double* wp = rowp(r);
      if (CS) {
#pragma unroll
        for (int j = 0; j < N; ++j) stg_if(wp + j * CS, x[q][j], row_ok && j <= r && j < ncols);
      } else {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const bool lower = j <= r;
          const bool zero = P.zero_fill && r < j && (r >> 3) == (j >> 3);
          stg_if(wp, lower ? x[q][j] : 0.0, row_ok && j < ncols && (lower || zero));
          wp += cs;
        }
      }
      // +Inf pivots (rare): the diagonal is sqrt(+Inf) = +Inf, not the Inf * 0 in x
      if ((infp >> r) & 1u && row_ok && r < ncols)
        rowp(r)[(long long)r * cs] = __longlong_as_double(0x7ff0000000000000LL);
    }
    if (i == 0) P.info[p] = fail ? fail + P.info_offset : 0;
  } else if (live && i == 0) {
    P.info[p] = 0;
  }
}

template <int N, int W, int PM, int RR = 1>
static cudaError_t reg_launch_t(const PotrfRegArgs& P, cudaStream_t s) {
  constexpr int per_cta = kRegWarps * (32 / W);
  const unsigned grid = (unsigned)((P.batch + per_cta - 1) / per_cta);
  if constexpr (!PM) {
    if (!P.upper && !P.nvec && !P.offs && !P.zero_fill && P.n == N && P.lda == N) {
      potrf_reg_kernel<N, W, 0, N, RR><<<grid, 32 * kRegWarps, 0, s>>>(P);
      return cudaGetLastError();
    }
  }
  potrf_reg_kernel<N, W, PM, 0, RR><<<grid, 32 * kRegWarps, 0, s>>>(P);
  return cudaGetLastError();
}

template <int PM>
static cudaError_t reg_dispatch(const PotrfRegArgs& P, int nmax, cudaStream_t s) {
  if (nmax <= 4) return reg_launch_t<4, 8, PM>(P, s);
  if (nmax <= 8) return reg_launch_t<8, 8, PM>(P, s);
  if (nmax <= 12) return reg_launch_t<12, 16, PM>(P, s);
  if (nmax <= 16) return reg_launch_t<16, 8, PM, 2>(P, s);  // two rows per lane, four problems per warp
  if (nmax <= 24) return reg_launch_t<24, 32, PM>(P, s);
  if (nmax <= 32) return reg_launch_t<32, 32, PM>(P, s);
  return cudaErrorInvalidValue;
}

cudaError_t potrf_reg_launch(double* a, long long stride, const long long* offs, const int* nvec, int lda, int nmax,
                             int upper, int pm, int zero_fill, int* info, int info_offset, int skip_nonzero,
                             int batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  PotrfRegArgs P{a, stride, offs, nvec, lda, nmax, upper, batch, zero_fill, info, info_offset, skip_nonzero};
  return pm ? reg_dispatch<1>(P, nmax, s) : reg_dispatch<0>(P, nmax, s);
}

}  // namespace pbg
