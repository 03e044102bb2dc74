// Warp-per-problem, register-resident batched Cholesky for n <= 64 (sm_100a).
//
// The small-n branch of the size switch (the paper's small-size algorithm
// family; factor.hpp:45-99 on the reference side).  One warp owns one
// problem; the lower triangle lives in registers as DMMA m8n8k4 accumulator
// fragments of 8x8 tiles (lane 4g+t holds rows g, columns 2t and 2t+1 of
// every tile), so the whole right-looking factorization runs without shared
// memory and without block barriers:
//   1. diagonal tile: column by column with warp shuffles — pivot broadcast,
//      sqrt and reciprocal, scaled column, rank-1 update; failure is the
//      reference's `piv <= 0.0` (micro_kernel.hpp:314);
//   2. panel tiles X L^T = B by substitution (4-lane group reductions,
//      reciprocal scaling as edge_trsm_right);
//   3. trailing lower update A22 -= L21 L21^T straight into the accumulator
//      registers with FP64 tensor-core DMMA (A fragments = negated panel).
// Padding rows/columns (n % 8 != 0) are identity-padded.  On failure at
// column p the write-back reproduces the reference's stored set: all lower
// entries of rows < 8*floor(p/8) and, in that band, columns < 4*floor(p/4).
#include "common.cuh"
#include "launch.h"

namespace pbg {

struct PotrfWarpArgs {
  double* a;
  long long stride;
  int lda, n, upper, batch;
  int* info;
  int info_offset;
  int skip_nonzero;
};

__host__ __device__ constexpr int tix(int I, int J) { return I * (I + 1) / 2 + J; }

template <int T>
__global__ void __launch_bounds__(128) potrf_warp_kernel(const __grid_constant__ PotrfWarpArgs P) {
  constexpr int NT = T * (T + 1) / 2;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const long long p = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= P.batch) return;
  if (P.skip_nonzero && P.info[p] != 0) return;
  const int n = P.n;
  double* a = P.a + p * P.stride;
  const long long lda = P.lda;

  double acc[NT][2];
  // ---- load (lower problem; upper = transposed storage), identity padding ----
#pragma unroll
  for (int I = 0; I < T; ++I)
#pragma unroll
    for (int J = 0; J <= I; ++J)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * I + g, c = 8 * J + 2 * t + e;
        double v = (r == c) ? 1.0 : 0.0;
        if (r < n && c < n && (I != J || r >= c))
          v = P.upper ? a[c + r * lda] : a[r + c * lda];
        acc[tix(I, J)][e] = v;
      }

  int fail = 0;
#pragma unroll
  for (int k = 0; k < T; ++k) {
    if (fail) break;
    // ---- 1. diagonal tile ----
    double dinv[8];
    {
      double& d0 = acc[tix(k, k)][0];
      double& d1 = acc[tix(k, k)][1];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (!fail) {
          const double vc = (c & 1) ? d1 : d0;
          const double piv = __shfl_sync(FULL, vc, 4 * c + (c >> 1));
          if (8 * k + c < n && piv <= 0.0) {
            fail = 8 * k + c + 1;
          } else {
            const double s = sqrt(piv);
            const double inv = 1.0 / s;
            dinv[c] = inv;
            if (t == (c >> 1)) {
              double& x = (c & 1) ? d1 : d0;
              if (g == c) x = s;
              else if (g > c) x *= inv;
            }
            const double vs = (c & 1) ? d1 : d0;
            const double xg = __shfl_sync(FULL, vs, 4 * g + (c >> 1));
            const double f0 = __shfl_sync(FULL, vs, 8 * t + (c >> 1));
            const double f1 = __shfl_sync(FULL, vs, 8 * t + 4 + (c >> 1));
            if (2 * t > c && g >= 2 * t) d0 -= xg * f0;
            if (2 * t + 1 > c && g >= 2 * t + 1) d1 -= xg * f1;
          }
        }
      }
    }
    if (fail) break;
    if (k + 1 < T) {
      // ---- 2. panel tiles: X L^T = B ----
      double lc0[8], lc1[8];  // L(c, 2t), L(c, 2t+1)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        lc0[c] = __shfl_sync(FULL, acc[tix(k, k)][0], 4 * c + t);
        lc1[c] = __shfl_sync(FULL, acc[tix(k, k)][1], 4 * c + t);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
#pragma unroll
        for (int I = k + 1; I < T; ++I) {
          double& x0 = acc[tix(I, k)][0];
          double& x1 = acc[tix(I, k)][1];
          double part = (2 * t < c ? x0 * lc0[c] : 0.0);
          part = (2 * t + 1 < c) ? fma(x1, lc1[c], part) : part;
          part += __shfl_xor_sync(FULL, part, 1);
          part += __shfl_xor_sync(FULL, part, 2);
          if (t == (c >> 1)) {
            if (c & 1) x1 = (x1 - part) * dinv[c];
            else x0 = (x0 - part) * dinv[c];
          }
        }
      }
      // ---- 3. trailing update with DMMA: A(I,J) -= L(I,k) L(J,k)^T ----
      double fr[T][2];
#pragma unroll
      for (int I = k + 1; I < T; ++I)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int src = 4 * g + 2 * kk + (t >> 1);
          const double s0 = __shfl_sync(FULL, acc[tix(I, k)][0], src);
          const double s1 = __shfl_sync(FULL, acc[tix(I, k)][1], src);
          fr[I][kk] = (t & 1) ? s1 : s0;
        }
#pragma unroll
      for (int I = k + 1; I < T; ++I)
#pragma unroll
        for (int J = k + 1; J <= I; ++J)
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            dmma(acc[tix(I, J)][0], acc[tix(I, J)][1], -fr[I][kk], fr[J][kk]);
    }
  }

  // ---- write back (failure: only the tiles the reference had stored) ----
  int band_lo = n, band_cols = 0;
  if (fail) {
    band_lo = ((fail - 1) / 8) * 8;
    band_cols = ((fail - 1) / 4) * 4;
  }
#pragma unroll
  for (int I = 0; I < T; ++I)
#pragma unroll
    for (int J = 0; J <= I; ++J)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * I + g, c = 8 * J + 2 * t + e;
        if (r >= n || c >= n || r < c) continue;
        if (r >= band_lo + 8 || (r >= band_lo && c >= band_cols)) continue;
        if (P.upper) a[c + r * lda] = acc[tix(I, J)][e];
        else a[r + c * lda] = acc[tix(I, J)][e];
      }
  if (lane == 0) P.info[p] = fail ? fail + P.info_offset : 0;
}

cudaError_t potrf_warp_launch(double* a, long long stride, int lda, int n, int upper, int* info,
                              int info_offset, int skip_nonzero, int batch, cudaStream_t s) {
  PotrfWarpArgs P{a, stride, lda, n, upper, batch, info, info_offset, skip_nonzero};
  const int T = (n + 7) / 8;
  const int wpb = 4;
  const unsigned grid = (unsigned)((batch + wpb - 1) / wpb);
  switch (T) {
    case 1: potrf_warp_kernel<1><<<grid, 32 * wpb, 0, s>>>(P); break;
    case 2: potrf_warp_kernel<2><<<grid, 32 * wpb, 0, s>>>(P); break;
    case 3: potrf_warp_kernel<3><<<grid, 32 * wpb, 0, s>>>(P); break;
    case 4: potrf_warp_kernel<4><<<grid, 32 * wpb, 0, s>>>(P); break;
    case 5: potrf_warp_kernel<5><<<grid, 32 * wpb, 0, s>>>(P); break;
    case 6: potrf_warp_kernel<6><<<grid, 32 * wpb, 0, s>>>(P); break;
    case 7: potrf_warp_kernel<7><<<grid, 32 * wpb, 0, s>>>(P); break;
    case 8: potrf_warp_kernel<8><<<grid, 32 * wpb, 0, s>>>(P); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace pbg
