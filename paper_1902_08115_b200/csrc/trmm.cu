// Batched triangular multiply for sm_100a: D = alpha * X * op(A), A triangular.
//
// Replaces trmm_right_core / kernel_trmm_right / edge_trmm_right
// (level3.hpp:132-170, micro_kernel.hpp:357-378, 566-586) behind dtrmm
// (blas.hpp:166-176, all 16 flag sets; Left runs as the transposed right-side
// problem through 'twin' addressing, level3.hpp:263-265) and the panel-major
// trmm_rlnn_nd (level3.hpp:446-479, micro_kernel.hpp:588-601) that the
// Riccati recursion calls every stage (riccati.hpp:319).
//
// One CTA owns an R-row block of X (R = 64 down to 8, the largest whose
// staged rows fit in shared memory) of one problem.  The block is staged
// once (column stride R + 4 = 4 mod 16 doubles: conflict-free DMMA A
// fragments), so D may alias B: the CTA's own rows are read completely before
// the first store.  Then, per 8-column tile J of D, the tile's columns of
// op(A) restricted to the triangle are staged (zeros outside it, 1 on a unit
// diagonal, which is never read — micro_kernel.hpp:365-370), and every warp
// accumulates one 8x8 output tile over the triangle's k range on FP64
// tensor cores (DMMA m8n8k4, two independent accumulator chains) and stores
// alpha * acc.
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace pbg {

struct TrmmArgs {
  TrsmLaunch L;
  int rowblocks;
  int nn8;
};

template <int PM>
__device__ __forceinline__ long long tm_xoff(int twin, int ld, int r, int c) {
  if (PM) return (long long)(r >> 2) * 4 * ld + (long long)c * 4 + (r & 3);
  return twin ? (long long)c + (long long)r * ld : (long long)r + (long long)c * ld;
}
template <int PM>
__device__ __forceinline__ long long tm_aoff(int ld, int i, int j) {
  if (PM) return (long long)(i >> 2) * 4 * ld + (long long)j * 4 + (i & 3);
  return (long long)i + (long long)j * ld;
}

template <int PM, int R>
__global__ void __launch_bounds__(256) trmm_kernel(const __grid_constant__ TrmmArgs T) {
  extern __shared__ __align__(16) double sm[];
  constexpr int SX = R + 4;
  const TrsmLaunch& L = T.L;
  const int p = blockIdx.x / T.rowblocks, rb = blockIdx.x - p * T.rowblocks;
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
  const int nn = L.nn, mm = L.mm, nn8 = T.nn8, SP = nn8 + 4;
  const double* A = L.a + (long long)p * L.sa;
  const double* B = L.b + (long long)p * L.sb;
  double* D = L.d + (long long)p * L.sd;
  const int r0 = rb * R, rows = min(R, mm - r0);
  if (rows <= 0) return;
  double* X = sm;                        // SX x nn8
  double* Pn = sm + (size_t)SX * nn8;    // SP x 8: columns J*8.. of op(A) over the k range

  // Stage the block's rows of B (padding rows / columns zeroed).
  for (int e = tid; e < R * nn8; e += nthr) {
    int c, r;
    if (!PM && L.twin) { r = e / nn8; c = e - r * nn8; } else { c = e / R; r = e - c * R; }
    double v = 0.0;
    if (r < rows && c < nn) v = B[tm_xoff<PM>(L.twin, L.ldb, r0 + r, c)];
    X[r + c * SX] = v;
  }

  const int eff_lower = L.lower == !L.trans;
  const int g = lane >> 2, t = lane & 3;
  for (int J = 0; J * 8 < nn; ++J) {
    const int j0 = J * 8;
    const int kl = eff_lower ? j0 : 0, kh = eff_lower ? nn8 : j0 + 8;
    const int span = kh - kl;
    __syncthreads();  // X staged / previous tile's reads of Pn done
    for (int e = tid; e < 8 * span; e += nthr) {
      int q, l;
      if (L.trans) { q = e & 7; l = kl + (e >> 3); } else { l = kl + e % span; q = e / span; }
      const int j = j0 + q;
      double v = 0.0;
      if (j < nn && l < nn) {
        if (l == j) v = L.unit ? 1.0 : (L.trans ? A[tm_aoff<PM>(L.lda, j, l)] : A[tm_aoff<PM>(L.lda, l, j)]);
        else if (eff_lower ? l > j : l < j) v = L.trans ? A[tm_aoff<PM>(L.lda, j, l)] : A[tm_aoff<PM>(L.lda, l, j)];
      }
      Pn[l + q * SP] = v;
    }
    __syncthreads();
    for (int ti = warp; ti < R / 8; ti += (nthr >> 5)) {
      const int rr = ti * 8;
      if (rr >= rows) break;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
      int k0 = kl;
      for (; k0 + 8 <= kh; k0 += 8) {
        dmma(d0, d1, X[(rr + g) + (k0 + t) * SX], Pn[(k0 + t) + g * SP]);
        dmma(e0, e1, X[(rr + g) + (k0 + 4 + t) * SX], Pn[(k0 + 4 + t) + g * SP]);
      }
      if (k0 < kh) dmma(d0, d1, X[(rr + g) + (k0 + t) * SX], Pn[(k0 + t) + g * SP]);
      const int r = r0 + rr + g;
      if (rr + g < rows) {
        const int c = j0 + 2 * t;
        if (c < nn) D[tm_xoff<PM>(L.twin, L.ldd, r, c)] = (d0 + e0) * L.alpha;
        if (c + 1 < nn) D[tm_xoff<PM>(L.twin, L.ldd, r, c + 1)] = (d1 + e1) * L.alpha;
      }
    }
  }
}

template <int PM, int R>
static cudaError_t trmm_t(const TrmmArgs& T, size_t smem, cudaStream_t s) {
  cudaError_t e = smem_attr((const void*)trmm_kernel<PM, R>, (int)smem);
  if (e != cudaSuccess) return e;
  const long long grid = (long long)T.L.batch * T.rowblocks;
  trmm_kernel<PM, R><<<(unsigned)grid, 256, smem, s>>>(T);
  return cudaGetLastError();
}

cudaError_t trmm_launch(const TrsmLaunch& L, cudaStream_t s) {
  if (L.batch <= 0 || L.mm <= 0 || L.nn <= 0) return cudaSuccess;
  TrmmArgs T;
  T.L = L;
  T.nn8 = (L.nn + 7) & ~7;
  const size_t cap = 220 * 1024;
  auto smem_for = [&](int R) { return ((size_t)(R + 4) * T.nn8 + (size_t)(T.nn8 + 4) * 8) * sizeof(double); };
  int R = 64;
  while (R > 8 && smem_for(R) > cap) R /= 2;
  if (smem_for(R) > cap) return cudaErrorInvalidValue;  // nn > ~2000
  T.rowblocks = (L.mm + R - 1) / R;
  const size_t smem = smem_for(R);
#define PB_TRMM(RV) \
  case RV: return L.pm ? trmm_t<1, RV>(T, smem, s) : trmm_t<0, RV>(T, smem, s);
  switch (R) {
    PB_TRMM(64) PB_TRMM(32) PB_TRMM(16) PB_TRMM(8)
  }
#undef PB_TRMM
  return cudaErrorInvalidValue;
}

}  // namespace pbg
