// Batched triangular solve for sm_100a: X * op(A) = alpha * B on independent rows.
//
// Replaces trsm_right_core / kernel_trsm_right (level3.hpp:174-214,
// micro_kernel.hpp:522-543) and the panel-major trsm_rltn_nd
// (level3.hpp:484-526).  Left-side solves arrive here as the transposed
// right-side problem ('twin' addressing, level3.hpp:300-303).
//
// One CTA owns a 64-row block of X for one problem, staged in shared memory
// (column stride 68 = 4 mod 16 doubles: conflict-free DMMA fragments).  The
// triangle is consumed 8 columns at a time, right-looking, in dependency
// order (ascending when op(A) is effectively upper, descending when lower):
//   1. the 8 rows of op(A) for the block are staged in shared memory;
//   2. each thread solves its row against the 8x8 diagonal block (unfused
//      update, reciprocal scaling, as edge_trsm_right);
//   3. the remaining columns are updated B -= X_blk op(A)_blk with FP64
//      tensor-core DMMA m8n8k4 on 8x8 tiles.
// Exactly-zero non-unit diagonals are detected before anything is written
// (level3.hpp:292-299) and reported per problem.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace pbg {

constexpr int TR_R = 64;   // rows of X per CTA
constexpr int TR_SX = 68;  // smem column stride of the X block
constexpr int TR_SP = 12;  // smem column stride of the 8-row op(A) panel

struct TrsmArgs {
  TrsmLaunch L;
  int rowblocks;
  int nn8;
};

template <int PM>
__device__ __forceinline__ long long xoff(int twin, int ld, int r, int c) {
  if (PM) return (long long)(r >> 2) * 4 * ld + (long long)c * 4 + (r & 3);
  return twin ? (long long)c + (long long)r * ld : (long long)r + (long long)c * ld;
}
template <int PM>
__device__ __forceinline__ long long aoff(int ld, int i, int j) {
  if (PM) return (long long)(i >> 2) * 4 * ld + (long long)j * 4 + (i & 3);
  return (long long)i + (long long)j * ld;
}

template <int PM>
__global__ void __launch_bounds__(256) trsm_kernel(const __grid_constant__ TrsmArgs T) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int sh_zero;
  const TrsmLaunch& L = T.L;
  const int p = blockIdx.x / T.rowblocks, rb = blockIdx.x - p * T.rowblocks;
  if (L.skip_nonzero && L.info[p] != 0) return;
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
  int nn = L.nn, mm = L.mm;
  int lda = L.lda, ldb = L.ldb, ldd = L.ldd;
  const double *A, *B;
  double* D;
  if (L.nvec) {  // variable batch: square problems at per-problem offsets
    nn = mm = L.nvec[p];
    lda = ldb = ldd = PM ? ((nn + 3) & ~3) : nn;
    A = L.a + L.offs[p];
    B = L.b + L.offs[p];
    D = L.d + L.offs[p];
  } else {
    A = L.a + (long long)p * L.sa;
    B = L.b + (long long)p * L.sb;
    D = L.d + (long long)p * L.sd;
  }
  const int nn8 = (nn + 7) & ~7;
  const int r0 = rb * TR_R, rows = min(TR_R, mm - r0);
  if (rows <= 0) return;
  double* X = sm;                       // TR_SX x nn8
  double* Pn = sm + (size_t)TR_SX * nn8;  // TR_SP x nn8: rows c0..c0+7 of op(A)
  auto opA = [&](int l, int c) -> double {
    return L.trans ? A[aoff<PM>(lda, c, l)] : A[aoff<PM>(lda, l, c)];
  };

  // Zero-diagonal test before any store: smallest exactly-zero index.
  if (tid == 0) sh_zero = 0x7fffffff;
  __syncthreads();
  if (!L.unit)
    for (int i = tid; i < nn; i += nthr)
      if (A[aoff<PM>(lda, i, i)] == 0.0) atomicMin(&sh_zero, i + 1);
  __syncthreads();
  if (sh_zero != 0x7fffffff) {
    if (rb == 0 && tid == 0 && !L.skip_nonzero && L.info) L.info[p] = sh_zero;
    return;
  }

  // Stage alpha*B rows of this block (padding rows/columns zeroed).
  for (int e = tid; e < TR_R * nn8; e += nthr) {
    int c, r;
    if (!PM && L.twin) { r = e / nn8; c = e - r * nn8; } else { c = e / TR_R; r = e - c * TR_R; }
    double v = 0.0;
    if (r < rows && c < nn) v = L.alpha * B[xoff<PM>(L.twin, ldb, r0 + r, c)];
    X[r + c * TR_SX] = v;
  }

  const int eff_lower = L.lower == !L.trans;
  const int nblk = nn8 / 8;
  const int g = lane >> 2, t = lane & 3;
  for (int s = 0; s < nblk; ++s) {
    const int kb = eff_lower ? nblk - 1 - s : s;
    const int c0 = kb * 8, w = min(8, nn - c0);
    // remaining columns after this block: eff upper -> [c0+8, nn8), eff lower -> [0, c0)
    const int ulo = eff_lower ? 0 : c0 + 8, uhi = eff_lower ? c0 : nn8;
    // 1. stage rows c0..c0+7 of op(A) over the block and the remaining columns
    __syncthreads();
    {
      const int clo = eff_lower ? 0 : c0, chi = eff_lower ? c0 + 8 : nn8;
      const int span = chi - clo;
      for (int e = tid; e < 8 * span; e += nthr) {
        int q, c;
        if (L.trans) { c = clo + e % span; q = e / span; } else { q = e % 8; c = clo + e / 8; }
        double v = 0.0;
        if (q < w && c < nn) v = opA(c0 + q, c);
        Pn[q + c * TR_SP] = v;
      }
    }
    __syncthreads();
    // 2. per-row solve against the diagonal block
    if (tid < rows) {
      double x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = X[tid + (c0 + q) * TR_SX];
      if (!eff_lower) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < w) {
#pragma unroll
            for (int l = 0; l < q; ++l) x[q] -= x[l] * Pn[l + (c0 + q) * TR_SP];
            if (!L.unit) x[q] *= 1.0 / Pn[q + (c0 + q) * TR_SP];
          }
        }
      } else {
#pragma unroll
        for (int qq = 7; qq >= 0; --qq) {
          if (qq < w) {
#pragma unroll
            for (int l = qq + 1; l < 8; ++l)
              if (l < w) x[qq] -= x[l] * Pn[l + (c0 + qq) * TR_SP];
            if (!L.unit) x[qq] *= 1.0 / Pn[qq + (c0 + qq) * TR_SP];
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < w) X[tid + (c0 + q) * TR_SX] = x[q];
    }
    __syncthreads();
    // 3. trailing update of the unsolved columns: X[:, u] -= X[:, blk] * op(A)[blk, u]
    const int ucols = (uhi - ulo) / 8;
    const int ntiles = (TR_R / 8) * ucols;
    for (int idx = warp; idx < ntiles; idx += (nthr >> 5)) {
      const int ti = idx % (TR_R / 8), tj = idx / (TR_R / 8);
      const int rr = ti * 8, cc = ulo + tj * 8;
      if (rr >= rows) continue;
      double d0 = 0.0, d1 = 0.0;
      dmma(d0, d1, X[(rr + g) + (c0 + t) * TR_SX], Pn[t + (cc + g) * TR_SP]);
      dmma(d0, d1, X[(rr + g) + (c0 + 4 + t) * TR_SX], Pn[(4 + t) + (cc + g) * TR_SP]);
      X[(rr + g) + (cc + 2 * t) * TR_SX] -= d0;
      X[(rr + g) + (cc + 2 * t + 1) * TR_SX] -= d1;
    }
  }
  __syncthreads();
  if (!PM && L.twin) {  // storage columns are rows of X: coalesce over c
    for (int e = tid; e < rows * nn; e += nthr) {
      int r = e / nn, c = e - r * nn;
      D[xoff<0>(1, ldd, r0 + r, c)] = X[r + c * TR_SX];
    }
  } else {
    for (int e = tid; e < rows * nn; e += nthr) {
      int c = e / rows, r = e - c * rows;
      D[xoff<PM>(0, ldd, r0 + r, c)] = X[r + c * TR_SX];
    }
  }
  if (rb == 0 && tid == 0 && !L.skip_nonzero && L.info) L.info[p] = 0;
}

// trsm_rltn_nd with alpha == 0 (level3.hpp:493-504): the exact-zero diagonal
// test still runs first and reports before any store; otherwise D's m x n
// entries become +0 (scale_tiles_nd with beta 0: B is never read, pad lanes
// untouched).  One CTA per problem, panel-major operands.
__global__ void __launch_bounds__(256) trsm_nd_zero_kernel(const __grid_constant__ TrsmLaunch L) {
  __shared__ int sh_zero;
  const int p = blockIdx.x, tid = threadIdx.x;
  const double* A = L.a + (long long)p * L.sa;
  double* D = L.d + (long long)p * L.sd;
  if (tid == 0) sh_zero = 0x7fffffff;
  __syncthreads();
  for (int i = tid; i < L.nn; i += blockDim.x)
    if (A[aoff<1>(L.lda, i, i)] == 0.0) atomicMin(&sh_zero, i + 1);
  __syncthreads();
  const int z = sh_zero == 0x7fffffff ? 0 : sh_zero;
  if (tid == 0 && L.info) L.info[p] = z;
  if (z) return;
  for (int e = tid; e < L.mm * L.nn; e += blockDim.x) {
    const int c = e / L.mm, r = e - c * L.mm;
    D[aoff<1>(L.ldd, r, c)] = 0.0;
  }
}

cudaError_t trsm_nd_zero_launch(const TrsmLaunch& L, cudaStream_t s) {
  if (L.batch <= 0 || L.mm <= 0 || L.nn <= 0) return cudaSuccess;
  trsm_nd_zero_kernel<<<(unsigned)L.batch, 256, 0, s>>>(L);
  return cudaGetLastError();
}

cudaError_t trsm_launch(const TrsmLaunch& L, cudaStream_t s) {
  if (L.batch <= 0 || L.mm <= 0 || L.nn <= 0) return cudaSuccess;
  static const bool rlt = [] {  // PBGPU_TRSM_RLT=0 keeps this kernel for every flag set (A/B)
    const char* e = getenv("PBGPU_TRSM_RLT");
    return !(e && e[0] == '0');
  }();
  if (rlt && trsm_rlt_ok(L)) return trsm_rlt_launch(L, s);
  TrsmArgs T;
  T.L = L;
  T.rowblocks = (L.mm + TR_R - 1) / TR_R;
  T.nn8 = (L.nn + 7) & ~7;
  size_t smem = (size_t)(TR_SX + TR_SP) * T.nn8 * sizeof(double);
  if (smem > 220 * 1024) return cudaErrorInvalidValue;  // nn <= 340
  {
    cudaError_t e = smem_attr((const void*)(L.pm ? trsm_kernel<1> : trsm_kernel<0>), 220 * 1024);
    if (e != cudaSuccess) return e;
  }
  long long grid = (long long)L.batch * T.rowblocks;
  if (L.pm)
    trsm_kernel<1><<<(unsigned)grid, 256, smem, s>>>(T);
  else
    trsm_kernel<0><<<(unsigned)grid, 256, smem, s>>>(T);
  return cudaGetLastError();
}

}  // namespace pbg
