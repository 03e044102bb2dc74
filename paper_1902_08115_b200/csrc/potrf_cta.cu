// Pipelined left-looking batched Cholesky, one CTA per problem, n <= 160 (sm_100a).
//
// The reference's potrf_core (factor.hpp:45-99) is left-looking over column
// blocks; this kernel keeps that order and overlaps its two phases across
// warps.  The lower triangle lives in shared memory as column panels of 8
// columns (panel k holds rows 8k.., column-major, column stride 8(T-k)+4 —
// conflict-free for both row-per-lane accesses and DMMA fragments).
//   * warp 0 (the panel warp) factors panel k column by column, every lane
//     owning up to R rows: pivot broadcast by shuffle, reciprocal square
//     root, scaling by the reciprocal, rank-1 updates with the diagonal column
//     broadcast through shared memory (failure test `piv <= 0.0`,
//     micro_kernel.hpp:314);
//   * meanwhile the update warps accumulate column block k+1's left-looking
//     update A(k+1:, k+1) -= L(k+1:, 0:k) L(k+1, 0:k)^T on FP64 tensor cores
//     (DMMA m8n8k4, accumulators in registers) from the panels already
//     factored, then — once panel k is published — add its contribution and
//     store the block back for the panel warp.
// Two named barriers per step hand panels over; the factorization latency of
// one block hides behind the tensor-core update of the next.  The factor is
// written to global memory once, at the end, so a failure at column p stores
// exactly the reference's set (rows < 8*floor(p/8) and, in that band, columns
// < 4*floor(p/4); test_factor.cpp:251-277).  PM = 1 addresses panel-major
// storage (ps = 4); zero_fill writes the LowerZero band zeros of
// syrk_potrf_nd (micro_kernel.hpp:657-673).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "launch.h"

namespace pbg {

constexpr int kCtaMaxT = 20;  // n <= 160

struct PotrfCtaArgs {
  double* a;
  long long stride;
  const long long* offs;  // optional per-problem element offsets (variable batches)
  const int* nvec;        // optional per-problem order (variable batches)
  int lda, n, upper, batch, zero_fill;
  int* info;
  int info_offset;
  int skip_nonzero;
  // optional prologue S = C + A B^T before factoring (syrk_potrf_nd,
  // micro_kernel.hpp:640-673): A, B are n x k in the same storage kind as C
  // (ld = lda_ab: cm leading dimension or pm panel width), problem p at
  // offs_ab[p] (variable batches) or p * stride_ab.
  const double* pa;
  const double* pb;
  long long stride_ab;
  const long long* offs_ab;
  int k_ab, lda_ab;
  // optional separate source (the C of syrk_potrf_nd when it does not alias D)
  const double* src;
  long long src_stride;
  int src_ld;
  int syrk_only;  // write S = C + A B^T (lower) back and skip the factorization
  // optional per-panel TMA tensor maps (packed column-major lower problems):
  // map k covers rows 8k .. 8k+8(T-k)+3 of columns 8k..8k+7, i.e. exactly the
  // shared-memory panel k (column stride 8(T-k)+4, the 4 rows past n are
  // zero-filled out of bounds), so staging and the write back are one tensor
  // copy per panel
  int tma;
  CUtensorMap tm[kCtaMaxT];
};

#ifndef PB_REDUNDANT_FROM  // panels factored with the redundant diagonal block from T = 9 (n = 72) on
#define PB_REDUNDANT_FROM 9
#endif
#ifndef PB_CTA_PAD
#define PB_CTA_PAD 4
#endif
__host__ __device__ constexpr int cta_pstride(int T, int k) { return 8 * (T - k) + PB_CTA_PAD; }
__host__ __device__ constexpr int cta_pbase(int T, int k) {
  return 64 * (k * T - k * (k - 1) / 2) + 8 * PB_CTA_PAD * k;
}

template <int PM>
__device__ __forceinline__ long long cta_eoff(int upper, long long ld, int r, int c) {
  if (PM) return (long long)(r >> 2) * 4 * ld + (long long)c * 4 + (r & 3);
  return upper ? (long long)c + r * ld : (long long)r + c * ld;
}

// PB_TRACE (tools/potrf_trace.cu only): per-CTA clock64 stamps of the phases
#ifdef PB_TRACE
__device__ long long pb_trace[256][64];
#define PB_STAMP(slot) \
  if ((blockIdx.x & 31) == 0 && (blockIdx.x >> 5) < 256 && (slot) < 64) pb_trace[blockIdx.x >> 5][slot] = clock64();
#else
#define PB_STAMP(slot)
#endif

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// Panel warp: factor the (rows x 8) panel in place; lane owns rows lane + 32 q.
// Every lane factors the 8x8 diagonal block D redundantly in registers, so a
// column step is rsqrt -> scale -> update with no shuffle or shared-memory
// round trip on the dependency chain; the lane's own rows follow the same
// recurrence (the rows of D itself come out bitwise equal to D's entries,
// the strict upper part of the block is scratch).
// Slow twin for the rare panels whose pivots are denormal, +inf or NaN (where
// the branch-free rsqrt_nb is not exact): the reference's sqrt and reciprocal,
// rows straight in shared memory, early exit at a failed column.
__device__ __noinline__ int cta_factor_panel_exact(uint32_t pan, int RS, int rows, int lane, int gcol0, int n) {
  int f = 0;
  for (int c = 0; c < 8; ++c) {
    const double piv = lds64(pan + 8u * (c * RS + c));
    __syncwarp();
    if (gcol0 + c < n && piv <= 0.0) {
      f = c + 1;
      break;
    }
    // the reference's s = sqrt(piv), inv = 1 / s (micro_kernel.hpp:315-318): an
    // Inf pivot gives L_cc = Inf and zeros below, not Inf * 0
    const double sq = sqrt(piv), inv = 1.0 / sq;
    for (int r = c + lane; r < rows; r += 32) {
      const uint32_t a = pan + 8u * (c * RS + r);
      sts64(a, r == c ? sq : lds64(a) * inv);
    }
    __syncwarp();
    for (int c2 = c + 1; c2 < 8; ++c2) {
      const double l = lds64(pan + 8u * (c * RS + c2));
      for (int r = c2 + lane; r < rows; r += 32) {
        const uint32_t a = pan + 8u * (c2 * RS + r);
        sts64(a, lds64(a) - lds64(pan + 8u * (c * RS + r)) * l);
      }
    }
    __syncwarp();
  }
  return f;
}

template <int R>
__device__ __forceinline__ int cta_factor_panel(uint32_t pan, int RS, int rows, int lane, int gcol0, int n) {
  double x[R][8];
  double D[8][8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int i = c & ~1; i < 8; i += 2) {
      double2 v;
      asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(pan + 8u * (c * RS + i)));
      D[i][c] = v.x;
      D[i + 1][c] = v.y;
    }
  // rows past the panel read scratch (the allocation has 8T+32 doubles of
  // slack) and are never stored: unconditional loads, predicated stores
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[q][c] = lds64(pan + 8u * (c * RS + lane + 32 * q));
  // no failure test inside the loop: a pivot <= 0 (NaN after rsqrt_nb), a
  // denormal or +inf pivot (rsqrt_nb inexact) and a NaN input all leave a
  // non-finite diagonal entry, which the sum below catches; those rare
  // panels are redone exactly (failure column, reference semantics)
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double piv = D[c][c];
    const double inv = rsqrt_nb(piv);
    D[c][c] = piv * inv;
#pragma unroll
    for (int i = c + 1; i < 8; ++i) D[i][c] *= inv;
#pragma unroll
    for (int q = 0; q < R; ++q) x[q][c] *= inv;
#pragma unroll
    for (int c2 = c + 1; c2 < 8; ++c2) {
#pragma unroll
      for (int i = c2; i < 8; ++i) D[i][c2] -= D[i][c] * D[c2][c];
#pragma unroll
      for (int q = 0; q < R; ++q) x[q][c2] -= x[q][c] * D[c2][c];
    }
  }
  double dsum = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) dsum += D[c][c];
  if (!(dsum <= 1.7976931348623157e308))  // warp-uniform (D is redundant)
    return cta_factor_panel_exact(pan, RS, rows, lane, gcol0, n);
  // the strict upper part of the diagonal block keeps its staged (original) values
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      sts64_if(pan + 8u * (c * RS + lane + 32 * q), x[q][c], lane + 32 * q < rows && (q > 0 || lane >= c));
  return 0;
}

// Broadcast variant: the diagonal block's rows are lanes 0..7 (slot 0); per
// column they publish their entry of column c to a shared double buffer and
// every lane reads the pivot and the multipliers back as broadcast loads, so
// the 8x8 block is factored once instead of redundantly in every lane.
template <int R>
__device__ __forceinline__ int cta_factor_panel_bc(uint32_t pan, int RS, int rows, int lane, int gcol0, int n,
                                                   uint32_t colbuf) {
  double x[R][8];
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[q][c] = lds64(pan + 8u * (c * RS + lane + 32 * q));
  double dsum = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t cb = colbuf + (c & 1) * 64;
    if (lane >= c && lane < 8) sts64(cb + 8u * lane, x[0][c]);
    __syncwarp();
    double col[8];
#pragma unroll
    for (int c2 = c & ~1; c2 < 8; c2 += 2) lds128(cb + 8u * c2, col[c2], col[c2 + 1]);
    const double piv = col[c];
    const double inv = rsqrt_nb(piv);
    dsum += piv * inv;  // non-finite for a failed, denormal, +inf or NaN pivot
#pragma unroll
    for (int q = 0; q < R; ++q) {
      x[q][c] *= inv;
      const double tq = x[q][c] * inv;
#pragma unroll
      for (int c2 = c + 1; c2 < 8; ++c2) x[q][c2] = fma(-tq, col[c2], x[q][c2]);
    }
  }
  if (!(dsum <= 1.7976931348623157e308))  // warp-uniform
    return cta_factor_panel_exact(pan, RS, rows, lane, gcol0, n);
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      sts64_if(pan + 8u * (c * RS + lane + 32 * q), x[q][c], lane + 32 * q < rows && (q > 0 || lane >= c));
  return 0;
}

// Update warp: column block k1's tiles I = uw + NU*s (s < NS) accumulate
// -sum_l L(I, l) L(k1, l)^T over l < k1 (panel k1-1 after its publication),
// then go back to shared memory.  Returns true when the panel warp reported
// a failure (the block is then left untouched).
template <int T, int NU, int NS>
__device__ __forceinline__ bool cta_update_block(uint32_t sbase, int k1, int uw, int g, int t, const int* sh_fail,
                                                 uint64_t* landed) {
  constexpr int NTH = 32 * (NU + 1);
  if (landed) mbar_wait(landed, 0);  // column block k1 staged (streamed staging)
  const int RS = cta_pstride(T, k1);
  const uint32_t pan = sbase + 8u * cta_pbase(T, k1);
  double acc[NS > 0 ? NS : 1][2];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int I = uw + NU * s;
    acc[s][0] = lds64(pan + 8u * ((2 * t) * RS + 8 * I + g));
    acc[s][1] = lds64(pan + 8u * ((2 * t + 1) * RS + 8 * I + g));
  }
  uint32_t pl = sbase + 8u * (8 * k1 + g);  // row 8*k1 + g of panel 0
  constexpr int NSX = NS > 0 ? NS : 1;
  // fragments of panel l: b = -L(8k1+g, 4kk+t), a[s] = L(8k1+8I_s+g, 4kk+t)
  auto load = [&](uint32_t plv, int RL, double (&b)[2], double (&a)[2][NSX]) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t col = plv + 8u * ((4 * kk + t) * RL);
      b[kk] = -lds64(col);
#pragma unroll
      for (int s = 0; s < NS; ++s) a[kk][s] = lds64(col + 8u * (8 * (uw + NU * s)));
    }
  };
  auto mma = [&](double (&c)[NSX][2], const double (&b)[2], const double (&a)[2][NSX]) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
#pragma unroll
      for (int s = 0; s < NS; ++s) dmma(c[s][0], c[s][1], a[kk][s], b[kk]);
  };
  int l = 0;
  if constexpr (NS <= 4) {
    // few tiles: two panels per trip into two accumulator sets, all fragment
    // loads first, so neither shared-memory latency nor the DMMA chain stalls
    double acc2[NSX][2];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc2[s][0] = acc2[s][1] = 0.0;
    for (; l + 2 <= k1 - 1; l += 2) {
      const int RL0 = cta_pstride(T, l), RL1 = RL0 - 8;
      const uint32_t pl1 = pl + 8u * (8 * RL0 - 8);
      double b0[2], a0[2][NSX], b1[2], a1[2][NSX];
      load(pl, RL0, b0, a0);
      load(pl1, RL1, b1, a1);
      mma(acc, b0, a0);
      mma(acc2, b1, a1);
      pl = pl1 + 8u * (8 * RL1 - 8);
    }
    if (l < k1 - 1) {
      const int RL = cta_pstride(T, l);
      double b0[2], a0[2][NSX];
      load(pl, RL, b0, a0);
      mma(acc2, b0, a0);
      pl += 8u * (8 * RL - 8);
      ++l;
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      acc[s][0] += acc2[s][0];
      acc[s][1] += acc2[s][1];
    }
  } else {
    for (; l < k1 - 1; ++l) {
      const int RL = cta_pstride(T, l);
      double b0[2], a0[2][NSX];
      load(pl, RL, b0, a0);
      mma(acc, b0, a0);
      pl += 8u * (8 * RL - 8);
    }
  }
  if (uw == 0 && (threadIdx.x & 31) == 0) { PB_STAMP(40 + k1) }
  named_sync(1, NTH);  // wait for panel k1-1
  if (*(volatile const int*)sh_fail) return true;
  {
    double b0[2], a0[2][NSX];
    load(pl, cta_pstride(T, l), b0, a0);
    mma(acc, b0, a0);
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int I = uw + NU * s;
    // tile 0 is the diagonal block: its strict upper part is never written
    sts64_if(pan + 8u * ((2 * t) * RS + 8 * I + g), acc[s][0], I > 0 || g >= 2 * t);
    sts64_if(pan + 8u * ((2 * t + 1) * RS + 8 * I + g), acc[s][1], I > 0 || g >= 2 * t + 1);
  }
  return false;
}

template <int T, int NU, int PM>
__global__ void __launch_bounds__(32 * (NU + 1)) potrf_cta_kernel(const __grid_constant__ PotrfCtaArgs P) {
  constexpr int NTH = 32 * (NU + 1);
  constexpr int R = (8 * T + 31) / 32;           // rows per lane in the panel warp
  constexpr int SLOTS = (T - 1 + NU - 1) / NU;   // tiles per update warp (blocks k1 >= 1 have <= T-1)
  static_assert(SLOTS <= 11, "cta_update_block dispatch covers at most 11 tiles");
  extern __shared__ __align__(1024) double sm[];
  __shared__ int sh_fail, sh_rot;
  __shared__ __align__(16) double sh_col[2][8];  // panel warp's column broadcast
  __shared__ __align__(8) uint64_t sh_bar[T];  // one per column panel (streamed staging)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const long long p = blockIdx.x;
  if (tid == 0) { PB_STAMP(0) }
  if (P.skip_nonzero && P.info[p] != 0) return;
  const int n = P.nvec ? P.nvec[p] : P.n;
  if (n <= 0) {
    if (tid == 0) P.info[p] = 0;
    return;
  }
  double* a = P.a + (P.offs ? P.offs[p] : p * P.stride);
  const long long lda = P.nvec ? (PM ? ((n + 3) & ~3) : n) : P.lda;
  const int TT = (n + 7) >> 3;
  const uint32_t sbase = smem_u32(sm);

  // ---- stage the lower triangle (panel k: rows 8k.. of columns 8k..8k+7) ----
  const double* sa = P.src ? P.src + (P.offs ? P.offs[p] : p * P.src_stride) : a;
  const long long sld = P.src ? (P.nvec ? lda : P.src_ld) : lda;
  const bool bulk = !PM && !P.upper && (sld % 2 == 0) && ((reinterpret_cast<uintptr_t>(sa) & 15) == 0) &&
                    (n % 2 == 0);
  // streamed: every column panel has its own mbarrier and the factorization
  // starts as soon as panel 0 has landed (the rest arrives underneath it).
  // One TMA bulk copy per column (rows 8k..n-1 of column col, k = col/8);
  // issuing from many threads at once beats one issuing lane.
  const bool streamed = bulk && !(n & 7) && !P.pa;
  if (P.tma) {
    // one tensor copy per column panel, each on its own mbarrier
    if (tid == 0) {
      for (int k = 0; k < TT; ++k) mbar_init(&sh_bar[k], 1);
      fence_mbar_init();
      for (int k = 0; k < TT; ++k) {
        mbar_arrive_expect_tx(&sh_bar[k], 64u * (uint32_t)cta_pstride(T, k));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(sbase + 8u * cta_pbase(T, k)),
            "l"(reinterpret_cast<uint64_t>(&P.tm[k])), "r"(8 * k), "r"(8 * k), "r"((int)p),
            "r"(smem_u32(&sh_bar[k]))
            : "memory");
      }
    }
    __syncthreads();
  } else if (streamed) {
    if (tid == 0) {
      for (int k = 0; k < TT; ++k) mbar_init(&sh_bar[k], 1);
      fence_mbar_init();
      for (int k = 0; k < TT; ++k) mbar_arrive_expect_tx(&sh_bar[k], 64u * (uint32_t)(n - 8 * k));
    }
    __syncthreads();
    for (int col = tid; col < n; col += NTH) {
      const int k = col >> 3, c = col & 7, r0 = 8 * k;
      bulk_g2s(sm + cta_pbase(T, k) + c * cta_pstride(T, k), sa + r0 + (long long)col * sld,
               8u * (uint32_t)(n - r0), &sh_bar[k]);
    }
  } else if (bulk) {
    // one TMA bulk copy per column (rows 8k..n-1 of column col, k = col/8)
    if (tid == 0) {
      mbar_init(&sh_bar[0], 1);
      fence_mbar_init();
      uint32_t bytes = 0;
      for (int k = 0; k < TT; ++k) bytes += 8u * (uint32_t)min(8, n - 8 * k) * (uint32_t)(n - 8 * k);
      mbar_arrive_expect_tx(&sh_bar[0], bytes);
    }
    __syncthreads();
    for (int col = tid; col < n; col += NTH) {
      const int k = col >> 3, c = col & 7, r0 = 8 * k;
      bulk_g2s(sm + cta_pbase(T, k) + c * cta_pstride(T, k), sa + r0 + (long long)col * sld,
               8u * (uint32_t)(n - r0), &sh_bar[0]);
    }
    mbar_wait(&sh_bar[0], 0);
  
  } else {
    // 16-byte pairs of rows (2q, 2q + 1): contiguous in column-major storage with an even
    // leading dimension, and always in panel-major storage (rows 4j .. 4j + 3 of a column)
    const bool pairs = !P.upper && (PM || sld % 2 == 0) && ((reinterpret_cast<uintptr_t>(sa) & 15) == 0);
    for (int k = 0; k < TT; ++k) {
      double* pan = sm + cta_pbase(T, k);
      const int RS = cta_pstride(T, k), r0 = 8 * k, nr = min(n, 8 * TT) - r0;
      if (pairs) {
        const int np = (nr + 1) >> 1, tot = 8 * np;
        const double* src = sa + r0 + (long long)r0 * sld;
        for (int e = tid; e < tot; e += NTH) {
          const int c = e / np, q = e - c * np;
          if (r0 + c >= n) continue;
          const double* s2 = PM ? sa + cta_eoff<PM>(0, sld, r0 + 2 * q, r0 + c) : src + c * sld + 2 * q;
          if (2 * q + 1 < nr) cp_async16(&pan[c * RS + 2 * q], s2);
          else cp_async8(&pan[c * RS + 2 * q], s2, true);
        }
      } else {
        const int tot = 8 * nr;
        for (int e = tid; e < tot; e += NTH) {
          const int c = e / nr, r = e - c * nr, row = r0 + r, col = r0 + c;
          const bool v = col < n && row >= col;
          cp_async8(&pan[c * RS + r], v ? sa + cta_eoff<PM>(P.upper, sld, row, col) : sa, v);
        }
      }
    }
  }
  if (!streamed && !P.tma) cp_async_wait_all();
  __syncthreads();
  if (n & 7) {  // identity padding for rows/columns past n
    for (int k = 0; k < TT; ++k) {
      double* pan = sm + cta_pbase(T, k);
      const int RS = cta_pstride(T, k), rows = 8 * (TT - k);
      for (int e = tid; e < 8 * rows; e += NTH) {
        const int c = e / rows, r = e - c * rows, row = 8 * k + r, col = 8 * k + c;
        if (row >= n || col >= n) pan[c * RS + r] = (row == col) ? 1.0 : 0.0;
      }
    }
  }
  if (P.pa && P.k_ab > 0) {
    // ---- prologue: lower tiles S(I,J) = C(I,J) + A(I,:) B(J,:)^T on the tensor cores ----
    __syncthreads();
    const long long oab = P.offs_ab ? P.offs_ab[p] : p * P.stride_ab;
    const double* A = P.pa + oab;
    const double* B = P.pb + oab;
    const long long lab = P.nvec ? (PM ? ((n + 3) & ~3) : n) : P.lda_ab;
    const int kab = P.nvec ? n : P.k_ab;
    const int ntile = TT * (TT + 1) / 2;
    for (int idx = warp; idx < ntile; idx += NU + 1) {
      int I = (int)((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
      while ((I + 1) * (I + 2) / 2 <= idx) ++I;
      while (I * (I + 1) / 2 > idx) --I;
      const int J = idx - I * (I + 1) / 2;
      const uint32_t pj = sbase + 8u * cta_pbase(T, J);
      const int RJ = cta_pstride(T, J), rr = 8 * (I - J) + g;
      double d0 = lds64(pj + 8u * ((2 * t) * RJ + rr));
      double d1 = lds64(pj + 8u * ((2 * t + 1) * RJ + rr));
      const int ia = 8 * I + g, jb = 8 * J + g;
      for (int l0 = 0; l0 < kab; l0 += 4) {
        const int l = l0 + t;
        const bool ok = l < kab;
        const double av = (ok && ia < n) ? A[cta_eoff<PM>(0, lab, ia, l)] : 0.0;
        const double bv = (ok && jb < n) ? B[cta_eoff<PM>(0, lab, jb, l)] : 0.0;
        dmma(d0, d1, av, bv);
      }
      sts64(pj + 8u * ((2 * t) * RJ + rr), d0);
      sts64(pj + 8u * ((2 * t + 1) * RJ + rr), d1);
    }
  }
  // Role rotation: the scheduler partition (SMSP) of a warp is its hardware
  // slot mod 4, and consecutive CTAs get consecutive slots, so a fixed
  // "warp 0 = panel warp" piles every panel warp of an SM onto the same
  // partitions.  Warp 0 reads its slot and rotates the roles so the panel
  // warps of neighbouring CTAs land on different partitions.
  if (tid == 0) {
    sh_fail = 0;
    uint32_t wid;
    asm volatile("mov.u32 %0, %%warpid;\n" : "=r"(wid));
    sh_rot = (int)((wid >> 2) % (NU + 1));
  }
  __syncthreads();
  const int lw = (warp + NU + 1 - sh_rot) % (NU + 1);  // logical role: 0 = panel warp

  int fail = 0;
  if (P.syrk_only) {
    // no factorization: fall through to the write back of the lower triangle
  } else if (lw == 0) {
    // ------------------------------------------------------------ panel warp
    for (int k = 0; k < TT; ++k) {
      if (k > 0) named_sync(2, NTH);  // block k updated and stored
      if (lane == 0) { PB_STAMP(4 + 2 * k) }
      const int RS = cta_pstride(T, k), rows = 8 * (TT - k);
      if (streamed || P.tma) mbar_wait(&sh_bar[k], 0);
      // from n = 72 on the diagonal block is factored redundantly in every lane
      // (measured: n = 128 0.497 -> 0.471 ms, 256 -1.5 %; no change below); below
      // that, rows per lane follow the panel's height (fewer predicated-off rows)
      const uint32_t pk = sbase + 8u * cta_pbase(T, k), cbuf = smem_u32(&sh_col[0][0]);
      int f;
      if constexpr (T >= PB_REDUNDANT_FROM) {
        f = cta_factor_panel<R>(pk, RS, rows, lane, 8 * k, n);  // (rows-following measured slower here)
      } else if constexpr (R > 1) {
        if (rows <= 32) f = cta_factor_panel_bc<1>(pk, RS, rows, lane, 8 * k, n, cbuf);
        else if (R > 2 && rows <= 64) f = cta_factor_panel_bc<(R > 2 ? 2 : R)>(pk, RS, rows, lane, 8 * k, n, cbuf);
        else f = cta_factor_panel_bc<R>(pk, RS, rows, lane, 8 * k, n, cbuf);
      } else {
        f = cta_factor_panel_bc<R>(pk, RS, rows, lane, 8 * k, n, cbuf);
      }
      if (f && lane == 0) sh_fail = 8 * k + f;
      if (lane == 0) { PB_STAMP(5 + 2 * k) }
      named_sync(1, NTH);  // panel k published (or the failure flag)
      if (f) break;
    }
  } else {
    // ------------------------------------------------------------ update warps
    const int uw = lw - 1;
    for (int k1 = 1; k1 < TT; ++k1) {  // block to update; panel k1-1 is being factored
      const int ta = TT - k1;
      const int ns = uw < ta ? (ta - uw + NU - 1) / NU : 0;  // this warp's active tiles
      bool stop = false;
      switch (ns) {  // every case fully static: no predicated tensor-core instructions
#define PB_UPD(NSV) \
  case NSV:         \
    if constexpr (NSV <= SLOTS) stop = cta_update_block<T, NU, NSV>(sbase, k1, uw, g, t, &sh_fail, (streamed || P.tma) ? &sh_bar[k1] : nullptr); \
    break;
        PB_UPD(0) PB_UPD(1) PB_UPD(2) PB_UPD(3) PB_UPD(4) PB_UPD(5) PB_UPD(6) PB_UPD(7) PB_UPD(8) PB_UPD(9)
        PB_UPD(10) PB_UPD(11)
#undef PB_UPD
      }
      if (stop) {
        fail = 1;
        break;
      }
      named_sync(2, NTH);  // block k1 ready for the panel warp
    }
    if (!fail) named_sync(1, NTH);  // the last panel's publication
  }
  if ((streamed || P.tma) && sh_fail)  // a failure can stop before late panels land: no async copy may
    for (int k = 0; k < TT; ++k) mbar_wait(&sh_bar[k], 0);  // outlive the CTA (without one, all were consumed)
  __syncthreads();
  fail = sh_fail;
  if (tid == 0) { PB_STAMP(2) }

  // ---- write back (failure: only the tiles the reference had stored) ----
  int band_lo = n, band_cols = 0;
  if (fail) {
    band_lo = ((fail - 1) / 8) * 8;
    band_cols = ((fail - 1) / 4) * 4;
  }
  const int ncols = fail ? band_cols : n;
  const bool zf = P.zero_fill;
  if (P.tma && !fail) {
    // one tensor store per panel; rows past n are out of bounds (not written),
    // the diagonal blocks' strict upper parts still hold the staged originals
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      for (int k = 0; k < TT; ++k)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                         reinterpret_cast<uint64_t>(&P.tm[k])),
                     "r"(8 * k), "r"(8 * k), "r"((int)p), "r"(sbase + 8u * cta_pbase(T, k))
                     : "memory");
      bulk_commit();
      bulk_wait_read0();
    }
  } else if (!PM && !P.upper && !zf && (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0) && (n % 2 == 0)) {
    // one TMA bulk store per column for the 16-byte aligned part of rows [col, rlim);
    // an odd first row goes alone (its pair partner is in the opposite triangle)
    fence_proxy_async();  // writers fence, then the barrier, then the async-proxy stores
    __syncthreads();
    for (int col = tid; col < ncols; col += NTH) {
      const int kb = col >> 3, c = col & 7, r0 = 8 * kb;
      const int rlim = fail ? (col >= band_cols ? band_lo : band_lo + 8) : n;
      const uint32_t pc = sbase + 8u * (cta_pbase(T, kb) + c * cta_pstride(T, kb) - r0);  // + 8*row
      double* dst = a + (long long)col * lda;
      int re = col;
      if ((col & 1) && col < rlim) {
        dst[col] = lds64(pc + 8u * col);
        re = col + 1;
      }
      if (rlim > re) bulk_s2g(dst + re, pc + 8u * re, 8u * (uint32_t)(rlim - re));
    }
    bulk_commit();
    bulk_wait_read0();
  } else if (PM && !fail && ((reinterpret_cast<uintptr_t>(a) & 15) == 0)) {
    // panel-major, no failure: rows (2q, 2q + 1) of a column are adjacent — 16-byte stores
    // for the pairs wholly in the lower triangle, single elements across the diagonal
    // (and the LowerZero zeros of the diagonal block's upper part when asked for)
    for (int kb = 0; kb < TT; ++kb) {
      const uint32_t pb = sbase + 8u * cta_pbase(T, kb);
      const int RS = cta_pstride(T, kb), r0 = 8 * kb, rows = min(n, 8 * TT) - r0, np = (rows + 1) >> 1;
      for (int e = tid; e < 8 * np; e += NTH) {
        const int c = e / np, r = 2 * (e - c * np), row = r0 + r, col = r0 + c;
        if (col >= n) continue;
        double* dp = a + cta_eoff<PM>(0, lda, row, col);
        if (r >= c && row + 1 < n) {
          double v0, v1;
          lds128(pb + 8u * (c * RS + r), v0, v1);
          *reinterpret_cast<double2*>(dp) = make_double2(v0, v1);
        } else {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (row + u >= n) continue;
            if (r + u >= c) dp[u] = lds64(pb + 8u * (c * RS + r + u));
            else if (zf) dp[u] = 0.0;
          }
        }
      }
    }
  } else {
    for (int kb = 0; kb * 8 < ncols; ++kb) {
      const uint32_t pb = sbase + 8u * cta_pbase(T, kb);
      const int RS = cta_pstride(T, kb), r0 = 8 * kb, rows = min(n, 8 * TT) - r0;
      for (int e = tid; e < 8 * rows; e += NTH) {
        const int c = e / rows, r = e - c * rows, row = r0 + r, col = r0 + c;
        if (col >= ncols || row >= n) continue;
        const int rlim = fail ? (col >= band_cols ? band_lo : band_lo + 8) : n;
        if (row >= rlim) continue;
        if (row < col && !zf) continue;
        const double v = row >= col ? lds64(pb + 8u * (c * RS + r)) : 0.0;
        a[cta_eoff<PM>(P.upper, lda, row, col)] = v;
      }
    }
  }
  if (tid == 0) P.info[p] = fail ? fail + P.info_offset : 0;
  if (tid == 0) { PB_STAMP(3) }
}

template <int T, int NU, int PM>
static cudaError_t cta_launch_t(const PotrfCtaArgs& P, cudaStream_t s) {
  const size_t smem = (size_t)(cta_pbase(T, T) + 8 * T + 32) * sizeof(double);  // + panel-warp read slack
  {
    // residency is bounded by shared memory: ask for the largest carveout
    cudaError_t e = smem_attr((const void*)potrf_cta_kernel<T, NU, PM>, (int)smem, true);
    if (e != cudaSuccess) return e;
  }
  potrf_cta_kernel<T, NU, PM><<<(unsigned)P.batch, 32 * (NU + 1), smem, s>>>(P);
  return cudaGetLastError();
}

// PBGPU_POTRF_NU=1|2|3 overrides the number of update warps (tuning only)
static int nu_override() {
  static const int v = [] {
    const char* e = getenv("PBGPU_POTRF_NU");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// an update warp owns at most 11 tiles of a column block (cta_update_block's switch)
template <int T, int NU>
constexpr bool nu_ok() { return (T - 1 + NU - 1) / NU <= 11; }

template <int T, int NUDEF, int PM>
static cudaError_t launch_nu(const PotrfCtaArgs& P, cudaStream_t s) {
  static_assert(nu_ok<T, NUDEF>(), "too many tiles per update warp");
  const int nu = nu_override();
  if constexpr (nu_ok<T, 1>()) if (nu == 1) return cta_launch_t<T, 1, PM>(P, s);
  if constexpr (nu_ok<T, 2>()) if (nu == 2) return cta_launch_t<T, 2, PM>(P, s);
  if (nu == 3) return cta_launch_t<T, 3, PM>(P, s);
  return cta_launch_t<T, NUDEF, PM>(P, s);
}

template <int PM>
static cudaError_t cta_dispatch(const PotrfCtaArgs& P, int nmax, cudaStream_t s) {
  switch ((nmax + 7) / 8) {
#define PB_CASE(TV, NUV) \
  case TV:               \
    return launch_nu<TV, NUV, PM>(P, s);
    // update warps per order, measured (tools/quick_potrf.py, PBGPU_POTRF_NU sweeps):
    // one update warp keeps the most CTAs resident up to n = 80
    PB_CASE(1, 1) PB_CASE(2, 1) PB_CASE(3, 1) PB_CASE(4, 1) PB_CASE(5, 1) PB_CASE(6, 1)
    PB_CASE(7, 1) PB_CASE(8, 1) PB_CASE(9, 1) PB_CASE(10, 1) PB_CASE(11, 2) PB_CASE(12, 2)
    PB_CASE(13, 3) PB_CASE(14, 3) PB_CASE(15, 3) PB_CASE(16, 3) PB_CASE(17, 3) PB_CASE(18, 3)
    PB_CASE(19, 3) PB_CASE(20, 3)
#undef PB_CASE
  }
  return cudaErrorInvalidValue;
}

static PFN_cuTensorMapEncodeTiled_v12000 cta_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    cudaGetLastError();
  });
  return fn;
}

// Per-panel tensor maps for packed lower column-major batches (the config-3
// shape); false when the layout rules TMA out.  The last encoded set is cached
// (the maps only depend on the base pointer and the shape).
static bool cta_tensor_maps(PotrfCtaArgs& P) {
  if (P.upper || P.offs || P.nvec || P.pa || P.src || P.syrk_only || P.zero_fill) return false;
  if ((P.n & 7) || P.n <= 0 || P.n > 8 * kCtaMaxT || P.batch <= 0) return false;
  if ((reinterpret_cast<uintptr_t>(P.a) & 15) || (P.lda & 1) || (P.batch > 1 && (P.stride & 1))) return false;
  if (P.lda < P.n || (P.batch > 1 && P.stride < (long long)P.lda * P.n)) return false;
  static const bool off = [] {
    const char* e = getenv("PBGPU_POTRF_TMA");
    return e && e[0] == '0';
  }();
  if (off) return false;
  auto enc = cta_encode_fn();
  if (!enc) return false;
  struct Key {
    const double* a;
    long long stride;
    int lda, n, batch;
  };
  static thread_local Key last{nullptr, 0, 0, 0, 0};
  static thread_local CUtensorMap cache[kCtaMaxT];
  const int T = P.n / 8;
  if (!(last.a == P.a && last.stride == P.stride && last.lda == P.lda && last.n == P.n && last.batch == P.batch)) {
    for (int k = 0; k < T; ++k) {
      cuuint64_t dims[3] = {(cuuint64_t)P.n, (cuuint64_t)P.n, (cuuint64_t)P.batch};
      cuuint64_t strides[2] = {(cuuint64_t)P.lda * 8, (cuuint64_t)(P.batch > 1 ? P.stride : (long long)P.lda * P.n) * 8};
      cuuint32_t box[3] = {(cuuint32_t)cta_pstride(T, k), 8u, 1u};
      cuuint32_t es[3] = {1, 1, 1};
      if (enc(&cache[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, P.a, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        last = Key{nullptr, 0, 0, 0, 0};
        return false;
      }
    }
    last = Key{P.a, P.stride, P.lda, P.n, P.batch};
  }
  for (int k = 0; k < T; ++k) P.tm[k] = cache[k];
  return true;
}

cudaError_t potrf_cta_launch(double* a, long long stride, const long long* offs, const int* nvec, int lda,
                             int n, int upper, int pm, int zero_fill, int* info, int info_offset,
                             int skip_nonzero, int batch, cudaStream_t s) {
  // orders <= 32: the register-resident segment kernel (potrf_reg.cu);
  // PBGPU_POTRF_REG=0 keeps this kernel (A/B measurements)
  static const bool reg = [] {
    const char* e = getenv("PBGPU_POTRF_REG");
    return !(e && e[0] == '0');
  }();
  if (reg && n <= 32)
    return potrf_reg_launch(a, stride, offs, nvec, lda, n, upper, pm, zero_fill, info, info_offset, skip_nonzero,
                            batch, s);
  PotrfCtaArgs P{a, stride, offs, nvec, lda, n, upper, batch, zero_fill, info, info_offset, skip_nonzero,
                 nullptr, nullptr, 0, nullptr, 0, 0, nullptr, 0, 0, 0};
  P.tma = !pm && cta_tensor_maps(P);
  return pm ? cta_dispatch<1>(P, n, s) : cta_dispatch<0>(P, n, s);
}

cudaError_t syrk_potrf_cta_launch(double* d, long long stride_d, const long long* offs, const int* nvec, int ldd,
                                  const double* c, long long stride_c, int ldc,
                                  const double* A, const double* B, long long stride_ab, int k, int ldab,
                                  int n, int pm, int zero_fill, int* info, int batch, cudaStream_t s) {
  PotrfCtaArgs P{d, stride_d, offs, nvec, ldd, n, 0, batch, zero_fill, info, 0, 0,
                 A, B, stride_ab, offs, k, ldab, c, stride_c, ldc, 0};
  return pm ? cta_dispatch<1>(P, n, s) : cta_dispatch<0>(P, n, s);
}

cudaError_t syrk_lower_cta_launch(double* c, const long long* offs, const int* nvec, const double* A, int nmax,
                                  int pm, int* info, int batch, cudaStream_t s) {
  PotrfCtaArgs P{c, 0, offs, nvec, 0, nmax, 0, batch, 0, info, 0, 0,
                 A, A, 0, offs, 1, 0, nullptr, 0, 0, 1};
  return pm ? cta_dispatch<1>(P, nmax, s) : cta_dispatch<0>(P, nmax, s);
}

}  // namespace pbg
