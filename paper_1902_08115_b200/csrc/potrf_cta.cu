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
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace pbg {

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
};

__host__ __device__ constexpr int cta_pstride(int T, int k) { return 8 * (T - k) + 4; }
__host__ __device__ constexpr int cta_pbase(int T, int k) { return 64 * (k * T - k * (k - 1) / 2) + 32 * k; }

template <int PM>
__device__ __forceinline__ long long cta_eoff(int upper, long long ld, int r, int c) {
  if (PM) return (long long)(r >> 2) * 4 * ld + (long long)c * 4 + (r & 3);
  return upper ? (long long)c + r * ld : (long long)r + c * ld;
}

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// Panel warp: factor the (rows x 8) panel in place; lane owns rows lane + 32 q.
template <int R>
__device__ __forceinline__ int cta_factor_panel(uint32_t pan, int RS, int rows, int lane, uint32_t colb,
                                                int gcol0, int n) {
  const unsigned FULL = 0xffffffffu;
  double x[R][8];
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[q][c] = (lane + 32 * q < rows) ? lds64(pan + 8u * (c * RS + lane + 32 * q)) : 0.0;
  int f = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double piv = __shfl_sync(FULL, x[0][c], c);
    if (gcol0 + c < n && piv <= 0.0) {
      f = c + 1;
      break;
    }
    const double inv = rsqrt(piv);
    if (lane == c) x[0][c] = piv * inv;
    else if (lane > c) x[0][c] *= inv;
#pragma unroll
    for (int q = 1; q < R; ++q) x[q][c] *= inv;
    if (c < 7) {
      if (lane > c && lane < 8) sts64(colb + 8u * lane, x[0][c]);
      __syncwarp();
      double fc[8];
#pragma unroll
      for (int c2 = (c + 1) & ~1; c2 < 8; c2 += 2) {
        double2 v;
        asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(colb + 8u * c2));
        fc[c2] = v.x;
        fc[c2 + 1] = v.y;
      }
#pragma unroll
      for (int c2 = c + 1; c2 < 8; ++c2) {
        if (lane >= c2) x[0][c2] -= x[0][c] * fc[c2];
#pragma unroll
        for (int q = 1; q < R; ++q) x[q][c2] -= x[q][c] * fc[c2];
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (lane + 32 * q < rows) sts64(pan + 8u * (c * RS + lane + 32 * q), x[q][c]);
  return f;
}

// Update warp: column block k1's tiles I = uw + NU*s (s < NS) accumulate
// -sum_l L(I, l) L(k1, l)^T over l < k1 (panel k1-1 after its publication),
// then go back to shared memory.  Returns true when the panel warp reported
// a failure (the block is then left untouched).
template <int T, int NU, int NS>
__device__ __forceinline__ bool cta_update_block(uint32_t sbase, int k1, int uw, int g, int t, const int* sh_fail) {
  constexpr int NTH = 32 * (NU + 1);
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
  for (int l = 0; l < k1; ++l) {
    if (l == k1 - 1) {
      named_sync(1, NTH);  // wait for panel k1-1
      if (*(volatile const int*)sh_fail) return true;
    }
    const int RL = cta_pstride(T, l);
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t col = pl + 8u * ((4 * kk + t) * RL);
      const double bneg = -lds64(col);
#pragma unroll
      for (int s = 0; s < NS; ++s) dmma(acc[s][0], acc[s][1], lds64(col + 8u * (8 * (uw + NU * s))), bneg);
    }
    pl += 8u * (8 * RL - 8);
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int I = uw + NU * s;
    sts64(pan + 8u * ((2 * t) * RS + 8 * I + g), acc[s][0]);
    sts64(pan + 8u * ((2 * t + 1) * RS + 8 * I + g), acc[s][1]);
  }
  return false;
}

template <int T, int NU, int PM>
__global__ void __launch_bounds__(32 * (NU + 1)) potrf_cta_kernel(const __grid_constant__ PotrfCtaArgs P) {
  constexpr int NTH = 32 * (NU + 1);
  constexpr int R = (8 * T + 31) / 32;           // rows per lane in the panel warp
  constexpr int SLOTS = (T + NU - 1) / NU;       // tiles per update warp
  extern __shared__ __align__(16) double sm[];
  __shared__ int sh_fail;
  __shared__ __align__(8) uint64_t sh_bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const long long p = blockIdx.x;
  if (P.skip_nonzero && P.info[p] != 0) return;
  const int n = P.nvec ? P.nvec[p] : P.n;
  if (n <= 0) {
    if (tid == 0) P.info[p] = 0;
    return;
  }
  double* a = P.a + (P.offs ? P.offs[p] : p * P.stride);
  const long long lda = P.nvec ? (PM ? ((n + 3) & ~3) : n) : P.lda;
  const int TT = (n + 7) >> 3;
  const uint32_t sbase = smem_u32(sm), colb = sbase + 8u * cta_pbase(T, T);

  // ---- stage the lower triangle (panel k: rows 8k.. of columns 8k..8k+7) ----
  const double* sa = P.src ? P.src + (P.offs ? P.offs[p] : p * P.src_stride) : a;
  const long long sld = P.src ? (P.nvec ? lda : P.src_ld) : lda;
  const bool bulk = !PM && !P.upper && (sld % 2 == 0) && ((reinterpret_cast<uintptr_t>(sa) & 15) == 0) &&
                    (n % 2 == 0);
  if (bulk) {
    // one TMA bulk copy per column (rows 8k..n-1 of column col, k = col/8)
    if (tid == 0) {
      mbar_init(&sh_bar, 1);
      fence_mbar_init();
      uint32_t bytes = 0;
      for (int k = 0; k < TT; ++k) bytes += 8u * (uint32_t)min(8, n - 8 * k) * (uint32_t)(n - 8 * k);
      mbar_arrive_expect_tx(&sh_bar, bytes);
    }
    __syncthreads();
    for (int col = tid; col < n; col += NTH) {
      const int k = col >> 3, c = col & 7, r0 = 8 * k;
      bulk_g2s(sm + cta_pbase(T, k) + c * cta_pstride(T, k), sa + r0 + (long long)col * sld,
               8u * (uint32_t)(n - r0), &sh_bar);
    }
    mbar_wait(&sh_bar, 0);
  } else {
    const bool pairs = !PM && !P.upper && (sld % 2 == 0) && ((reinterpret_cast<uintptr_t>(sa) & 15) == 0);
    for (int k = 0; k < TT; ++k) {
      double* pan = sm + cta_pbase(T, k);
      const int RS = cta_pstride(T, k), r0 = 8 * k, nr = min(n, 8 * TT) - r0;
      if (pairs) {
        const int np = (nr + 1) >> 1, tot = 8 * np;
        const double* src = sa + r0 + (long long)r0 * sld;
        for (int e = tid; e < tot; e += NTH) {
          const int c = e / np, q = e - c * np;
          if (r0 + c >= n) continue;
          if (2 * q + 1 < nr) cp_async16(&pan[c * RS + 2 * q], src + c * sld + 2 * q);
          else cp_async8(&pan[c * RS + 2 * q], src + c * sld + 2 * q, true);
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
  cp_async_wait_all();
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
  if (tid == 0) sh_fail = 0;
  __syncthreads();

  int fail = 0;
  if (P.syrk_only) {
    // no factorization: fall through to the write back of the lower triangle
  } else if (warp == 0) {
    // ------------------------------------------------------------ panel warp
    for (int k = 0; k < TT; ++k) {
      if (k > 0) named_sync(2, NTH);  // block k updated and stored
      const int RS = cta_pstride(T, k), rows = 8 * (TT - k);
      const int f = cta_factor_panel<R>(sbase + 8u * cta_pbase(T, k), RS, rows, lane, colb, 8 * k, n);
      if (f && lane == 0) sh_fail = 8 * k + f;
      named_sync(1, NTH);  // panel k published (or the failure flag)
      if (f) break;
    }
  } else {
    // ------------------------------------------------------------ update warps
    const int uw = warp - 1;
    for (int k1 = 1; k1 < TT; ++k1) {  // block to update; panel k1-1 is being factored
      const int ta = TT - k1;
      const int ns = uw < ta ? (ta - uw + NU - 1) / NU : 0;  // this warp's active tiles
      bool stop = false;
      switch (ns) {  // every case fully static: no predicated tensor-core instructions
#define PB_UPD(NSV) \
  case NSV:         \
    if constexpr (NSV <= SLOTS) stop = cta_update_block<T, NU, NSV>(sbase, k1, uw, g, t, &sh_fail); \
    break;
        PB_UPD(0) PB_UPD(1) PB_UPD(2) PB_UPD(3) PB_UPD(4) PB_UPD(5) PB_UPD(6) PB_UPD(7)
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
  __syncthreads();
  fail = sh_fail;

  // ---- write back (failure: only the tiles the reference had stored) ----
  int band_lo = n, band_cols = 0;
  if (fail) {
    band_lo = ((fail - 1) / 8) * 8;
    band_cols = ((fail - 1) / 4) * 4;
  }
  const int ncols = fail ? band_cols : n;
  const bool zf = P.zero_fill;
  if (!PM && !P.upper && !zf && (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0) && (n % 2 == 0)) {
    // one TMA bulk store per column for the 16-byte aligned part of rows [col, rlim);
    // an odd first row goes alone (its pair partner is in the opposite triangle)
    fence_proxy_async();
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
}

template <int T, int NU, int PM>
static cudaError_t cta_launch_t(const PotrfCtaArgs& P, cudaStream_t s) {
  const size_t smem = (size_t)(cta_pbase(T, T) + 8) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(potrf_cta_kernel<T, NU, PM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  potrf_cta_kernel<T, NU, PM><<<(unsigned)P.batch, 32 * (NU + 1), smem, s>>>(P);
  return cudaGetLastError();
}

template <int PM>
static cudaError_t cta_dispatch(const PotrfCtaArgs& P, int nmax, cudaStream_t s) {
  switch ((nmax + 7) / 8) {
#define PB_CASE(TV, NUV) \
  case TV:               \
    return cta_launch_t<TV, NUV, PM>(P, s);
    PB_CASE(1, 1) PB_CASE(2, 1) PB_CASE(3, 1) PB_CASE(4, 1) PB_CASE(5, 2) PB_CASE(6, 2)
    PB_CASE(7, 3) PB_CASE(8, 3) PB_CASE(9, 3) PB_CASE(10, 3) PB_CASE(11, 3) PB_CASE(12, 3)
    PB_CASE(13, 3) PB_CASE(14, 3) PB_CASE(15, 3) PB_CASE(16, 3) PB_CASE(17, 3) PB_CASE(18, 3)
    PB_CASE(19, 3) PB_CASE(20, 3)
#undef PB_CASE
  }
  return cudaErrorInvalidValue;
}

cudaError_t potrf_cta_launch(double* a, long long stride, const long long* offs, const int* nvec, int lda,
                             int n, int upper, int pm, int zero_fill, int* info, int info_offset,
                             int skip_nonzero, int batch, cudaStream_t s) {
  PotrfCtaArgs P{a, stride, offs, nvec, lda, n, upper, batch, zero_fill, info, info_offset, skip_nonzero,
                 nullptr, nullptr, 0, nullptr, 0, 0, nullptr, 0, 0, 0};
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
