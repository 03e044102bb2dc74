// Warp-per-problem batched Cholesky for n <= 64 (sm_100a), left-looking.
//
// The small-n branch of the size switch (the paper's small-size algorithm
// family; potrf_core, factor.hpp:45-99, is left-looking too).  One warp owns
// one problem and keeps its whole lower triangle in shared memory as column
// panels of 8 columns (row stride 9 doubles: row-per-lane accesses are
// conflict-free).  For every column block k:
//   1. the block's 8x8 tiles are updated, left-looking, with FP64 tensor-core
//      DMMA m8n8k4: A(k:, k) -= L(k:, 0:k) L(k, 0:k)^T, accumulators in
//      registers, fragments read straight from the factored panels;
//   2. the tall panel is factored column by column with every lane owning up
//      to two rows: pivot broadcast by shuffle, reciprocal square root,
//      scaling by the reciprocal, rank-1 updates with the diagonal column
//      broadcast through shared memory (the reference's failure test is
//      `piv <= 0.0`, micro_kernel.hpp:314; edge arithmetic in the style of
//      edge_potrf / edge_trsm_right, micro_kernel.hpp:309-356).
// Registers hold only one column block, so many problems stay resident per
// SM.  The factor is written to global memory once, coalesced, at the end:
// a failure at column p stores exactly the reference's set — all lower
// entries of rows < 8*floor(p/8) and, in that band, columns < 4*floor(p/4)
// (test_factor.cpp:251-277).  Padding rows/columns (n % 8) are identity.
//
// PM = 1 addresses panel-major storage (ps = 4, panel_mat.hpp:39-42); with
// zero_fill the strictly-upper entries of each 8-row diagonal band are
// written as zeros, the LowerZero store of syrk_potrf_nd (micro_kernel.hpp:
// 657-673, level3.hpp:528-531).
#include <cstdlib>

#include "common.cuh"
#include <cstdint>
#include "launch.h"

namespace pbg {

struct PotrfWarpArgs {
  double* a;
  long long stride;
  const long long* offs;  // optional per-problem element offsets (variable batches)
  const int* nvec;        // optional per-problem order (variable batches)
  int lda, n, upper, batch, pm, zero_fill;
  int* info;
  int info_offset;
  int skip_nonzero;
  int debug;  // profiling aid (PBGPU_POTRF_DEBUG=1 skips the factorization)
};

constexpr int kWarpsPerCta = 2;

// Panel k (rows 8k.., 8 columns) is column-major with column stride
// pstride(T, k) = 8(T-k) + 4 doubles (4 or 12 mod 16): consecutive rows are
// consecutive banks (row-per-lane accesses) and DMMA fragment loads are
// conflict-free.  Both helpers are closed forms (no loops in address math).
__host__ __device__ constexpr int pstride(int T, int k) { return 8 * (T - k) + 4; }
__host__ __device__ constexpr int panel_base(int T, int k) {
  return 64 * (k * T - k * (k - 1) / 2) + 32 * k;  // sum_{q<k} 8 * pstride(T, q)
}

template <int PM>
__device__ __forceinline__ long long eoff(int upper, long long ld, int r, int c) {
  // lower-problem element (r, c); upper runs on the transposed storage
  if (PM) return (long long)(r >> 2) * 4 * ld + (long long)c * 4 + (r & 3);
  return upper ? (long long)c + r * ld : (long long)r + c * ld;
}

// Factors the (rows x 8) panel at `pan` (column stride RS) in place; lane owns
// row `lane` and, when TWO, row `lane + 32`.  Returns 0 or the failing local
// column (1-based).  `gcol0` is the panel's first global column (failure test
// only applies to real columns < n).
template <bool TWO>
__device__ __forceinline__ int factor_panel(uint32_t pan, int RS, int rows, int lane, uint32_t colb,
                                            int gcol0, int n) {
  const unsigned FULL = 0xffffffffu;
  const bool has0 = lane < rows, has1 = TWO && lane + 32 < rows;
  double x[8], y[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    x[c] = has0 ? lds64(pan + 8u * (c * RS + lane)) : 0.0;
    if (TWO) y[c] = has1 ? lds64(pan + 8u * (c * RS + lane + 32)) : 0.0;
  }
  int f = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double piv = __shfl_sync(FULL, x[c], c);
    if (gcol0 + c < n && piv <= 0.0) {
      f = c + 1;
      break;
    }
    const double inv = rsqrt(piv);
    const double sq = piv * inv;
    if (lane == c) x[c] = sq;
    else if (lane > c) x[c] *= inv;
    if (TWO) y[c] *= inv;
    if (c < 7) {
      // L(c+1..7, c) broadcast through shared memory (8-aligned slots)
      if (lane > c && lane < 8) sts64(colb + 8u * lane, x[c]);
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
        if (lane >= c2) x[c2] -= x[c] * fc[c2];
        if (TWO) y[c2] -= y[c] * fc[c2];
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (has0) sts64(pan + 8u * (c * RS + lane), x[c]);
    if (TWO && has1) sts64(pan + 8u * (c * RS + lane + 32), y[c]);
  }
  __syncwarp();
  return f;
}

// One left-looking step k with TA = T - k active 8x8 tiles below/at the
// diagonal: DMMA update of column block k from the factored panels 0..k-1,
// then the panel factorization.  Returns 0 or the failing local column.
template <int T, int TA>
__device__ __forceinline__ int potrf_step(uint32_t sbase, int k, int lane, int g, int t, uint32_t colb, int n) {
  const int RS = pstride(T, k);
  const uint32_t pan = sbase + 8u * panel_base(T, k);
  if (k > 0) {
    double acc[TA][2];
#pragma unroll
    for (int I = 0; I < TA; ++I) {
      acc[I][0] = lds64(pan + 8u * ((2 * t) * RS + 8 * I + g));
      acc[I][1] = lds64(pan + 8u * ((2 * t + 1) * RS + 8 * I + g));
    }
    uint32_t pl = sbase + 8u * (8 * k);  // row 8k of panel 0
    for (int l = 0; l < k; ++l) {
      const int RL = pstride(T, l);
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint32_t col = pl + 8u * ((4 * kk + t) * RL + g);
        const double bneg = -lds64(col);  // -L(8k+g, 8l+4kk+t)
#pragma unroll
        for (int I = 0; I < TA; ++I) dmma(acc[I][0], acc[I][1], lds64(col + 8u * (8 * I)), bneg);
      }
      pl += 8u * (8 * RL - 8);  // next panel, same global row 8k
    }
#pragma unroll
    for (int I = 0; I < TA; ++I) {
      sts64(pan + 8u * ((2 * t) * RS + 8 * I + g), acc[I][0]);
      sts64(pan + 8u * ((2 * t + 1) * RS + 8 * I + g), acc[I][1]);
    }
    __syncwarp();
  }
  return factor_panel<(TA > 4)>(pan, RS, 8 * TA, lane, colb, 8 * k, n);
}

template <int T, int PM>
__global__ void __launch_bounds__(32 * kWarpsPerCta) potrf_warp_kernel(const __grid_constant__ PotrfWarpArgs P) {
  constexpr int WS = panel_base(T, T) + 8;  // doubles of shared memory per warp (+ broadcast slot)
  extern __shared__ __align__(16) double smem_all[];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  const long long p = (long long)blockIdx.x * kWarpsPerCta + w;
  if (p >= P.batch) return;
  if (P.skip_nonzero && P.info[p] != 0) return;
  double* sm = smem_all + (size_t)w * WS;
  const uint32_t sbase = smem_u32(sm), colb = sbase + 8u * (WS - 8);
  const int n = P.nvec ? P.nvec[p] : P.n;
  if (n <= 0) {
    if (lane == 0) P.info[p] = 0;
    return;
  }
  double* a = P.a + (P.offs ? P.offs[p] : p * P.stride);
  const long long lda = P.nvec ? (PM ? ((n + 3) & ~3) : n) : P.lda;
  const int TT = (n + 7) >> 3;  // active tile count (<= T for variable batches)
  const bool pairs = !PM && !P.upper && (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0);

  // ---- load the lower triangle into the panels, every copy in flight at once:
  // 16-byte cp.async.cg row pairs where aligned, else 8-byte zero-filling
  // copies.  The upper entries of the diagonal tiles that come along are never
  // used; rows/columns past n become identity. ----
  for (int k = 0; k < TT; ++k) {
    double* pan = sm + panel_base(T, k);
    const int RS = pstride(T, k), r0 = 8 * k, nr = min(n, 8 * TT) - r0;
    if (pairs) {
      const double* src = a + r0 + (long long)r0 * lda;
      const int np = nr >> 1;
      // np <= 32 (rows <= 64): one predicated copy per lane and column
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (lane < np && r0 + c < n) cp_async16(&pan[c * RS + 2 * lane], src + c * lda + 2 * lane);
      if ((nr & 1) && lane < 8 && r0 + lane < n)
        cp_async8(&pan[lane * RS + nr - 1], src + lane * lda + nr - 1, true);
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int col = r0 + c;
        for (int r = lane; r < nr; r += 32) {
          const int row = r0 + r;
          const bool v = col < n && row >= col;
          cp_async8(&pan[c * RS + r], v ? a + eoff<PM>(P.upper, lda, row, col) : a, v);
        }
      }
    }
  }
  cp_async_wait_all();
  if (n & 7) {  // identity padding: rows >= n of every panel, columns >= n of the last
    for (int k = 0; k < TT; ++k) {
      double* pan = sm + panel_base(T, k);
      const int RS = pstride(T, k), rows = 8 * (TT - k);
      for (int e = lane; e < 8 * rows; e += 32) {
        const int c = e / rows, r = e - c * rows, row = 8 * k + r, col = 8 * k + c;
        if (row >= n || col >= n) pan[c * RS + r] = (row == col) ? 1.0 : 0.0;
      }
    }
  }
  __syncwarp();

  int fail = 0;
  for (int k = 0; k < TT && P.debug != 1; ++k) {
    int f = 0;
    switch (TT - k) {  // every step body is fully static in its active tile count
#define PB_STEP(TA) \
  case TA:          \
    if constexpr (TA <= T) f = potrf_step<T, TA>(sbase, k, lane, g, t, colb, n); \
    break;
      PB_STEP(1) PB_STEP(2) PB_STEP(3) PB_STEP(4) PB_STEP(5) PB_STEP(6) PB_STEP(7) PB_STEP(8)
#undef PB_STEP
    }
    if (f) {
      fail = 8 * k + f;
      break;
    }
  }

  // ---- write back, coalesced (failure: only the tiles the reference had stored) ----
  int band_lo = n, band_cols = 0;
  if (fail) {
    band_lo = ((fail - 1) / 8) * 8;
    band_cols = ((fail - 1) / 4) * 4;
  }
  const int ncols = fail ? band_cols : n;
  const bool zf = P.zero_fill;
  for (int kb = 0; kb * 8 < ncols; ++kb) {
    const uint32_t pb = sbase + 8u * panel_base(T, kb);
    const int RS = pstride(T, kb), r0 = 8 * kb;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = r0 + c;
      if (col < ncols) {
        const int rlim = min(n, fail ? (col >= band_cols ? band_lo : band_lo + 8) : n);
        const uint32_t pc = pb + 8u * (c * RS - r0);  // + 8*row
        if (pairs && !zf) {
          // 16-byte row pairs; an odd first row goes alone (its partner is upper)
          double* dst = a + (long long)col * lda;
          const int q0 = col >> 1, q1 = rlim >> 1;
          const int q = q0 + lane;  // q1 - q0 <= 32: one predicated pair per lane
          if (q < q1) {
            const int row = 2 * q;
            if (row >= col) {
              double2 v;
              asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(pc + 8u * row));
              *reinterpret_cast<double2*>(dst + row) = v;
            } else {
              dst[row + 1] = lds64(pc + 8u * (row + 1));
            }
          }
          if ((rlim & 1) && lane == 0 && rlim - 1 >= col) dst[rlim - 1] = lds64(pc + 8u * (rlim - 1));
        } else {
          const int rlo = zf ? r0 : col;  // zero_fill: the band's upper part too
          for (int row = rlo + lane; row < rlim; row += 32) {
            const double v = row >= col ? lds64(pc + 8u * row) : 0.0;
            a[eoff<PM>(P.upper, lda, row, col)] = v;
          }
        }
      }
    }
  }
  if (lane == 0) P.info[p] = fail ? fail + P.info_offset : 0;
}

static int debug_mode() {
  static int m = [] {
    const char* e = getenv("PBGPU_POTRF_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return m;
}

template <int T, int PM>
static cudaError_t launch_t(const PotrfWarpArgs& P, cudaStream_t s) {
  const size_t smem = (size_t)kWarpsPerCta * (panel_base(T, T) + 8) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(potrf_warp_kernel<T, PM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const unsigned grid = (unsigned)((P.batch + kWarpsPerCta - 1) / kWarpsPerCta);
  potrf_warp_kernel<T, PM><<<grid, 32 * kWarpsPerCta, smem, s>>>(P);
  return cudaGetLastError();
}

template <int PM>
static cudaError_t dispatch(const PotrfWarpArgs& P, int nmax, cudaStream_t s) {
  switch ((nmax + 7) / 8) {
    case 1: return launch_t<1, PM>(P, s);
    case 2: return launch_t<2, PM>(P, s);
    case 3: return launch_t<3, PM>(P, s);
    case 4: return launch_t<4, PM>(P, s);
    case 5: return launch_t<5, PM>(P, s);
    case 6: return launch_t<6, PM>(P, s);
    case 7: return launch_t<7, PM>(P, s);
    case 8: return launch_t<8, PM>(P, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t potrf_warp_launch(double* a, long long stride, int lda, int n, int upper, int* info,
                              int info_offset, int skip_nonzero, int batch, cudaStream_t s) {
  PotrfWarpArgs P{a, stride, nullptr, nullptr, lda, n, upper, batch, 0, 0, info, info_offset, skip_nonzero, debug_mode()};
  return dispatch<0>(P, n, s);
}

cudaError_t potrf_warp_pm_launch(double* a, long long stride, const long long* offs, const int* nvec,
                                 int cn, int n, int zero_fill, int* info, int batch, cudaStream_t s) {
  PotrfWarpArgs P{a, stride, offs, nvec, cn, n, 0, batch, 1, zero_fill, info, 0, 0, 0};
  return dispatch<1>(P, n, s);
}

}  // namespace pbg
