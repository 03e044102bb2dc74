// Square batched LU with partial pivoting, n = 8T (40..96), one CTA per problem,
// every shape a compile-time constant (sm_100a).
//
// The same algorithm as getrf_cta.cu (factor.hpp:105-230: panel warp with
// virtual interchanges, update warps with look-ahead, DMMA trailing updates)
// specialised for the config-4 shapes: the order n and the shared-memory column
// stride S are template constants, so every shared-memory access is a 32-bit
// address plus an immediate, no loop carries 64-bit index math, and the panel
// code is instantiated per remaining height.  getrf_cta spent ~15.6K warp
// instructions per 48x48 problem, most of them address arithmetic and
// predication of the generic shape (ncu: issue-bound at 43 % of the issue
// slots with 18 warps per SM); this kernel does the same arithmetic in a third
// of the instructions.
//   * Pivot rule (factor.hpp:141-148): strict '>' scan from the diagonal, ties
//     to the lowest current position, a NaN diagonal keeps its row, NaN
//     candidates never win — one 64-bit key per row (|v| bits; all-ones for a
//     NaN diagonal, 0 for other NaNs), reduced as a redux.sync max of the high
//     word and a ballot; only a tie in the high word takes the low-word and
//     position reductions.
//   * Every lane forms the correctly rounded reciprocal of ITS OWN candidate
//     while the reductions are in flight; the winner publishes it with its
//     row, so the reciprocal's latency is off the per-column chain (same value
//     as 1.0 / pivot, factor.hpp:154).
//   * Zero pivot: first failing column recorded, no swap, no scaling
//     (157-158); zero multipliers skip only the rest of their nr = 4 column
//     group (160-165).
//   * Update warps, per 8-column tile: the block's interchanges (175-183) as
//     ONE composed move list (<= 16 rows change position per block: all loads,
//     then all stores — no dependent swap chain; left tiles too, eagerly), the
//     unit-lower solve of U12 (188-199) as inv(L11) A12 on DMMA with the exact
//     substitution for any tile whose result is not finite (the explicit
//     inverse would turn 0 * Inf into NaN where the reference never multiplies),
//     and A22 -= L21 U12 accumulated straight into the C tiles on DMMA.  Tile
//     k+1 goes first (exact substitution, no wait for the inverse) and is
//     handed to the panel warp (look-ahead), row tiles split across the warps.
// Measured (tools/getrf_trace.cu): the panel warp is the critical path at
// ~800-1000 cycles per column under load (460 alone); splitting it over one
// warp per 32 rows, and a one-redux pivot search with the reciprocal pinned
// ahead of it, were both neutral (profiles/r02_experiments).
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace pbg {

struct GetrfSqArgs {
  double* a;
  long long stride;
  int lda;
  int* ipiv;
  long long sp;
  int* info;
  int piv_offset;  // added to the recorded pivots / failing column (trailing block of the blocked path)
  int keep_info;   // keep an info already set by an earlier panel
  int left_cols;   // columns left of the block (same rows) that take its interchanges at the end
};

__host__ __device__ constexpr int sq_stride(int T) {  // = 4 mod 16 doubles: conflict-free DMMA fragments
  const int r = 8 * T;
  const int s = ((r - 4 + 15) / 16) * 16 + 4;
  return s < r ? s + 16 : s;
}

// PB_SQ_TRACE (tools/getrf_trace.cu only): clock64 stamps of the phases of a few CTAs
#ifdef PB_SQ_TRACE
__device__ long long sq_trace[128][128];
#define SQ_STAMP(slot) \
  if ((blockIdx.x & 63) == 0 && (blockIdx.x >> 6) < 128 && (slot) < 128) sq_trace[blockIdx.x >> 6][slot] = clock64();
#else
#define SQ_STAMP(slot)
#endif

__device__ __forceinline__ void sq_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// Panel warp: factor block k (columns c0..c0+7, rows c0..N-1; RK rows per lane)
// in registers with virtual interchanges, write it back at the final positions
// and record the pivots.  Returns the updated first-zero column (1-based, 0 = none).
template <int T, int RK>
__device__ __forceinline__ int sq_panel(uint32_t sbase, int c0, int lane, uint32_t scr, int* piv_all, int* mv,
                                        int* perm, int fz) {
  constexpr int N = 8 * T, S = sq_stride(T);
  double x[RK][8];
  int pos[RK];
  bool done[RK];
  const uint32_t blk = sbase + 8u * (uint32_t)(c0 + c0 * S);  // (c0, c0)
#pragma unroll
  for (int q = 0; q < RK; ++q) {
    const int r = c0 + lane + 32 * q;
    pos[q] = r;
    done[q] = r >= N;
#pragma unroll
    for (int c = 0; c < 8; ++c) x[q][c] = r < N ? lds64(blk + 8u * (uint32_t)(lane + 32 * q + c * S)) : 0.0;
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int col = c0 + c;
    // ---- this lane's best candidate ----
    unsigned long long bk = 0;
    unsigned bp = 0xffffffffu;
    double bv = 1.0;
#pragma unroll
    for (int q = 0; q < RK; ++q) {
      const double v = fabs(x[q][c]);
      const unsigned long long key =
          isnan(v) ? (pos[q] == col ? ~0ull : 0ull) : (unsigned long long)__double_as_longlong(v);
      const bool better = !done[q] && (key > bk || (key == bk && (unsigned)pos[q] < bp));
      bk = better ? key : bk;
      bp = better ? (unsigned)pos[q] : bp;
      bv = better ? x[q][c] : bv;
    }
    const double rcp = __drcp_rn(bv);  // speculative: overlaps the reductions below
    const bool has = bp != 0xffffffffu;
    const unsigned hi = (unsigned)(bk >> 32), lo = (unsigned)bk;
    const unsigned khi = __reduce_max_sync(0xffffffffu, has ? hi : 0u);
    bool win = has && hi == khi;
    if (__popc(__ballot_sync(0xffffffffu, win)) != 1) {  // tie in the high word (rare): full key, lowest position
      const unsigned klo = __reduce_max_sync(0xffffffffu, win ? lo : 0u);
      win = win && lo == klo;
      const unsigned q0 = __reduce_min_sync(0xffffffffu, win ? bp : 0xffffffffu);
      win = win && bp == q0;
    }
    // ---- the winner publishes its row (from column c, in pairs), reciprocal and position ----
    const uint32_t ub = scr + (c & 1) * 80;
    if (win) {
#pragma unroll
      for (int q = 0; q < RK; ++q)
        if (!done[q] && (unsigned)pos[q] == bp) {
#pragma unroll
          for (int cc = c & ~1; cc < 8; cc += 2) sts128(ub + 8u * cc, x[q][cc], x[q][cc + 1]);
        }
      sts128(ub + 64, rcp, __longlong_as_double((long long)bp));
    }
    __syncwarp();
    double u[8], inv, pbits;
#pragma unroll
    for (int cc = c & ~1; cc < 8; cc += 2) lds128(ub + 8u * cc, u[cc], u[cc + 1]);
    lds128(ub + 64, inv, pbits);
    const int pr = (int)__double_as_longlong(pbits);
    const bool nz = u[c] != 0.0;
    if (lane == 0) piv_all[col] = pr;
    if (!nz && fz == 0) fz = col + 1;
#pragma unroll
    for (int q = 0; q < RK; ++q) {
      if (nz && !done[q]) pos[q] = pos[q] == pr ? col : (pos[q] == col ? pr : pos[q]);
      const bool act = !done[q] && pos[q] != col;
      done[q] = done[q] || pos[q] == col;
      if (act) {
        if (nz) x[q][c] *= inv;
        const double f = x[q][c];
        // zero multipliers skip only the rest of the nr = 4 column group
        // (factor.hpp:160-165); the next group takes the plain update
#pragma unroll
        for (int c2 = c + 1; c2 < 8; ++c2)
          if (f != 0.0 || c2 > (c | 3)) x[q][c2] = fma(-f, u[c2], x[q][c2]);
      }
    }
  }
  // rows at their final positions (the positions are a permutation of the rows),
  // and the block's interchanges composed into a move list for the other
  // columns: mv[1 + i] = src | dst << 16 for every row whose position changed
  // (at most 16: eight pivot rows up, the rows they displaced down), mv[0] = count
  const uint32_t colb = sbase + 8u * (uint32_t)(c0 * S);
  int base = 0;
#pragma unroll
  for (int q = 0; q < RK; ++q) {
    const int r = c0 + lane + 32 * q;
    if (r < N) {
      const uint32_t d = colb + 8u * (uint32_t)pos[q];
#pragma unroll
      for (int c = 0; c < 8; ++c) sts64(d + 8u * (uint32_t)(c * S), x[q][c]);
    }
    const bool moved = r < N && pos[q] != r;
    const unsigned m = __ballot_sync(0xffffffffu, moved);
    if (moved) mv[1 + base + __popc(m & ((1u << lane) - 1u))] = r | (pos[q] << 16);
    base += __popc(m);
  }
  if (lane == 0) mv[0] = base;
  if (perm) {  // warp-uniform: running row permutation (final position <- original row) for the left columns
    __syncwarp();
    const int e = lane < base ? mv[1 + lane] : 0;
    const int src = lane < base ? perm[e & 0xffff] : 0;
    __syncwarp();
    if (lane < base) perm[e >> 16] = src;
  }
  return fz;
}

// Update warps: block k's interchanges on the 8 columns of tile J, as the
// composed move list (all loads, then all stores).  Lane = column (lane & 7) x
// move slot (lane >> 3); up to 16 moves.
template <int T>
__device__ __forceinline__ void sq_tile_moves(uint32_t sbase, int J, const int* mv, int lane) {
  constexpr int S = sq_stride(T);
  const int cnt = mv[0];
  if (cnt == 0) return;  // warp-uniform
  const uint32_t colb = sbase + 8u * (uint32_t)((8 * J + (lane & 7)) * S);
  const int s = lane >> 3;
  double v[4];
  int dst[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = s + 4 * i;
    const int e = m < cnt ? mv[1 + m] : 0;
    dst[i] = e >> 16;
    v[i] = m < cnt ? lds64(colb + 8u * (uint32_t)(e & 0xffff)) : 0.0;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (s + 4 * i < cnt) sts64(colb + 8u * (uint32_t)dst[i], v[i]);
  __syncwarp();
}

// inv(L11) of block k (unit lower 8x8): lane j < 8 solves column j against e_j;
// mbuf[col * 8 + row] (the layout of the DMMA A fragments below)
template <int T>
__device__ __forceinline__ void sq_inverse(uint32_t sbase, int c0, uint32_t mbuf, int lane) {
  constexpr int S = sq_stride(T);
  if (lane >= 8) return;
  const uint32_t lb = sbase + 8u * (uint32_t)(c0 + c0 * S);  // L11
  double y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double sacc = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int l = 0; l < i; ++l) sacc = fma(-lds64(lb + 8u * (uint32_t)(i + l * S)), y[l], sacc);
    y[i] = sacc;
  }
#pragma unroll
  for (int i = 0; i < 8; i += 2) sts128(mbuf + 8u * (uint32_t)(lane * 8 + i), y[i], y[i + 1]);
}

// U12 tile J: U(k,J) = inv(L11) A(k,J) on DMMA.  A tile whose result is not
// finite (Inf/NaN operands, overflow: 0 * Inf of the explicit inverse would
// differ from the reference's substitution, factor.hpp:188-199) is redone by
// that substitution, one lane per column.
template <int T>
__device__ __forceinline__ void sq_tile_solve(uint32_t sbase, int c0, int J, uint32_t mbuf, int lane, int g,
                                              int t) {
  constexpr int S = sq_stride(T);
  const uint32_t bcol = sbase + 8u * (uint32_t)(c0 + t + (8 * J + g) * S);
  const double b0 = lds64(bcol), b1 = lds64(bcol + 32);
  const double m0 = lds64(mbuf + 8u * (uint32_t)(t * 8 + g)), m1 = lds64(mbuf + 8u * (uint32_t)((4 + t) * 8 + g));
  // transposed product U^T = A12^T inv(L11)^T: the lane's results are rows 2t, 2t+1 of column g
  double d0 = 0.0, d1 = 0.0;
  dmma(d0, d1, b0, m0);
  dmma(d0, d1, b1, m1);
  const bool fin = fabs(d0) <= 1.7976931348623157e308 && fabs(d1) <= 1.7976931348623157e308;
  if (__all_sync(0xffffffffu, fin)) {
    sts128(sbase + 8u * (uint32_t)(c0 + 2 * t + (8 * J + g) * S), d0, d1);
  } else if (lane < 8) {
    const uint32_t ub = sbase + 8u * (uint32_t)(c0 + (8 * J + lane) * S);
    const uint32_t lb = sbase + 8u * (uint32_t)(c0 + c0 * S);
    double u[8];
#pragma unroll
    for (int c = 0; c < 8; c += 2) lds128(ub + 8u * c, u[c], u[c + 1]);
#pragma unroll
    for (int c = 1; c < 8; ++c)
#pragma unroll
      for (int l = 0; l < c; ++l) u[c] -= u[l] * lds64(lb + 8u * (uint32_t)(c + l * S));
#pragma unroll
    for (int c = 0; c < 8; c += 2) sts128(ub + 8u * c, u[c], u[c + 1]);
  }
  __syncwarp();
}

// Exact unit-lower solve of U12 for columns [j0, j1) against L11 (factor.hpp:188-199),
// one thread per column (the look-ahead tile; its interchanges are already applied).
template <int T, int NU>
__device__ __forceinline__ void sq_swap_solve(uint32_t sbase, int c0, const int* piv_all, int j0, int j1, int utid) {
  constexpr int S = sq_stride(T), NUT = 32 * NU;
  (void)piv_all;
  for (int j = j0 + utid; j < j1; j += NUT) {
    const uint32_t ub = sbase + 8u * (uint32_t)(c0 + j * S);
    const uint32_t lb = sbase + 8u * (uint32_t)(c0 + c0 * S);  // L11
    double u[8];
#pragma unroll
    for (int c = 0; c < 8; c += 2) lds128(ub + 8u * c, u[c], u[c + 1]);
#pragma unroll
    for (int c = 1; c < 8; ++c)
#pragma unroll
      for (int l = 0; l < c; ++l) u[c] -= u[l] * lds64(lb + 8u * (uint32_t)(c + l * S));
#pragma unroll
    for (int c = 0; c < 8; c += 2) sts128(ub + 8u * c, u[c], u[c + 1]);
  }
}

// One column tile J against row tiles I = i0, i0 + istep, .. < ti: C(I,J) -= L(I,k) U(k,J),
// computed as the transposed product C^T -= U^T L^T (the DMMA operands swap
// roles), so a lane's two accumulators are rows 2t, 2t+1 of ONE column of the
// tile: one 16-byte shared-memory access each way instead of two 8-byte ones
// two columns apart (ncu: the C tiles were 39 % of the kernel's shared-memory
// wavefronts, half of them bank conflicts of the column-pair pattern).
template <int T>
__device__ __forceinline__ void sq_tile_col(uint32_t sbase, int c0, int J, int i0, int istep, int ti, int g,
                                            int t) {
  constexpr int S = sq_stride(T);
  const uint32_t ucol = sbase + 8u * (uint32_t)(c0 + t + (8 * J + g) * S);
  const double b0 = -lds64(ucol), b1 = -lds64(ucol + 32);                           // U(k,J)^T fragments (A operand)
  const uint32_t arow = sbase + 8u * (uint32_t)(c0 + 8 + g + (c0 + t) * S);         // L(I,k)^T fragments (B operand)
  const uint32_t crow = sbase + 8u * (uint32_t)(c0 + 8 + 2 * t + (8 * J + g) * S);  // C(I,J): rows 2t, 2t+1 of column g
  int I = i0;
  for (; I + istep < ti; I += 2 * istep) {  // two tiles in flight
    const uint32_t a = arow + 64u * (uint32_t)I, cc = crow + 64u * (uint32_t)I;
    const uint32_t a2 = a + 64u * (uint32_t)istep, cc2 = cc + 64u * (uint32_t)istep;
    const double a0 = lds64(a), a1 = lds64(a + 8u * (4 * S));
    const double e0 = lds64(a2), e1 = lds64(a2 + 8u * (4 * S));
    double d0, d1, f0, f1;
    lds128(cc, d0, d1);
    lds128(cc2, f0, f1);
    dmma(d0, d1, b0, a0);
    dmma(f0, f1, b0, e0);
    dmma(d0, d1, b1, a1);
    dmma(f0, f1, b1, e1);
    sts128(cc, d0, d1);
    sts128(cc2, f0, f1);
  }
  if (I < ti) {
    const uint32_t a = arow + 64u * (uint32_t)I, cc = crow + 64u * (uint32_t)I;
    const double a0 = lds64(a), a1 = lds64(a + 8u * (4 * S));
    double d0, d1;
    lds128(cc, d0, d1);
    dmma(d0, d1, b0, a0);
    dmma(d0, d1, b1, a1);
    sts128(cc, d0, d1);
  }
}

__host__ __device__ constexpr int sq_min_blocks(int T, int NU) {
  const int by_smem = 233472 / (8 * sq_stride(T) * 8 * T + 2048);
  const int by_regs = 65536 / (32 * (NU + 1) * 104);
  const int b = by_smem < by_regs ? by_smem : by_regs;
  return b < 1 ? 1 : b;
}

template <int T, int NU>
__global__ void __launch_bounds__(32 * (NU + 1), sq_min_blocks(T, NU)) getrf_sq_kernel(const __grid_constant__ GetrfSqArgs P) {
  constexpr int N = 8 * T, S = sq_stride(T), NTH = 32 * (NU + 1), R = (N + 31) / 32;
  extern __shared__ __align__(16) double sm[];
  __shared__ int piv_all[N];                  // 0-based pivot row of every column
  __shared__ __align__(16) double scr[2][10];  // pivot row broadcast: 8 values, reciprocal, position
  __shared__ int mvl[2][20];                   // composed interchanges of block k (double-buffered)
  __shared__ int perm_s[N];                    // left_cols > 0: final position <- original row of the block
  __shared__ __align__(16) double minv[64];    // inv(L11) of the current block
  __shared__ int first_zero;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long p = blockIdx.x;
  double* a = P.a + p * P.stride;
  const uint32_t sbase = smem_u32(sm);
  if (tid == 0) { SQ_STAMP(0) }

  // ---- stage: one TMA bulk copy per column ----
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bar, 8u * N * N);
    first_zero = 0;
  }
  if (P.left_cols > 0)
    for (int i = tid; i < N; i += NTH) perm_s[i] = i;
  __syncthreads();
  for (int j = tid; j < N; j += NTH) bulk_g2s(sm + j * S, a + (long long)j * P.lda, 8u * N, &bar);
  mbar_wait(&bar, 0);
  __syncthreads();

  if (warp == 0) {
    // ---------------------------------------------------------------- panel warp
    int fz = 0;
    const uint32_t scr0 = smem_u32(&scr[0][0]);
    for (int k = 0; k < T; ++k) {
      if (k > 0) sq_sync(2, NTH);  // block k fully updated
      if (tid == 0) { SQ_STAMP(4 * k + 4) }
      const int c0 = 8 * k;
      const int rk = (N - c0 + 31) >> 5;  // rows per lane follow the remaining height
      int* mv = mvl[k & 1];
      int* perm = P.left_cols > 0 ? perm_s : nullptr;
      if (R >= 3 && rk == 3) fz = sq_panel<T, (R >= 3 ? 3 : 1)>(sbase, c0, lane, scr0, piv_all, mv, perm, fz);
      else if (R >= 2 && rk == 2) fz = sq_panel<T, (R >= 2 ? 2 : 1)>(sbase, c0, lane, scr0, piv_all, mv, perm, fz);
      else fz = sq_panel<T, 1>(sbase, c0, lane, scr0, piv_all, mv, perm, fz);
      if (tid == 0) { SQ_STAMP(4 * k + 5) }
      sq_sync(1, NTH);  // panel k and its pivots published
    }
    if (lane == 0) first_zero = fz;
  } else {
    // ---------------------------------------------------------------- update warps
    const int uw = warp - 1, g = lane >> 2, t = lane & 3;
    const uint32_t mbuf = smem_u32(&minv[0]);
    for (int k = 0; k < T; ++k) {
      sq_sync(1, NTH);  // panel k published
      const int c0 = 8 * k, ti = T - k - 1;  // row tiles below the block
      const int* mv = mvl[k & 1];
      if (k + 1 < T) {
        // look-ahead: tile k+1 first (update warp 0 moves and solves it by the
        // exact substitution, no wait for the inverse), row tiles split across the warps
        if (uw == 0) {
          sq_tile_moves<T>(sbase, k + 1, mv, lane);
          sq_swap_solve<T, 1>(sbase, c0, piv_all, c0 + 8, c0 + 16, lane);
        }
        if (NU > 1) sq_sync(3, 32 * NU);
        else __syncwarp();
        sq_tile_col<T>(sbase, c0, k + 1, uw, NU, ti, g, t);
        if (uw == 0 && lane == 0) { SQ_STAMP(4 * k + 6) }
        sq_sync(2, NTH);  // block k+1 ready for the panel warp
        // the rest: inv(L11), then per column tile the interchanges (left tiles
        // too), the DMMA solve and the trailing update
        if (uw == 0) sq_inverse<T>(sbase, c0, mbuf, lane);
        for (int J = uw; J < k; J += NU) sq_tile_moves<T>(sbase, J, mv, lane);
        if (NU > 1) sq_sync(3, 32 * NU);
        else __syncwarp();
        for (int J = k + 2 + uw; J < T; J += NU) {
          sq_tile_moves<T>(sbase, J, mv, lane);
          sq_tile_solve<T>(sbase, c0, J, mbuf, lane, g, t);
          sq_tile_col<T>(sbase, c0, J, 0, 1, ti, g, t);
        }
        if (uw == 0 && lane == 0) { SQ_STAMP(4 * k + 7) }
      } else {
        for (int J = uw; J < k; J += NU) sq_tile_moves<T>(sbase, J, mv, lane);
      }
    }
  }
  __syncthreads();
  // ---- write back ----
  fence_proxy_async();
  __syncthreads();
  for (int j = tid; j < N; j += NTH) bulk_s2g(a + (long long)j * P.lda, sbase + 8u * (uint32_t)(j * S), 8u * N);
  bulk_commit();
  for (int j = tid; j < N; j += NTH) P.ipiv[p * P.sp + j] = piv_all[j] + 1 + P.piv_offset;
  if (tid == 0 && !(P.keep_info && P.info[p] != 0)) P.info[p] = first_zero ? first_zero + P.piv_offset : 0;
  // the block's interchanges on the columns left of it (the trailing block of the
  // blocked path; LAPACK swaps whole rows, factor.hpp:175-183): every row moves
  // from its original position to its final one, 16 columns per round, reads and
  // writes separated by barriers (the moves form a permutation)
  if (P.left_cols > 0) {
    constexpr int RR = (N + NTH - 1) / NTH;  // rows per thread
    constexpr int CW = RR > 1 ? 8 : 16;      // columns per round
    int from[RR];
    bool mvr[RR];
#pragma unroll
    for (int i = 0; i < RR; ++i) {
      const int r = tid + i * NTH;
      from[i] = r < N ? perm_s[r] : 0;
      mvr[i] = r < N && from[i] != r;
    }
    for (int q0 = -P.left_cols; q0 < 0; q0 += CW) {
      double v[RR][CW];
#pragma unroll
      for (int i = 0; i < RR; ++i)
#pragma unroll
        for (int u = 0; u < CW; ++u)
          v[i][u] = ldg_if(a + from[i] + (long long)(q0 + u) * P.lda, mvr[i] && q0 + u < 0, 0.0);
      __syncthreads();
#pragma unroll
      for (int i = 0; i < RR; ++i)
#pragma unroll
        for (int u = 0; u < CW; ++u)
          stg_if(a + tid + i * NTH + (long long)(q0 + u) * P.lda, v[i][u], mvr[i] && q0 + u < 0);
      __syncthreads();
    }
  }
  bulk_wait_read0();
  if (tid == 0) { SQ_STAMP(1) }
}

template <int T, int NU>
static cudaError_t sq_launch_t(const GetrfSqArgs& P, int batch, cudaStream_t s) {
  const size_t smem = (size_t)sq_stride(T) * 8 * T * sizeof(double);
  cudaError_t e = smem_attr((const void*)getrf_sq_kernel<T, NU>, (int)smem, true);
  if (e != cudaSuccess) return e;
  getrf_sq_kernel<T, NU><<<(unsigned)batch, 32 * (NU + 1), smem, s>>>(P);
  return cudaGetLastError();
}

// square, n = 40..96 in steps of 8, every column 16-byte aligned (TMA bulk copies)
bool getrf_sq_ok(const double* a, long long stride, int lda, int m, int n) {
  static const bool off = [] {
    const char* e = getenv("PBGPU_GETRF_SQ");
    return e && e[0] == '0';
  }();
  return !off && m == n && n >= 40 && n <= 96 && n % 8 == 0 && lda % 2 == 0 && stride % 2 == 0 &&
         (reinterpret_cast<uintptr_t>(a) & 15) == 0;
}

cudaError_t getrf_sq_launch(double* a, long long stride, int lda, int n, int* ipiv, long long sp, int* info,
                            int piv_offset, int keep_info, int left_cols, int batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  GetrfSqArgs P{a, stride, lda, ipiv, sp, info, piv_offset, keep_info, left_cols};
  // update warps per order (PBGPU_GETRF_SQ_NU = 1|2|3 overrides, tuning only)
  static const int nu_env = [] {
    const char* e = getenv("PBGPU_GETRF_SQ_NU");
    return e ? atoi(e) : 0;
  }();
  switch (n / 8) {
#define PB_SQ(TV, NUDEF)                                                     \
  case TV:                                                                   \
    if (nu_env == 1) return sq_launch_t<TV, 1>(P, batch, s);                 \
    if (nu_env == 2) return sq_launch_t<TV, 2>(P, batch, s);                 \
    if (nu_env == 3) return sq_launch_t<TV, 3>(P, batch, s);                 \
    return sq_launch_t<TV, NUDEF>(P, batch, s);
    PB_SQ(5, 1) PB_SQ(6, 1) PB_SQ(7, 2) PB_SQ(8, 2) PB_SQ(9, 3) PB_SQ(10, 3) PB_SQ(11, 3) PB_SQ(12, 3)
#undef PB_SQ
  }
  return cudaErrorInvalidValue;
}

}  // namespace pbg
