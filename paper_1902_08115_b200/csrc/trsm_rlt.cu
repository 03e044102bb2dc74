// Batched right-side triangular solve X * A^T = alpha * B with A lower
// ("rltn"/"rltu": the config-5 step, trsm_rltn_nd and the blocked Cholesky's
// panel solve), warp-per-8-rows, left-looking on FP64 tensor cores (sm_100a).
//
// Replaces trsm_right_core / kernel_trsm_right (level3.hpp:174-214,
// micro_kernel.hpp:522-543) and trsm_rltn_nd (level3.hpp:484-526) for this
// flag set.  Rows of X are independent, so one warp owns 8 rows of one
// problem and needs no barrier at all.  For column tile J (8 columns, in
// dependency order: A^T is upper, so ascending):
//   1. C = alpha * B(rows, J) - X(rows, 0:8J) * A(J, 0:8J)^T, accumulated with
//      DMMA m8n8k4 in registers: the solved X lives in the warp's shared
//      memory slice already in A-fragment order (one conflict-free 256-byte
//      load per DMMA), the A(J, :) fragments come through L1;
//   2. the 8x8 diagonal block is solved by substitution inside each quad of
//      lanes (a lane owns two columns of a row; the solved value travels by
//      shuffle), with the reference's reciprocal multiply
//      (micro_kernel.hpp:351-352);
//   3. the tile is stored and re-laid as A fragments for the next tiles.
// An exactly-zero non-unit diagonal is found before any store and reported
// (level3.hpp:292-299).  Column- and panel-major (ps = 4) storage; uniform or
// variable (config-5) batches.
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace pbg {

constexpr int kRltWarps = 4;

struct RltArgs {
  TrsmLaunch L;
  int rbmax;  // row blocks (8 rows) per problem slot in the grid
  int ntmax;  // column tiles of the largest problem (shared-memory slice)
  double* W;  // inverses of the 8x8 diagonal blocks, [problem][tile][kk][lane] (B-fragment order)
};

template <int PM>
__device__ __forceinline__ long long rlt_off(long long ld, int r, int c) {
  if (PM) return (long long)(r >> 2) * 4 * ld + (long long)c * 4 + (r & 3);
  return (long long)r + (long long)c * ld;
}

// Inverses of the 8x8 diagonal blocks of A, one thread per (problem, tile,
// column j): forward substitution L y = e_j with reciprocal multiplies
// (identity past n; a unit diagonal is taken as 1).  Stored where lane
// (g, t) of the solve reads its B fragment inv(L)[g][4 kk + t].
template <int PM>
__global__ void __launch_bounds__(256) diag_inv8_kernel(const __grid_constant__ RltArgs R) {
  const TrsmLaunch& L = R.L;
  const long long e = (long long)blockIdx.x * 256 + threadIdx.x;
  const long long p = e / (R.ntmax * 8);
  if (p >= L.batch) return;
  const int rem = (int)(e - p * R.ntmax * 8), J = rem >> 3, j = rem & 7;
  int n = L.nn;
  long long lda = L.lda;
  const double* A;
  if (L.nvec) {
    n = L.nvec[p];
    lda = PM ? ((n + 3) & ~3) : n;
    A = L.a + L.offs[p];
  } else {
    A = L.a + (L.offs_a ? L.offs_a[p] : p * L.sa);
  }
  if (8 * J >= n) return;
  auto el = [&](int i, int l) -> double {  // L_JJ(i, l), l <= i
    const int r = 8 * J + i, c = 8 * J + l;
    if (r >= n || c >= n) return i == l ? 1.0 : 0.0;
    if (i == l && L.unit) return 1.0;
    return A[rlt_off<PM>(lda, r, c)];
  };
  double y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i < j) {
      y[i] = 0.0;
    } else {
      double acc = i == j ? 1.0 : 0.0;
#pragma unroll
      for (int l = 0; l < i; ++l)
        if (l >= j) acc = fma(-el(i, l), y[l], acc);
      y[i] = acc * __drcp_rn(el(i, i));
    }
  }
  double* w = R.W + (p * R.ntmax + J) * 64 + (j >> 2) * 32 + (j & 3);
#pragma unroll
  for (int i = 0; i < 8; ++i) w[4 * i] = y[i];
}

// Staged rows of A: column c of the 8-row block at c*8, rows XOR-swizzled so
// a B-fragment load (rows g, columns 4K + t) touches 16 distinct banks per
// half-warp.
__device__ __forceinline__ int ab_idx(int c, int g) { return c * 8 + (g ^ (((c >> 1) & 1) << 2)); }

// Exact redo of one warp's 8 rows when its fast solve met an Inf / NaN (rare):
// substitution in the reference's order (edge_trsm_right, micro_kernel.hpp:
// 330-356) straight from B, which the fast path leaves untouched until its
// final store — so no structural zero of inv(L_JJ) meets an Inf or NaN
// (0 * Inf = NaN there, not in the reference).  Lane g (t == 0) owns row g.
template <int PM>
__device__ __noinline__ void rlt_rows_exact(const TrsmLaunch& L, const double* A, const double* B, double* D,
                                            long long lda, long long ldb, long long ldd, int n, int m, int r0,
                                            int lane) {
  const int r = r0 + (lane >> 2);
  if ((lane & 3) != 0 || r >= m) return;
  auto xo = [&](long long ld, int rr, int cc) -> long long {
    return (!PM && L.twin) ? (long long)cc + (long long)rr * ld : rlt_off<PM>(ld, rr, cc);
  };
  for (int c = 0; c < n; ++c) {
    double x = L.alpha * B[xo(ldb, r, c)];
    for (int l = 0; l < c; ++l) x -= D[xo(ldd, r, l)] * A[rlt_off<PM>(lda, c, l)];
    if (!L.unit) x *= 1.0 / A[rlt_off<PM>(lda, c, c)];
    D[xo(ldd, r, c)] = x;
  }
}

// NT > 0: register-resident variant for up to NT column tiles — the solved X
// stays in registers (A-fragment order, 2 doubles per tile and lane), the
// tile loops are fully unrolled, and shared memory holds only the staged rows
// of A, so residency is no longer bounded by 8 rows x n of X per warp.
template <int PM, int NT>
__global__ void __launch_bounds__(32 * kRltWarps, NT > 20 ? 3 : NT > 12 ? 4 : NT > 0 ? 5 : 1)
    trsm_rlt_kernel(const __grid_constant__ RltArgs R) {  // (register caps at the residency the X tiles allow)
  extern __shared__ __align__(16) double sm_all[];
  const TrsmLaunch& L = R.L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, tid = threadIdx.x;
  const int cpp = (R.rbmax + kRltWarps - 1) / kRltWarps;  // CTAs per problem
  const long long p = blockIdx.x / cpp;
  const int rb = (int)(blockIdx.x - p * cpp) * kRltWarps + warp;
  if (p >= L.batch) return;                              // CTA-uniform
  if (L.skip_nonzero && L.info[p] != 0) return;          // CTA-uniform
  int n = L.nn, m = L.mm;
  long long lda = L.lda, ldb = L.ldb, ldd = L.ldd;
  const double *A, *B;
  double* D;
  if (L.nvec) {
    n = m = L.nvec[p];
    lda = ldb = ldd = PM ? ((n + 3) & ~3) : n;
    A = L.a + L.offs[p];
    B = L.b + L.offs[p];
    D = L.d + L.offs[p];
  } else {
    A = L.a + (L.offs_a ? L.offs_a[p] : p * L.sa);
    B = L.b + (L.offs_b ? L.offs_b[p] : p * L.sb);
    D = L.d + (L.offs_b ? L.offs_b[p] : p * L.sd);
  }
  if ((rb - warp) * 8 >= m) return;  // CTA-uniform: no row of this CTA exists
  // ---- zero diagonal: smallest exactly-zero index, before any store ----
  if (!L.unit) {
    unsigned z = 0xffffffffu;
    for (int i = lane; i < n; i += 32)
      if (A[rlt_off<PM>(lda, i, i)] == 0.0) z = min(z, (unsigned)i);
    z = __reduce_min_sync(0xffffffffu, z);
    if (z != 0xffffffffu) {  // same verdict in every warp: the CTA leaves together
      if (rb == 0 && lane == 0 && L.info && !L.skip_nonzero) L.info[p] = (int)z + 1;
      return;
    }
  }
  const int nt = (n + 7) >> 3;
  const int r = rb * 8 + g;
  const bool rok = r < m;
  constexpr bool REG = NT > 0;
  // right-hand sides / inverse fragments two tiles ahead: 24 more registers, which the
  // variants sitting on their register cap (NT = 20, 32) would spill (measured slower there)
  constexpr bool DEEP = REG && NT != 20 && NT != 32;
  const uint32_t xs = smem_u32(sm_all + (size_t)warp * R.ntmax * 64);  // [tile][kk][lane] (shared variant)
  double* ab_base = sm_all + (REG ? 0 : (size_t)kRltWarps * R.ntmax * 64);  // 2 x [8 * ntmax * 8]
  double xr[NT > 0 ? NT : 1][2];                                          // (register variant)
  const int abs = R.ntmax * 64;
  const double alpha = L.alpha;
  // stage rows 8J..8J+7, columns 0..8J+7 of A (16-byte pairs of rows; rows past n are zero)
  // stage rows 8J..8J+7, columns 0..8J+7 of A (16-byte pairs of rows; rows past n are zero):
  // thread tid always copies the pair (8J + 2(tid & 3), +1) of columns tid/4, tid/4 + 32, ...
  const bool pair_al = (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (PM || lda % 2 == 0);
  auto stage = [&](int J) {
    double* ab = ab_base + (REG ? J % 3 : J & 1) * abs;
    const int cols = 8 * J + 8, g2 = (tid & 3) * 2, row = 8 * J + g2;
    const bool r0 = row < n, r1 = row + 1 < n;
    if (r1 && pair_al && cols <= n) {
      // every pair whole and aligned (all tiles but a ragged last one): one
      // pointer pair stepped by 32 columns, no per-copy index math or checks
      // (the generic loop below had cost half of the kernel's instructions)
      int c = tid >> 2;
      const double* src = A + rlt_off<PM>(lda, row, c);
      const long long sstep = PM ? 4LL * 8 * kRltWarps : (long long)lda * 8 * kRltWarps;
      double* dst = ab + ab_idx(c, g2);
      for (; c < cols; c += 8 * kRltWarps, src += sstep, dst += 64 * kRltWarps) cp_async16(dst, src);
      return;
    }
    for (int c = tid >> 2; c < cols; c += 8 * kRltWarps) {
      double* dst = ab + ab_idx(c, g2);
      const bool v0 = r0 && c < n, v1 = r1 && c < n;
      const double* src = A + rlt_off<PM>(lda, v0 ? row : 0, v0 ? c : 0);
      if (v1 && pair_al) {
        cp_async16(dst, src);
      } else {
        cp_async8(dst, src, v0);
        cp_async8(dst + 1, v1 ? A + rlt_off<PM>(lda, row + 1, c) : A, v1);
      }
    }
  };
  // register variant: three row buffers, staged two tiles ahead in cp.async
  // groups (the wait at a tile's top is for a copy issued two tiles earlier)
  stage(0);
  if constexpr (REG) {
    cp_async_commit();
    if (nt > 1) stage(1);
    cp_async_commit();
  }
  // X(r, c) of the effective problem: B / D element (r, c), or (c, r) for a Left
  // solve run as its transposed twin (level3.hpp:300-303; column-major only)
  auto xo = [&](long long ld, int rr, int cc) -> long long {
    return (!PM && L.twin) ? (long long)cc + (long long)rr * ld : rlt_off<PM>(ld, rr, cc);
  };
  bool bad = false;  // this lane saw a non-finite X
  double wn0 = R.W[p * R.ntmax * 64 + lane], wn1 = R.W[p * R.ntmax * 64 + 32 + lane];  // tile 0's inverse
  // this lane's right-hand sides: B(r, 8J + 2t) and its right neighbour, tile J at brow + J * bstep8
  const double* brow = B + xo(ldb, rok ? r : 0, 2 * t);
  const long long bstep1 = (!PM && L.twin) ? 1 : PM ? 4 : ldb, bstep8 = 8 * bstep1;
  // register variant: slot J % 3 holds tile J's right-hand side pair and inverse
  // fragments, loaded two tiles ahead (early tiles are shorter than a DRAM round trip)
  double pb0[3], pb1[3], pw0[3], pw1[3];
  auto ld_rhs = [&](int J, double& b0, double& b1) {
    const int ca = 8 * J + 2 * t;
    b0 = (rok && ca < n) ? brow[J * bstep8] : 0.0;
    b1 = (rok && ca + 1 < n) ? brow[J * bstep8 + bstep1] : 0.0;
  };
  auto ld_inv = [&](int J, double& w0, double& w1) {
    const double* w = R.W + (p * R.ntmax + J) * 64 + lane;
    w0 = w[0];
    w1 = w[32];
  };
  double nb0 = (rok && 2 * t < n) ? brow[0] : 0.0;
  double nb1 = (rok && 2 * t + 1 < n) ? brow[bstep1] : 0.0;
  if constexpr (DEEP) {
    pb0[0] = nb0; pb1[0] = nb1; pw0[0] = wn0; pw1[0] = wn1;
    pb0[1] = pb1[1] = pw0[1] = pw1[1] = 0.0;
    if (nt > 1) { ld_rhs(1, pb0[1], pb1[1]); ld_inv(1, pw0[1], pw1[1]); }
  }
#pragma unroll
  for (int J = 0; J < (REG ? NT : 1 << 30); ++J) {
    if (J >= nt) break;
    if constexpr (REG) cp_async_wait_group1();
    else cp_async_wait_all();
    __syncthreads();  // rows of tile J staged; every warp is done with tile J-1's buffer
    if constexpr (REG) {
      if (J + 2 < nt) stage(J + 2);
      cp_async_commit();  // (an empty group keeps the count in step)
    } else {
      if (J + 1 < nt) stage(J + 1);
    }
    const double* ab = ab_base + (REG ? J % 3 : J & 1) * abs;
    const uint32_t abu = smem_u32(ab);
    const int ca = 8 * J + 2 * t, cb = ca + 1;
    double acc0, acc1;
    if constexpr (DEEP) {
      acc0 = alpha * pb0[J % 3];
      acc1 = alpha * pb1[J % 3];
      if (J + 2 < nt) ld_rhs(J + 2, pb0[(J + 2) % 3], pb1[(J + 2) % 3]);
    } else {
      acc0 = alpha * nb0;
      acc1 = alpha * nb1;
      if (J + 1 < nt) {  // next tile's right-hand side, loaded under this tile's work
        nb0 = (rok && ca + 8 < n) ? brow[(J + 1) * bstep8] : 0.0;
        nb1 = (rok && cb + 8 < n) ? brow[(J + 1) * bstep8 + bstep1] : 0.0;
      }
    }
    // ---- C -= X(:, 0:8J) A(J, 0:8J)^T ----
    double e0 = 0.0, e1 = 0.0;  // second accumulator pair: two independent DMMA chains
    int T2 = 0;
#pragma unroll
    for (; T2 + 2 <= J; T2 += 2) {
      double xa[4], bf[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if constexpr (REG) xa[u] = xr[T2 + (u >> 1)][u & 1];
        else xa[u] = lds64(xs + 8u * ((2 * T2 + u) * 32 + lane));
        bf[u] = -lds64(abu + 8u * ab_idx(8 * T2 + 4 * u + t, g));
      }
      dmma(acc0, acc1, xa[0], bf[0]);
      dmma(e0, e1, xa[2], bf[2]);
      dmma(acc0, acc1, xa[1], bf[1]);
      dmma(e0, e1, xa[3], bf[3]);
    }
    if (T2 < J) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        double xa;
        if constexpr (REG) xa = xr[T2][u];
        else xa = lds64(xs + 8u * ((2 * T2 + u) * 32 + lane));
        const double bf = -lds64(abu + 8u * ab_idx(8 * T2 + 4 * u + t, g));
        dmma(acc0, acc1, xa, bf);
      }
    }
    acc0 += e0;
    acc1 += e1;
    // ---- 8x8 diagonal block: X = C inv(L_JJ)^T on the tensor cores (C re-laid as A fragments) ----
    {
      const int s0 = (lane & ~3) | (t >> 1), s1 = (lane & ~3) | (2 + (t >> 1));
      const double u00 = __shfl_sync(0xffffffffu, acc0, s0), u01 = __shfl_sync(0xffffffffu, acc1, s0);
      const double u10 = __shfl_sync(0xffffffffu, acc0, s1), u11 = __shfl_sync(0xffffffffu, acc1, s1);
      double w0, w1;
      if constexpr (DEEP) {
        w0 = pw0[J % 3];
        w1 = pw1[J % 3];
        if (J + 2 < nt) ld_inv(J + 2, pw0[(J + 2) % 3], pw1[(J + 2) % 3]);
      } else {
        w0 = wn0;
        w1 = wn1;
        if (J + 1 < nt) ld_inv(J + 1, wn0, wn1);  // next tile's inverse fragments, under this tile's solve
      }
      acc0 = acc1 = 0.0;
      dmma(acc0, acc1, (t & 1) ? u01 : u00, w0);
      dmma(acc0, acc1, (t & 1) ? u11 : u10, w1);
      // an Inf / NaN in C or in inv(L_JJ) always leaves a non-finite X
      bad |= !(isfinite(acc0) && isfinite(acc1));
    }
    // ---- re-lay as A fragments: kk = 0 needs column t, kk = 1 column 4 + t ----
    const int src0 = (lane & ~3) | (t >> 1), src1 = (lane & ~3) | (2 + (t >> 1));
    const double v00 = __shfl_sync(0xffffffffu, acc0, src0), v01 = __shfl_sync(0xffffffffu, acc1, src0);
    const double v10 = __shfl_sync(0xffffffffu, acc0, src1), v11 = __shfl_sync(0xffffffffu, acc1, src1);
    if constexpr (REG) {
      xr[REG ? J : 0][0] = (t & 1) ? v01 : v00;
      xr[REG ? J : 0][1] = (t & 1) ? v11 : v10;
    } else {
      sts64(xs + 8u * ((2 * J) * 32 + lane), (t & 1) ? v01 : v00);
      sts64(xs + 8u * ((2 * J + 1) * 32 + lane), (t & 1) ? v11 : v10);
      __syncwarp();
    }
  }
  cp_async_wait_all();
  // D is written only now (B, which it may alias, is intact until here): the
  // fast result, or — when a tile met an Inf / NaN — the exact redo of the rows
  if (__any_sync(0xffffffffu, bad)) {
    rlt_rows_exact<PM>(L, A, B, D, lda, ldb, ldd, n, m, rb * 8, lane);
  } else {
    // lane (g, t) holds X(r, 8J + t) and X(r, 8J + 4 + t) (A-fragment order)
    double* drow = D + xo(ldd, rok ? r : 0, t);
    const long long dstep1 = (!PM && L.twin) ? 1 : PM ? 4 : ldd;
#pragma unroll
    for (int J = 0; J < (REG ? NT : 1 << 30); ++J) {
      if (J >= nt) break;
      double v0, v1;
      if constexpr (REG) {
        v0 = xr[REG ? J : 0][0];
        v1 = xr[REG ? J : 0][1];
      } else {
        v0 = lds64(xs + 8u * ((2 * J) * 32 + lane));
        v1 = lds64(xs + 8u * ((2 * J + 1) * 32 + lane));
      }
      const int c0 = 8 * J + t, c1 = c0 + 4;
      if (rok && c0 < n) drow[J * 8 * dstep1] = v0;
      if (rok && c1 < n) drow[(J * 8 + 4) * dstep1] = v1;
    }
  }
  if (rb == 0 && lane == 0 && L.info && !L.skip_nonzero) L.info[p] = 0;
}


bool trsm_rlt_ok(const TrsmLaunch& L) { return !(L.twin && L.pm) && L.lower && L.trans && L.nn <= 512; }
// (offs_a / offs_b are honoured only here: trsm_launch forwards every such launch to this kernel)

cudaError_t trsm_rlt_launch(const TrsmLaunch& L, cudaStream_t s) {
  if (L.batch <= 0 || L.mm <= 0 || L.nn <= 0) return cudaSuccess;
  RltArgs R;
  R.L = L;
  R.ntmax = (L.nn + 7) / 8;
  R.rbmax = L.nvec ? R.ntmax : (L.mm + 7) / 8;
  // register variant up to 32 tiles (PBGPU_TRSM_REG=0 disables it: A/B)
  static const bool reg_ok = [] {
    const char* e = getenv("PBGPU_TRSM_REG");
    return !(e && e[0] == '0');
  }();
  // (measured: no gain up to 8 tiles, 1.2x at 16, 1.6x at 32)
  const int ntr = !reg_ok || R.ntmax <= 8 || R.ntmax > 32 ? 0 : ((R.ntmax + 3) & ~3);  // a multiple of 4 tiles
  // register variant: 3 staged A row buffers; shared variant: the warps' X slices + 2 buffers
  const size_t smem = (size_t)(ntr ? 3 : kRltWarps + 2) * R.ntmax * 64 * sizeof(double);
  {
    cudaError_t e = smem_attr((const void*)(L.pm ? trsm_rlt_kernel<1, 0> : trsm_rlt_kernel<0, 0>), 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  const unsigned grid = (unsigned)((long long)L.batch * ((R.rbmax + kRltWarps - 1) / kRltWarps));
  mempool_keep();
  cudaError_t e = cudaMallocAsync(&R.W, sizeof(double) * 64 * R.ntmax * (size_t)L.batch, s);
  if (e != cudaSuccess) return e;
  const unsigned igrid = (unsigned)(((long long)L.batch * R.ntmax * 8 + 255) / 256);
  if (L.pm) diag_inv8_kernel<1><<<igrid, 256, 0, s>>>(R);
  else diag_inv8_kernel<0><<<igrid, 256, 0, s>>>(R);
#define PB_RLT(PMV, NTV) trsm_rlt_kernel<PMV, NTV><<<grid, 32 * kRltWarps, smem, s>>>(R)
  switch (ntr * 2 + L.pm) {
    case 24: PB_RLT(0, 12); break;
    case 25: PB_RLT(1, 12); break;
    case 40: PB_RLT(0, 20); break;
    case 41: PB_RLT(1, 20); break;
    case 56: PB_RLT(0, 28); break;
    case 57: PB_RLT(1, 28); break;
    case 32: PB_RLT(0, 16); break;
    case 33: PB_RLT(1, 16); break;
    case 48: PB_RLT(0, 24); break;
    case 49: PB_RLT(1, 24); break;
    case 64: PB_RLT(0, 32); break;
    case 65: PB_RLT(1, 32); break;
    default:
      if (L.pm) PB_RLT(1, 0);
      else PB_RLT(0, 0);
  }
#undef PB_RLT
  e = cudaGetLastError();
  cudaFreeAsync(R.W, s);
  return e;
}

}  // namespace pbg
