// Batched FP64 tiled gemm engine for sm_100a.
//
// Replaces the reference's five CPU packing variants (gemm.hpp:249-400) and
// the panel-major native gemm (level3.hpp:360-403) with ONE persistent,
// warp-specialised kernel:
//   * work item = (problem, 64x64 tile of C); items are dealt round-robin to
//     one resident CTA per SM;
//   * a producer warp streams op(A)/op(B) k-chunks (BK = 32) into a ring of
//     shared-memory stages with ONE TMA tensor copy per operand per stage
//     (cp.async.bulk.tensor, complete_tx on an mbarrier).  The tensor maps
//     describe the whole batch (problem index = outermost dimension) and
//     their boxes are 4 doubles wider than the tile along the contiguous
//     dimension: the TMA engine zero-fills the out-of-range lanes, which
//     gives a padded shared-memory layout (stride = 4 mod 16 doubles) so
//     every DMMA fragment load is a conflict-free 2-wavefront LDS.64.
//     Panel-major operands (ps = 4) map to 4-D tensors whose boxes land in
//     shared memory already panel-interleaved.  Misaligned operands fall
//     back to zero-filling 8-byte cp.async;
//   * eight consumer warps run FP64 tensor-core DMMA m8n8k4 on 32x16 warp
//     tiles of D' = C^T = op(B)^T op(A)^T.  Computing the transpose makes
//     every lane own two vertically adjacent C elements, so the epilogue
//     loads and stores C/D as 16-byte pairs in both column-major and
//     panel-major storage;
//   * the epilogue applies alpha/beta (beta == 0 never reads C,
//     micro_kernel.hpp:263-268) with C prefetched one item ahead, and the
//     uplo mask used by syrk (level3.hpp:220-246, 407-441).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "launch.h"

namespace pbg {

constexpr int TM = 64, TN = 64, BK = 32;
// warp tile: WH row tiles x WF column tiles of 8x8 (of D' = C^T); measured: WH = 4
// (four 32x32-tile warps, half the fragment loads per DMMA) is 25 % slower than
// eight 32x16-tile warps (WH = 2) at every compute-bound size
constexpr int WH = 2, WF = 4;
constexpr int NWR = TM / (8 * WH);                 // warps along the tile's rows
constexpr int NCW = NWR * (TN / (8 * WF));         // consumer warps
constexpr int NTHREADS = (NCW + 1) * 32;

template <int L>
struct LayT;
template <>
struct LayT<L_MNC> {  // smem (x, l) at l*S + x ; TMA box {S, BK}
  static constexpr int S = TM + 4;
  static constexpr int SIZE = BK * S;
  __device__ static __forceinline__ int at(int x, int l) { return l * S + x; }
  __device__ static __forceinline__ long long g(int ld, int x, int l) {
    return (long long)x + (long long)l * ld;
  }
};
template <>
struct LayT<L_KC> {  // smem (x, l) at x*S + l ; TMA box {S, TM}
  static constexpr int S = BK + 4;
  static constexpr int SIZE = TM * S;
  __device__ static __forceinline__ int at(int x, int l) { return x * S + l; }
  __device__ static __forceinline__ long long g(int ld, int x, int l) {
    return (long long)l + (long long)x * ld;
  }
};
template <>
struct LayT<L_PMX> {  // smem panels over x: (x/4)*P + l*4 + x%4 ; TMA box {4, BK, TM/4}
  static constexpr int P = 4 * BK;
  static constexpr int SIZE = (TM / 4) * P;
  __device__ static __forceinline__ int at(int x, int l) { return (x >> 2) * P + l * 4 + (x & 3); }
  __device__ static __forceinline__ long long g(int cn, int x, int l) {
    return (long long)(x >> 2) * 4 * cn + (long long)l * 4 + (x & 3);
  }
};
template <>
struct LayT<L_PML> {  // smem panels over l: (l/4)*P + x*4 + l%4 ; TMA box {4, TM, BK/4}
  static constexpr int P = 4 * TM;
  static constexpr int SIZE = (BK / 4) * P;
  __device__ static __forceinline__ int at(int x, int l) { return (l >> 2) * P + x * 4 + (l & 3); }
  __device__ static __forceinline__ long long g(int cn, int x, int l) {
    return (long long)(l >> 2) * 4 * cn + (long long)x * 4 + (l & 3);
  }
};

struct KParams {
  CUtensorMap tmA, tmB;  // valid when the side's `tma` flag is set
  OpDesc a, b;
  OutDesc o;
  int tmaA, tmaB;
  int bulkA, bulkB;                // per-problem offsets: column / panel bulk copies instead of a tensor map
  int batched_mapA, batched_mapB;  // 1: the tensor map has a problem dimension, 2: per-problem offset dimensions
  int m, n, k;
  double alpha, beta;
  int uplo;
  int tiles_m, tiles_n, tiles_per_problem, nk;
  long long items;
  int nstages;
  const int* skip;
  int stagger;  // cycles the second consumer warp of every scheduler partition starts late (see the consumers)
};

// tile r of a problem -> (tm, tn)
__device__ __forceinline__ void tile_of(const KParams& P, int r, int& tm, int& tn) {
  if (P.uplo == 0) {
    tn = (unsigned)r / (unsigned)P.tiles_m;
    tm = r - tn * P.tiles_m;
  } else {
    // triangular tile enumeration: r -> (hi, lo) with hi >= lo
    int hi = (int)((sqrtf(8.0f * r + 1.0f) - 1.0f) * 0.5f);
    while ((hi + 1) * (hi + 2) / 2 <= r) ++hi;
    while (hi * (hi + 1) / 2 > r) --hi;
    int lo = r - hi * (hi + 1) / 2;
    if (P.uplo == 1) { tm = hi; tn = lo; } else { tm = lo; tn = hi; }
  }
}

// A CTA's walk over its items (item = blockIdx.x + i * gridDim.x) as (problem,
// tile-in-problem), advanced without the 64-bit division per item.
struct ItemCursor {
  long long item;
  int p, r, dq, dr, tpp;
  __device__ __forceinline__ void init(const KParams& P) {
    tpp = P.tiles_per_problem;
    dq = (int)(gridDim.x / (unsigned)tpp);
    dr = (int)(gridDim.x - (unsigned)dq * (unsigned)tpp);
    item = blockIdx.x;
    p = (int)(blockIdx.x / (unsigned)tpp);
    r = (int)(blockIdx.x - (unsigned)p * (unsigned)tpp);
  }
  __device__ __forceinline__ void next() {
    item += gridDim.x;
    p += dq;
    r += dr;
    if (r >= tpp) { r -= tpp; ++p; }
  }
};

__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* tm, const int (&c)[5], int rank,
                                         uint64_t* bar) {
  const uint64_t desc = reinterpret_cast<uint64_t>(tm);
  const uint32_t d = smem_u32(dst), b = smem_u32(bar);
  if (rank == 3)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(d), "l"(desc), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(b)
        : "memory");
  else if (rank == 4)
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(d), "l"(desc), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]),
        "r"(b)
        : "memory");
  else if (rank == 5)
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(d), "l"(desc), "r"(c[0]), "r"(c[1]), "r"(c[2]),
        "r"(c[3]), "r"(c[4]), "r"(b)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(d), "l"(desc), "r"(c[0]), "r"(c[1]), "r"(b)
        : "memory");
}

// Producer, TMA path: one tensor copy for this side's chunk (lane 0).
// Coordinates innermost first.  mode 1: the map has a problem dimension
// (uniform stride); mode 2: per-problem element offsets — the map carries two
// extra dimensions of 16-byte and 16-MiB stride whose coordinates spell the
// (even) offset, so offset batches stream through the same tensor copies.
template <int L>
__device__ __forceinline__ void tma_side(const CUtensorMap* tm, int mode, int p, long long off, int x0, int l0,
                                         double* s, uint64_t* bar) {
  int c[5] = {0, 0, 0, 0, 0};
  int rank;
  if (L == L_MNC) { c[0] = x0; c[1] = l0; rank = 2; }
  else if (L == L_KC) { c[0] = l0; c[1] = x0; rank = 2; }
  else if (L == L_PMX) { c[1] = l0; c[2] = x0 >> 2; rank = 3; }
  else { c[1] = x0; c[2] = l0 >> 2; rank = 3; }
  if (mode == 1) {
    c[rank++] = p;
  } else if (mode == 2) {
    const long long o = off >> 1;
    c[rank++] = (int)(o & 0xfffff);
    c[rank++] = (int)(o >> 20);
  }
  tma_load(s, tm, c, rank, bar);
}

// Producer, fallback path: every (x, l) of the 64 x kvalid4 chunk through
// 8-byte cp.async, out-of-range entries zero-filled.
template <int L>
__device__ __forceinline__ void elem_side(const OpDesc& d, int p, int x0, int xvalid, int l0,
                                          int kvalid, double* s, int lane) {
  using T = LayT<L>;
  const double* g = d.base + (d.offs ? d.offs[p] : (long long)p * d.stride);
  const int kvalid4 = (kvalid + 3) & ~3;
  for (int e = lane; e < kvalid4 * TM; e += 32) {
    int x, l;
    if (L == L_KC || L == L_PMX) { l = e % kvalid4; x = e / kvalid4; } else { x = e % TM; l = e / TM; }
    bool v = x < xvalid && l < kvalid;
    const double* src = v ? g + T::g(d.ld, x0 + x, l0 + l) : d.base;
    cp_async8(s + T::at(x, l), src, v);
  }
}

// Producer, per-problem-offset path (no tensor map can describe the batch):
// one bulk copy per column (column-major, x contiguous: xvalid doubles) or per
// 4-row panel (panel-major: 4 kvalid doubles), spread over the lanes; k
// columns in [kvalid, kvalid rounded up to 4) are zeroed.  Lane 0 registers
// the chunk's bytes on the stage barrier once, before any lane issues.
template <int L>
__device__ __forceinline__ void bulk_side(const OpDesc& d, int p, int x0, int xvalid, int l0, int kvalid, double* s,
                                          int lane, uint64_t* bar) {
  const double* g = d.base + (d.offs ? d.offs[p] : (long long)p * d.stride);
  const int kvalid4 = (kvalid + 3) & ~3;
  if constexpr (L == L_MNC) {
    const uint32_t bytes = 8u * (uint32_t)xvalid;  // xvalid even (host check)
    if (lane == 0) mbar_expect_tx(bar, bytes * (uint32_t)kvalid);
    __syncwarp();
    const int l = lane;  // BK == 32 columns, one per lane
    if (l < kvalid) {
      bulk_g2s(s + LayT<L>::at(0, l), g + LayT<L>::g(d.ld, x0, l0 + l), bytes, bar);
    } else if (l < kvalid4) {
      for (int x = 0; x < TM; x += 2) sts128(smem_u32(s + LayT<L>::at(x, l)), 0.0, 0.0);
    }
  } else {  // L_PMX: panel q = rows x0 + 4q .. x0 + 4q + 3, columns l0 .. l0 + kvalid - 1 contiguous
    const uint32_t bytes = 32u * (uint32_t)kvalid;
    const int np = min(TM / 4, (xvalid + 3) >> 2);
    if (lane == 0) mbar_expect_tx(bar, bytes * (uint32_t)np);
    __syncwarp();
    const int q = lane;
    if (q < np) {
      bulk_g2s(s + LayT<L>::at(4 * q, 0), g + LayT<L>::g(d.ld, x0 + 4 * q, l0), bytes, bar);
      for (int e = 4 * kvalid; e < 4 * kvalid4; e += 2) sts128(smem_u32(s + LayT<L>::at(4 * q, 0) + e), 0.0, 0.0);
    }
  }
}

template <int OUT_PM>
__device__ __forceinline__ long long out_off(int ld, int i, int j) {
  if (OUT_PM) return (long long)(i >> 2) * 4 * ld + (long long)j * 4 + (i & 3);
  return (long long)i + (long long)j * ld;
}

// One item's k loop for a warp whose tile has FA x HA live 8x8 fragments (the
// others lie wholly outside m x n or the uplo triangle and stay zero): only
// the live fragments are loaded and multiplied.  Every warp, live or not,
// waits for each stage and releases it, so the ring's phases stay in step.
template <int FA, int HA, class TA, class TB>
__device__ __forceinline__ void engine_k_loop(const KParams& P, const double* smem, uint64_t* full, uint64_t* empty,
                                              int stage_doubles, int& stage, uint32_t& phase, int ib, int jb, int g,
                                              int t, int lane, double (&acc)[WF][WH][2]) {
  for (int kc = 0; kc < P.nk; ++kc) {
    const int kvalid = min(BK, P.k - kc * BK);
    mbar_wait(&full[stage], phase);
    const double* sA = smem + (size_t)stage * stage_doubles;
    const double* sB = sA + TA::SIZE;
    if constexpr (FA > 0 && HA > 0) {
      if (kvalid == BK) {
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
          const int l = ks * 4 + t;
          double av[FA], bv[HA];
#pragma unroll
          for (int f = 0; f < FA; ++f) av[f] = sB[TB::at(jb + f * 8 + g, l)];
#pragma unroll
          for (int h = 0; h < HA; ++h) bv[h] = sA[TA::at(ib + h * 8 + g, l)];
#pragma unroll
          for (int f = 0; f < FA; ++f)
#pragma unroll
            for (int h = 0; h < HA; ++h) dmma(acc[f][h][0], acc[f][h][1], av[f], bv[h]);
        }
      } else {
        // Tail chunk: lanes past k contribute exact zeros whatever the stage
        // holds (pad lanes of panel-major operands are unspecified data).
        const int ksteps = (kvalid + 3) >> 2;
        for (int ks = 0; ks < ksteps; ++ks) {
          const int l = ks * 4 + t;
          const bool in = l < kvalid;
          double av[FA], bv[HA];
#pragma unroll
          for (int f = 0; f < FA; ++f) av[f] = in ? sB[TB::at(jb + f * 8 + g, l)] : 0.0;
#pragma unroll
          for (int h = 0; h < HA; ++h) bv[h] = in ? sA[TA::at(ib + h * 8 + g, l)] : 0.0;
#pragma unroll
          for (int f = 0; f < FA; ++f)
#pragma unroll
            for (int h = 0; h < HA; ++h) dmma(acc[f][h][0], acc[f][h][1], av[f], bv[h]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == P.nstages) { stage = 0; phase ^= 1; }
  }
}

// EDGE = 1: launches with ragged tiles (m or n not a multiple of 64) or an uplo
// mask pick each warp's live fragments per item; EDGE = 0 (every tile full)
// keeps the plain loop — the per-item dispatch measured 4 % slower at k = 128.
template <int LA, int LB, int OUT_PM, int EDGE>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_tiles_kernel(const __grid_constant__ KParams P) {
  using TA = LayT<LA>;
  using TB = LayT<LB>;
  constexpr int STAGE = TA::SIZE + TB::SIZE;  // doubles
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)P.nstages * STAGE);
  uint64_t* empty = full + P.nstages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < P.nstages; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NCW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      if (P.tmaA) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&P.tmA) : "memory");
      if (P.tmaB) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&P.tmB) : "memory");
    }
    constexpr uint32_t BYTES_A = TA::SIZE * 8, BYTES_B = TB::SIZE * 8;
    int stage = 0;
    uint32_t phase = 0;
    ItemCursor cur;
    for (cur.init(P); cur.item < P.items; cur.next()) {
      const int p = cur.p;
      int tm, tn;
      tile_of(P, cur.r, tm, tn);
      if (P.skip && P.skip[p]) continue;
      const int i0 = tm * TM, j0 = tn * TN;
      const int mvalid = min(TM, P.m - i0), nvalid = min(TN, P.n - j0);
      const long long offA = P.batched_mapA == 2 ? P.a.offs[p] : 0, offB = P.batched_mapB == 2 ? P.b.offs[p] : 0;
      for (int kc = 0; kc < P.nk; ++kc) {
        const int l0 = kc * BK, kvalid = min(BK, P.k - l0);
        mbar_wait(&empty[stage], phase ^ 1);
        double* sA = smem + (size_t)stage * STAGE;
        double* sB = sA + TA::SIZE;
        if (lane == 0) {
          const uint32_t bytes = (P.tmaA ? BYTES_A : 0) + (P.tmaB ? BYTES_B : 0);
          if (bytes) mbar_expect_tx(&full[stage], bytes);
          if (P.tmaA) tma_side<LA>(&P.tmA, P.batched_mapA, p, offA, i0, l0, sA, &full[stage]);
          if (P.tmaB) tma_side<LB>(&P.tmB, P.batched_mapB, p, offB, j0, l0, sB, &full[stage]);
        }
        if constexpr (LA == L_MNC || LA == L_PMX)
          if (P.bulkA) bulk_side<LA>(P.a, p, i0, mvalid, l0, kvalid, sA, lane, &full[stage]);
        if constexpr (LB == L_MNC || LB == L_PMX)
          if (P.bulkB) bulk_side<LB>(P.b, p, j0, nvalid, l0, kvalid, sB, lane, &full[stage]);
        const bool elemA = !P.tmaA && !P.bulkA, elemB = !P.tmaB && !P.bulkB;
        if (elemA || elemB) {
          fence_proxy_async();
          if (elemA) elem_side<LA>(P.a, p, i0, mvalid, l0, kvalid, sA, lane);
          if (elemB) elem_side<LB>(P.b, p, j0, nvalid, l0, kvalid, sB, lane);
          mbar_arrive_cpasync(&full[stage]);
        } else {
          mbar_arrive(&full[stage]);  // (release: covers the zero-fill stores of bulk sides)
        }
        if (++stage == P.nstages) { stage = 0; phase ^= 1; }
      }
    }
    cp_async_wait_all();
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = lane >> 2, t = lane & 3;
  // warps w and w + 4 share a scheduler partition: with ragged tiles the second
  // half takes its row blocks rotated by two, so the live warps of an edge tile
  // (few valid rows) fall on different partitions, and the warps a diagonal
  // syrk tile skips (0, 1 lower / 4, 5 upper) sit on the producer warp's
  const int jb = (EDGE ? 1 - warp / NWR : warp / NWR) * 8 * WF;
  const int ib = ((warp + (EDGE ? 2 : 0) * (warp / NWR)) % NWR) * 8 * WH;
  const bool use_c = P.beta != 0.0;
  // fragment (f, h) of an interior tile sits at a fixed element offset from the
  // lane's first pair: f * sf + h * sh (no per-element bounds or index math)
  const long long sfc = OUT_PM ? 32 : 8LL * P.o.ldc, shc = OUT_PM ? 8LL * P.o.ldc : 8;
  const long long sfd = OUT_PM ? 32 : 8LL * P.o.ldd, shd = OUT_PM ? 8LL * P.o.ldd : 8;
  // a tile moved as 16-byte pairs from one base pointer: aligned storage, an even
  // m (a pair is inside or outside as a whole) and no uplo diagonal through it.
  // Full-tile launches (EDGE = 0) move every pair; ragged ones predicate each
  // pair on its row and column — no per-element masks or index arithmetic.
  auto interior = [&](int tm, int tn) {
    if (!(P.o.vec && (P.uplo == 0 || (P.uplo == 1 ? tm > tn : tm < tn)))) return false;
    if (EDGE) return (P.m & 1) == 0;
    return (tm + 1) * TM <= P.m && (tn + 1) * TN <= P.n;
  };
  // beta*C operands for this lane's 4x2 fragments, prefetched one item ahead
  // so their DRAM latency hides behind a whole item of tensor-core work.
  double cv[WF][WH][2], cn[WF][WH][2];
  auto load_c = [&](int p, int tm, int tn, double (&dst)[WF][WH][2]) {
    const double* cbase =
        P.o.c + (P.o.offs_c ? P.o.offs_c[p] : P.o.offs ? P.o.offs[p] : (long long)p * P.o.sc);
    const bool live = !(P.skip && P.skip[p]);
    if (live && interior(tm, tn)) {
      const int ir = tm * TM + ib + 2 * t, jr = tn * TN + jb + g;
      const double* cp0 = cbase + out_off<OUT_PM>(P.o.ldc, ir, jr);
#pragma unroll
      for (int f = 0; f < WF; ++f)
#pragma unroll
        for (int h = 0; h < WH; ++h) {
          double2 v = make_double2(0.0, 0.0);
          if (!EDGE || (ir + 8 * h < P.m && jr + 8 * f < P.n)) v = *reinterpret_cast<const double2*>(cp0 + f * sfc + h * shc);
          dst[f][h][0] = v.x;
          dst[f][h][1] = v.y;
        }
      return;
    }
#pragma unroll
    for (int f = 0; f < WF; ++f)
#pragma unroll
      for (int h = 0; h < WH; ++h) {
        const int i = tm * TM + ib + h * 8 + 2 * t, j = tn * TN + jb + f * 8 + g;
        dst[f][h][0] = dst[f][h][1] = 0.0;
        if (j < P.n && live) {
          const double* cp = cbase + out_off<OUT_PM>(P.o.ldc, i, j);
          if (P.o.vec && i + 1 < P.m) {
            double2 v = *reinterpret_cast<const double2*>(cp);
            dst[f][h][0] = v.x;
            dst[f][h][1] = v.y;
          } else {
            if (i < P.m) dst[f][h][0] = cp[0];
            if (i + 1 < P.m) dst[f][h][1] = cbase[out_off<OUT_PM>(P.o.ldc, i + 1, j)];
          }
        }
      }
  };
  // The two consumer warps of a scheduler partition (warp w and w + 4) would
  // otherwise walk the stages in lockstep and reach their epilogues together,
  // leaving the partition's FP64 tensor pipe idle for the whole epilogue.  The
  // second warp starts late once; the offset then persists (while one warp is
  // in its epilogue the other has the pipe alone), so one warp's epilogue runs
  // under the other's DMMAs.
  if (P.stagger && warp >= NCW / 2) {
    const long long t0 = clock64();
    while (clock64() - t0 < P.stagger) {}
  }
  ItemCursor cur;
  cur.init(P);
  int tm = 0, tn = 0, tmn = 0, tnn = 0;
  if (cur.item < P.items) {
    tile_of(P, cur.r, tmn, tnn);
    if (use_c) load_c(cur.p, tmn, tnn, cn);
  }
  int stage = 0;
  uint32_t phase = 0;
  while (cur.item < P.items) {
    const int p = cur.p;
    tm = tmn;
    tn = tnn;
    cur.next();
    const bool more = cur.item < P.items;
    if (more) tile_of(P, cur.r, tmn, tnn);
    if (use_c) {
#pragma unroll
      for (int f = 0; f < WF; ++f)
#pragma unroll
        for (int h = 0; h < WH; ++h) { cv[f][h][0] = cn[f][h][0]; cv[f][h][1] = cn[f][h][1]; }
      if (more) load_c(cur.p, tmn, tnn, cn);
    }
    if (P.skip && P.skip[p]) continue;
    const int i0 = tm * TM, j0 = tn * TN;
    double* dbase = P.o.d + (P.o.offs ? P.o.offs[p] : (long long)p * P.o.sd);

    double acc[WF][WH][2];
#pragma unroll
    for (int f = 0; f < WF; ++f)
#pragma unroll
      for (int h = 0; h < WH; ++h) acc[f][h][0] = acc[f][h][1] = 0.0;

#define PB_KL(F, H) \
  engine_k_loop<F, H, TA, TB>(P, smem, full, empty, STAGE, stage, phase, ib, jb, g, t, lane, acc)
    if constexpr (!EDGE) {
      PB_KL(WF, WH);
    } else {
      // live fragments of this warp's tile: those with an element inside m x n;
      // on a diagonal syrk tile a warp wholly in the opposite triangle has none
      static_assert(WH == 2 && WF == 4, "the live-fragment dispatch is written for 4 x 2 fragments");
      int ha = min(WH, max(0, (P.m - i0 - ib + 7) >> 3)), fa = min(WF, max(0, (P.n - j0 - jb + 7) >> 3));
      if (P.uplo && tm == tn && (P.uplo == 1 ? ib + 8 * WH - 1 < jb : jb + 8 * WF - 1 < ib)) fa = 0;
      if (ha == 0) fa = 0;
      // (three live column fragments run as four: seven variants instead of nine —
      // different warps run different variants at once and the kernel is sensitive
      // to its code size; a single fragment, the thin edge tile, keeps its own)
      if (fa > 2 && ha == WH) PB_KL(4, 2);
      else if (fa == 0) PB_KL(0, 0);
      else if (ha == 2) { if (fa == 2) PB_KL(2, 2); else PB_KL(1, 2); }
      else if (fa > 2) PB_KL(4, 1);
      else if (fa == 2) PB_KL(2, 1);
      else PB_KL(1, 1);
    }
#undef PB_KL

    // Epilogue: d = alpha*acc + beta*c, masked to the problem and the uplo triangle.
    if (interior(tm, tn)) {
      const int ir = i0 + ib + 2 * t, jr = j0 + jb + g;
      double* dp0 = dbase + out_off<OUT_PM>(P.o.ldd, ir, jr);
#pragma unroll
      for (int f = 0; f < WF; ++f)
#pragma unroll
        for (int h = 0; h < WH; ++h) {
          const double r0 = use_c ? fma(P.alpha, acc[f][h][0], P.beta * cv[f][h][0]) : acc[f][h][0] * P.alpha;
          const double r1 = use_c ? fma(P.alpha, acc[f][h][1], P.beta * cv[f][h][1]) : acc[f][h][1] * P.alpha;
          if (!EDGE || (ir + 8 * h < P.m && jr + 8 * f < P.n))
            *reinterpret_cast<double2*>(dp0 + f * sfd + h * shd) = make_double2(r0, r1);
        }
      continue;
    }
#pragma unroll
    for (int f = 0; f < WF; ++f)
#pragma unroll
      for (int h = 0; h < WH; ++h) {
        const int i = i0 + ib + h * 8 + 2 * t, j = j0 + jb + f * 8 + g;
        if (j >= P.n) continue;
        double r0 = use_c ? fma(P.alpha, acc[f][h][0], P.beta * cv[f][h][0]) : acc[f][h][0] * P.alpha;
        double r1 = use_c ? fma(P.alpha, acc[f][h][1], P.beta * cv[f][h][1]) : acc[f][h][1] * P.alpha;
        bool w0 = i < P.m, w1 = i + 1 < P.m;
        if (P.uplo == 1) { w0 &= i >= j; w1 &= i + 1 >= j; }
        if (P.uplo == 2) { w0 &= i <= j; w1 &= i + 1 <= j; }
        double* dp = dbase + out_off<OUT_PM>(P.o.ldd, i, j);
        if (w0 && w1 && P.o.vec) {
          *reinterpret_cast<double2*>(dp) = make_double2(r0, r1);
        } else {
          if (w0) dp[0] = r0;
          if (w1) dbase[out_off<OUT_PM>(P.o.ldd, i + 1, j)] = r1;
        }
      }
  }
}

template <int OUT_PM>
__global__ void scale_kernel(OutDesc o, int m, int n, double beta, int uplo, long long total) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long per = (long long)m * n;
    int p = (int)(e / per);
    int r = (int)(e - p * per);
    int i = r % m, j = r / m;
    if (uplo == 1 && i < j) continue;
    if (uplo == 2 && i > j) continue;
    double v = 0.0 * 0.0;  // scale_ab(alpha = 0): 0*0 (+ beta*c) — micro_kernel.hpp:263-273
    const long long oc = o.offs_c ? o.offs_c[p] : o.offs ? o.offs[p] : (long long)p * o.sc;
    const long long od = o.offs ? o.offs[p] : (long long)p * o.sd;
    if (beta != 0.0) v = __dadd_rn(v, __dmul_rn(beta, o.c[oc + out_off<OUT_PM>(o.ldc, i, j)]));
    o.d[od + out_off<OUT_PM>(o.ldd, i, j)] = v;
  }
}


// ------------------------------------------------------------------ tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// Builds the TMA map of one operand side; returns false when the operand's
// alignment rules it out (the kernel then uses the cp.async fallback).
static bool make_map(CUtensorMap* tm, int lay, const OpDesc& d, int xdim, int k, int batch,
                     int* batched) {
  auto enc = encode_fn();
  if (!enc || !d.base) return false;
  if ((reinterpret_cast<uintptr_t>(d.base) & 15) != 0) return false;
  if (((long long)d.ld * 8) % 16 != 0) return false;
  const bool bdim = !d.offs && batch > 1 && d.stride != 0;
  if (bdim && (d.stride * 8) % 16 != 0) return false;
  if (xdim <= 0 || k <= 0) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  int rank = 0;
  switch (lay) {
    case L_MNC:  // (x, l, p)
      dims[0] = xdim; dims[1] = k; strides[0] = (cuuint64_t)d.ld * 8;
      box[0] = LayT<L_MNC>::S; box[1] = BK;
      rank = 2;
      break;
    case L_KC:  // (l, x, p)
      dims[0] = k; dims[1] = xdim; strides[0] = (cuuint64_t)d.ld * 8;
      box[0] = LayT<L_KC>::S; box[1] = TM;
      rank = 2;
      break;
    case L_PMX:  // (x%4, l, x/4, p)
      dims[0] = 4; dims[1] = k; dims[2] = (xdim + 3) / 4;
      strides[0] = 32; strides[1] = (cuuint64_t)d.ld * 32;
      box[0] = 4; box[1] = BK; box[2] = TM / 4;
      rank = 3;
      break;
    default:  // L_PML: (l%4, x, l/4, p)
      dims[0] = 4; dims[1] = xdim; dims[2] = (k + 3) / 4;
      strides[0] = 32; strides[1] = (cuuint64_t)d.ld * 32;
      box[0] = 4; box[1] = TM; box[2] = BK / 4;
      rank = 3;
      break;
  }
  if (bdim) {
    dims[rank] = batch;
    strides[rank - 1] = (cuuint64_t)d.stride * 8;
    box[rank] = 1;
    ++rank;
  } else if (d.offs) {
    // per-problem offsets (even, caller-checked through `bulk`): offset / 2 =
    // lo + 2^20 hi as the coordinates of a 16-byte and a 16-MiB stride dimension
    dims[rank] = 1u << 20;
    strides[rank - 1] = 16;
    box[rank] = 1;
    ++rank;
    dims[rank] = 1u << 30;
    strides[rank - 1] = 16ull << 20;
    box[rank] = 1;
    ++rank;
  }
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(d.base), dims,
                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  *batched = d.offs ? 2 : bdim ? 1 : 0;
  return r == CUDA_SUCCESS;
}

template <int LA, int LB, int OUT_PM, int EDGE>
static cudaError_t launch_e(KParams& P, cudaStream_t s) {
  constexpr int STAGE = LayT<LA>::SIZE + LayT<LB>::SIZE;
  const size_t stage_bytes = (size_t)STAGE * 8;
  const size_t budget = 227 * 1024 - 256;
  int nst = (int)((budget - 16 * 16) / (stage_bytes + 16));
  nst = std::min(nst, 8);
  P.nstages = nst;
  size_t smem = (size_t)nst * stage_bytes + (size_t)nst * 16;
  auto kern = gemm_tiles_kernel<LA, LB, OUT_PM, EDGE>;
  {
    cudaError_t e = smem_attr((const void*)kern, (int)smem);
    if (e != cudaSuccess) return e;
  }
  long long grid = std::min<long long>(P.items, (long long)num_sms());
  if (P.items < 8 * grid) P.stagger = 0;
  kern<<<(int)grid, NTHREADS, smem, s>>>(P);
  return cudaGetLastError();
}

template <int LA, int LB, int OUT_PM>
static cudaError_t launch_t(KParams& P, cudaStream_t s) {
  const bool ragged = (P.m % TM) != 0 || (P.n % TN) != 0 || P.uplo != 0;
  return ragged ? launch_e<LA, LB, OUT_PM, 1>(P, s) : launch_e<LA, LB, OUT_PM, 0>(P, s);
}

cudaError_t gemm_launch(const GemmLaunch& g, cudaStream_t s) {
  if (g.batch <= 0 || g.m <= 0 || g.n <= 0) return cudaSuccess;
  KParams P;
  memset(&P, 0, sizeof(P));
  P.a = g.a;
  P.b = g.b;
  P.o = g.o;
  P.m = g.m;
  P.n = g.n;
  P.k = g.k;
  P.alpha = g.alpha;
  P.beta = g.beta;
  P.uplo = g.uplo;
  P.skip = g.skip;
  {
    // consumer offset in cycles (PBGPU_ENGINE_STAGGER overrides; 0 = lockstep);
    // measured +1 % at s >= 128, only worth its start-up delay on long item lists
    static const int stagger = [] {
      const char* e = getenv("PBGPU_ENGINE_STAGGER");
      return e ? atoi(e) : 6000;
    }();
    P.stagger = stagger;
  }
  P.tiles_m = (g.m + TM - 1) / TM;
  P.tiles_n = (g.n + TN - 1) / TN;
  if (g.uplo) {
    int t = P.tiles_m;  // square (syrk)
    P.tiles_per_problem = t * (t + 1) / 2;
  } else {
    P.tiles_per_problem = P.tiles_m * P.tiles_n;
  }
  P.nk = (g.k + BK - 1) / BK;
  P.items = (long long)g.batch * P.tiles_per_problem;
  P.nstages = 2;
  static const bool no_tma = [] {
    const char* e = getenv("PBGPU_NO_TMA");
    return e && e[0] == '1';
  }();
  // per-problem offsets ride on two extra tensor-map dimensions (make_map); should the
  // encode fail, those sides stream by column / panel bulk copies (bulk = every problem
  // base 16-byte aligned, caller-checked).  PBGPU_OFFS_TMA=0 forces the bulk copies.
  static const bool offs_tma = [] {
    const char* e = getenv("PBGPU_OFFS_TMA");
    return !(e && e[0] == '0');
  }();
  if (!no_tma && g.a.bulk && (!g.a.offs || offs_tma))
    P.tmaA = make_map(&P.tmA, g.lay_a, g.a, g.m, g.k, g.batch, &P.batched_mapA);
  if (!no_tma && g.b.bulk && (!g.b.offs || offs_tma))
    P.tmaB = make_map(&P.tmB, g.lay_b, g.b, g.n, g.k, g.batch, &P.batched_mapB);
  auto bulk_ok = [](int lay, const OpDesc& d, int x) {
    if (!d.offs || !d.bulk) return false;
    if (lay == L_PMX) return true;
    return lay == L_MNC && d.ld % 2 == 0 && x % 2 == 0;
  };
  P.bulkA = !P.tmaA && bulk_ok(g.lay_a, g.a, g.m);
  P.bulkB = !P.tmaB && bulk_ok(g.lay_b, g.b, g.n);
  if ((P.bulkA && !P.tmaB && !P.bulkB) || (P.bulkB && !P.tmaA && !P.bulkA)) P.bulkA = P.bulkB = 0;
  if (!g.out_pm) {
    if (g.lay_a == L_MNC && g.lay_b == L_MNC) return launch_t<L_MNC, L_MNC, 0>(P, s);
    if (g.lay_a == L_MNC && g.lay_b == L_KC) return launch_t<L_MNC, L_KC, 0>(P, s);
    if (g.lay_a == L_KC && g.lay_b == L_MNC) return launch_t<L_KC, L_MNC, 0>(P, s);
    if (g.lay_a == L_KC && g.lay_b == L_KC) return launch_t<L_KC, L_KC, 0>(P, s);
  } else {
    if (g.lay_a == L_PMX && g.lay_b == L_PMX) return launch_t<L_PMX, L_PMX, 1>(P, s);
    if (g.lay_a == L_PMX && g.lay_b == L_PML) return launch_t<L_PMX, L_PML, 1>(P, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t scale_launch(int out_pm, const OutDesc& o, int m, int n, double beta, int uplo,
                         int batch, cudaStream_t s) {
  long long total = (long long)m * n * batch;
  if (total <= 0) return cudaSuccess;
  int threads = 256;
  long long blocks = std::min<long long>((total + threads - 1) / threads, (long long)num_sms() * 16);
  if (out_pm)
    scale_kernel<1><<<(int)blocks, threads, 0, s>>>(o, m, n, beta, uplo, total);
  else
    scale_kernel<0><<<(int)blocks, threads, 0, s>>>(o, m, n, beta, uplo, total);
  return cudaGetLastError();
}

}  // namespace pbg
