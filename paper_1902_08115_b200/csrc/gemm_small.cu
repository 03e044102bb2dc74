// Small-size branch of the batched panel-major gemm_nd (level3.hpp:360-403),
// D = alpha * A * B^T + beta * C with m = n = k = s <= 32, s % 4 == 0, ps = 4,
// problems packed back to back (stride = s*s, pm = cn = s).
//
// The paper's size switch (gemm.hpp:190-204) picks a different algorithm for
// tiny operands; on the GPU the 64x64-tile engine would waste most of every
// tile and every TMA box at these sizes.  Here a persistent CTA streams
// CHUNKS of G consecutive problems: A, B and C of a chunk are each one
// contiguous TMA bulk copy into a double-buffered shared-memory ring, every
// warp computes whole problems with FP64 tensor-core DMMA m8n8k4 straight
// from the panel-major layout (fragment loads are conflict-free because a
// 4-row panel column is 32 contiguous bytes), D overwrites C in shared memory
// and leaves as one bulk store per chunk.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "launch.h"

namespace pbg {

struct SmallArgs {
  const double *a, *b, *c;
  double* d;
  double alpha, beta;
  long long batch;
  int s, G, nchunks;
};

constexpr int SM_WARPS = 4;

template <int T>  // T = ceil(s / 8) row/column tiles per problem
__global__ void __launch_bounds__(32 * SM_WARPS) gemm_small_kernel(const __grid_constant__ SmallArgs P) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int s = P.s, ss = s * s, G = P.G;
  const bool use_c = P.beta != 0.0;
  double* buf[2] = {sm, sm + 3 * (size_t)G * ss};
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int chunk, int slot) {
    const long long p0 = (long long)chunk * G;
    const int np = (int)(P.batch - p0 < G ? P.batch - p0 : G);
    const uint32_t bytes = 8u * (uint32_t)np * ss;
    double* sA = buf[slot];
    mbar_arrive_expect_tx(&full[slot], use_c ? 3 * bytes : 2 * bytes);
    bulk_g2s(sA, P.a + p0 * ss, bytes, &full[slot]);
    bulk_g2s(sA + (size_t)G * ss, P.b + p0 * ss, bytes, &full[slot]);
    if (use_c) bulk_g2s(sA + 2 * (size_t)G * ss, P.c + p0 * ss, bytes, &full[slot]);
  };
  int it = 0;
  int chunk = blockIdx.x;
  if (tid == 0 && chunk < P.nchunks) issue(chunk, 0);
  for (; chunk < P.nchunks; chunk += gridDim.x, ++it) {
    const int slot = it & 1;
    const int next = chunk + gridDim.x;
    // the other slot's bulk store (previous chunk) must have drained before reuse
    if (tid == 0) {
      bulk_wait_read0();
      if (next < P.nchunks) issue(next, slot ^ 1);
    }
    mbar_wait(&full[slot], (it >> 1) & 1);
    const long long p0 = (long long)chunk * G;
    const int np = (int)(P.batch - p0 < G ? P.batch - p0 : G);
    const double* sA = buf[slot];
    const double* sB = sA + (size_t)G * ss;
    double* sC = buf[slot] + 2 * (size_t)G * ss;  // D is written here, over C
    for (int q = warp; q < np; q += SM_WARPS) {
      const double* A = sA + (size_t)q * ss;
      const double* B = sB + (size_t)q * ss;
      double* Cq = sC + (size_t)q * ss;
      double acc[T][T][2];
#pragma unroll
      for (int I = 0; I < T; ++I)
#pragma unroll
        for (int J = 0; J < T; ++J) acc[I][J][0] = acc[I][J][1] = 0.0;
      for (int l0 = 0; l0 < s; l0 += 4) {
        double fa[T], fb[T];
#pragma unroll
        for (int I = 0; I < T; ++I) {
          // row 8I+g, column l0+t of a panel-major s x s operand; rows past s
          // read the neighbour's data and only feed discarded outputs
          const int r = 8 * I + g;
          const long long off = (long long)(r >> 2) * 4 * s + (l0 + t) * 4 + (r & 3);
          fa[I] = A[off];
          fb[I] = B[off];
        }
#pragma unroll
        for (int I = 0; I < T; ++I)
#pragma unroll
          for (int J = 0; J < T; ++J) dmma(acc[I][J][0], acc[I][J][1], fa[I], fb[J]);
      }
      __syncwarp();
#pragma unroll
      for (int I = 0; I < T; ++I)
#pragma unroll
        for (int J = 0; J < T; ++J)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = 8 * I + g, c = 8 * J + 2 * t + e;
            if (r < s && c < s) {
              const long long off = (long long)(r >> 2) * 4 * s + c * 4 + (r & 3);
              const double v = use_c ? fma(P.alpha, acc[I][J][e], P.beta * Cq[off]) : P.alpha * acc[I][J][e];
              Cq[off] = v;
            }
          }
    }
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async();
      bulk_s2g(P.d + p0 * ss, smem_u32(sC), 8u * (uint32_t)np * ss);
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_read0();
}

// s = 4: a problem is one 4x4 panel (element (i, l) at l*4 + i), 128 bytes per
// operand; the problem is pure HBM traffic.  A warp owns 32 consecutive
// problems: each operand's 4 KB arrive as 8 fully coalesced 512-byte warp
// loads (all three operands in flight at once), are transposed through a
// per-warp shared buffer (element e of problem p at e*33 + p: conflict-free
// both ways) so that each lane holds its own problem, 64 FMAs in registers,
// and D leaves through the same buffer as coalesced 512-byte stores.
constexpr int kTinyWarps = 8;
__global__ void __launch_bounds__(32 * kTinyWarps) gemm_tiny4_kernel(const __grid_constant__ SmallArgs P) {
  __shared__ double tb[kTinyWarps][16 * 33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p0 = ((long long)blockIdx.x * kTinyWarps + warp) * 32;
  if (p0 >= P.batch) return;
  const int np = (int)min(32LL, P.batch - p0);  // problems of this warp
  const bool use_c = P.beta != 0.0;
  double* buf = tb[warp];
  // coalesced loads: iteration i, lane L -> doubles 64 i + 2 L (+1) of the warp's 512
  double2 va[8], vb[8], vc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int pp = 4 * i + (lane >> 3);
    const long long off = p0 * 16 + 64 * i + 2 * lane;
    const bool ok = pp < np;
    va[i] = ok ? __ldcs(reinterpret_cast<const double2*>(P.a + off)) : make_double2(0.0, 0.0);
    vb[i] = ok ? __ldcs(reinterpret_cast<const double2*>(P.b + off)) : make_double2(0.0, 0.0);
    vc[i] = ok && use_c ? __ldcs(reinterpret_cast<const double2*>(P.c + off)) : make_double2(0.0, 0.0);
  }
  auto transpose_in = [&](const double2 (&v)[8], double (&x)[16]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int pp = 4 * i + (lane >> 3), e = 2 * (lane & 7);
      buf[e * 33 + pp] = v[i].x;
      buf[(e + 1) * 33 + pp] = v[i].y;
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < 16; ++e) x[e] = buf[e * 33 + lane];
    __syncwarp();
  };
  double a[16], b[16], c[16];
  transpose_in(va, a);
  transpose_in(vb, b);
  if (use_c) transpose_in(vc, c);
#pragma unroll
  for (int j = 0; j < 4; ++j)      // column j of D = row j of B
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // D(i, j) = sum_l A(i, l) B(j, l)
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < 4; ++l) acc = fma(a[l * 4 + i], b[l * 4 + j], acc);
      buf[(j * 4 + i) * 33 + lane] = use_c ? fma(P.alpha, acc, P.beta * c[j * 4 + i]) : P.alpha * acc;
    }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int pp = 4 * i + (lane >> 3), e = 2 * (lane & 7);
    if (pp < np)
      __stcs(reinterpret_cast<double2*>(P.d + p0 * 16 + 64 * i + 2 * lane),
             make_double2(buf[e * 33 + pp], buf[(e + 1) * 33 + pp]));
  }
}

// 28 <= s <= 108 (T = 4..14 tiles per side): one problem per CTA iteration,
// the problem split across warps by row tile (warp I computes the T output
// tiles of row tile I, so every A fragment feeds T independent DMMAs).  A and
// B arrive as one bulk copy each; up to s = 64 C is staged too and D leaves as
// one bulk store (two stages), above that C / D go straight to global memory
// and the stage count follows shared memory (2 stages up to s = 80, then 1).
// The engine's 64-wide tiles would waste up to 44 % (s = 48) and 64 % (s = 68)
// of every tile at these orders.
template <int T, bool SC, int NST, int SPL>
__global__ void __launch_bounds__(32 * T * SPL) gemm_mid_kernel(const __grid_constant__ SmallArgs P) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[2];
  constexpr int NOP = SC ? 3 : 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int s = P.s, ss = s * s;
  const bool use_c = P.beta != 0.0;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto bufp = [&](int slot) { return sm + (size_t)slot * NOP * ss; };
  auto issue = [&](long long prob, int slot) {
    const uint32_t bytes = 8u * (uint32_t)ss;
    double* sA = bufp(slot);
    const bool lc = SC && use_c;
    mbar_arrive_expect_tx(&full[slot], lc ? 3 * bytes : 2 * bytes);
    bulk_g2s(sA, P.a + prob * ss, bytes, &full[slot]);
    bulk_g2s(sA + ss, P.b + prob * ss, bytes, &full[slot]);
    if (lc) bulk_g2s(sA + 2 * ss, P.c + prob * ss, bytes, &full[slot]);
  };
  int it = 0;
  long long prob = blockIdx.x;
  if (tid == 0 && prob < P.batch) issue(prob, 0);
  for (; prob < P.batch; prob += gridDim.x, ++it) {
    const int slot = NST == 2 ? (it & 1) : 0;
    const uint32_t par = NST == 2 ? ((it >> 1) & 1) : (it & 1);
    const long long next = prob + gridDim.x;
    if (NST == 2 && tid == 0) {
      if (SC) bulk_wait_read0();  // the other slot's store (previous problem) has left shared memory
      if (next < P.batch) issue(next, slot ^ 1);
    }
    mbar_wait(&full[slot], par);
    const double* A = bufp(slot);
    const double* B = A + ss;
    double* Cq = bufp(slot) + 2 * ss;
    // SPL warps per row tile, each owning TJ column tiles starting at J0
    constexpr int TJ = (T + SPL - 1) / SPL;
    const int I = warp % T, J0 = (warp / T) * TJ, nj = min(TJ, T - J0);
    const double* Cg = P.c + prob * ss;
    double* Dg = P.d + prob * ss;
    double cpre[SC ? 1 : TJ][2];  // unstaged C: loaded before the k loop so its latency hides under it
    if constexpr (!SC) {
#pragma unroll
      for (int J = 0; J < TJ; ++J)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 8 * I + g, c = 8 * (J0 + J) + 2 * t + e;
          const long long off = (long long)(r >> 2) * 4 * s + c * 4 + (r & 3);
          cpre[J][e] = ldg_if(Cg + off, J < nj && use_c && r < s && c < s, 0.0);
        }
    }
    double acc[TJ][2];
#pragma unroll
    for (int J = 0; J < TJ; ++J) acc[J][0] = acc[J][1] = 0.0;
    const int ra = 8 * I + g;
    for (int l0 = 0; l0 < s; l0 += 4) {
      // rows past s read neighbouring data and only feed discarded outputs
      const double fa = A[(long long)(ra >> 2) * 4 * s + (l0 + t) * 4 + (ra & 3)];
      double fb[TJ];
#pragma unroll
      for (int J = 0; J < TJ; ++J) {
        const int rb = 8 * (J0 + J) + g;
        fb[J] = J < nj ? B[(long long)(rb >> 2) * 4 * s + (l0 + t) * 4 + (rb & 3)] : 0.0;
      }
#pragma unroll
      for (int J = 0; J < TJ; ++J)
        if (J < nj) dmma(acc[J][0], acc[J][1], fa, fb[J]);
    }
    if (NST == 1) {
      __syncthreads();  // every warp is done with the operands: load the next problem under the epilogue
      if (tid == 0 && next < P.batch) issue(next, 0);
    } else {
      __syncwarp();
    }
#pragma unroll
    for (int J = 0; J < TJ; ++J)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * I + g, c = 8 * (J0 + J) + 2 * t + e;
        if (J < nj && r < s && c < s) {
          const long long off = (long long)(r >> 2) * 4 * s + c * 4 + (r & 3);
          if constexpr (SC) Cq[off] = use_c ? fma(P.alpha, acc[J][e], P.beta * Cq[off]) : P.alpha * acc[J][e];
          else Dg[off] = use_c ? fma(P.alpha, acc[J][e], P.beta * cpre[J][e]) : P.alpha * acc[J][e];
        }
      }
    if (SC) {
      fence_proxy_async();  // every writer orders its generic-proxy stores before the async-proxy store
      __syncthreads();
      if (tid == 0) {
        bulk_s2g(P.d + prob * ss, smem_u32(Cq), 8u * (uint32_t)ss);
        bulk_commit();
      }
    } else if (NST == 2) {
      __syncthreads();  // this slot is reused two problems later
    }
  }
  if (SC && tid == 0) bulk_wait_read0();
}

// 84 <= s <= 96 (T = 11, 12): one problem does not fit twice in shared memory,
// so the operands stream in two k halves (columns [0, k0) and [k0, s) of every
// panel, k0 = 4 floor(s / 8)) into two slots: while one half is multiplied the
// other half — and then the next problem's first half — is in flight.  One
// bulk copy per panel and operand (issued by one thread), C prefetched into
// registers when the problem starts, D straight from the accumulators.
template <int T>
__global__ void __launch_bounds__(32 * T, 1) gemm_midk_kernel(const __grid_constant__ SmallArgs P) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int s = P.s, k0 = 4 * (s / 8), kh[2] = {k0, s - k0}, kmax = max(kh[0], kh[1]);
  const long long ss = (long long)s * s;
  const bool use_c = P.beta != 0.0;
  const int np = s / 4;  // panels per operand
  auto slot = [&](int h) { return sm + (size_t)h * 2 * s * kmax; };
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](long long prob, int h) {  // tid 0: half h of problem prob into slot h
    const int kc = kh[h], c0 = h ? k0 : 0;
    const uint32_t bytes = 32u * (uint32_t)kc;  // one panel's 4 rows x kc columns
    mbar_arrive_expect_tx(&full[h], 2u * (uint32_t)np * bytes);
    for (int o = 0; o < 2; ++o) {
      const double* src = (o ? P.b : P.a) + prob * ss + 4 * c0;
      double* dst = slot(h) + (size_t)o * s * kmax;
      for (int q = 0; q < np; ++q) bulk_g2s(dst + (size_t)q * 4 * kc, src + (long long)q * 4 * s, bytes, &full[h]);
    }
  };
  long long prob = blockIdx.x;
  if (tid == 0 && prob < P.batch) {
    issue(prob, 0);
    issue(prob, 1);
  }
  const int I = warp, ra = 8 * I + g;
  for (int it = 0; prob < P.batch; prob += gridDim.x, ++it) {
    const long long next = prob + gridDim.x;
    const double* Cg = P.c + prob * ss;
    double* Dg = P.d + prob * ss;
    double cpre[T][2];  // C loaded before the k loop so its latency hides under it
#pragma unroll
    for (int J = 0; J < T; ++J)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * I + g, c = 8 * J + 2 * t + e;
        cpre[J][e] = ldg_if(Cg + (long long)(r >> 2) * 4 * s + c * 4 + (r & 3), use_c && r < s && c < s, 0.0);
      }
    double acc[T][2];
#pragma unroll
    for (int J = 0; J < T; ++J) acc[J][0] = acc[J][1] = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mbar_wait(&full[h], (uint32_t)(it & 1));
      const double* A = slot(h);
      const double* B = A + (size_t)s * kmax;
      const int kc = kh[h];
      // element (r, c) of a half: (r/4) * 4 kc + 4 c + r%4; rows past s read the
      // neighbouring data / slack and only feed discarded outputs
      for (int l0 = 0; l0 < kc; l0 += 4) {
        const double fa = A[(ra >> 2) * 4 * kc + (l0 + t) * 4 + (ra & 3)];
        double fb[T];
#pragma unroll
        for (int J = 0; J < T; ++J) {
          const int rb = 8 * J + g;
          fb[J] = B[(rb >> 2) * 4 * kc + (l0 + t) * 4 + (rb & 3)];
        }
#pragma unroll
        for (int J = 0; J < T; ++J) dmma(acc[J][0], acc[J][1], fa, fb[J]);
      }
      __syncthreads();  // every warp is done with slot h
      if (tid == 0 && next < P.batch) issue(next, h);
    }
#pragma unroll
    for (int J = 0; J < T; ++J)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * I + g, c = 8 * J + 2 * t + e;
        if (r < s && c < s)
          Dg[(long long)(r >> 2) * 4 * s + c * 4 + (r & 3)] =
              use_c ? fma(P.alpha, acc[J][e], P.beta * cpre[J][e]) : P.alpha * acc[J][e];
      }
  }
}

template <int T>
static cudaError_t midk_t(SmallArgs& P, cudaStream_t st) {
  const int s = P.s, k0 = 4 * (s / 8), kmax = std::max(k0, s - k0);
  // two slots of A and B halves + one panel chunk of slack for the last tile's rows past s
  const size_t smem = ((size_t)2 * 2 * s * kmax + 4 * (size_t)kmax) * sizeof(double);
  {
    cudaError_t e = smem_attr((const void*)gemm_midk_kernel<T>, 220 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int grid = (int)std::min<long long>(P.batch, (long long)num_sms());
  gemm_midk_kernel<T><<<grid, 32 * T, smem, st>>>(P);
  return cudaGetLastError();
}

// PBGPU_GEMM_MIDK=0: the single-stage row-tile kernel above s = 80 (A/B only)
static bool midk_on() {
  static const bool v = [] {
    const char* e = getenv("PBGPU_GEMM_MIDK");
    return !(e && e[0] == '0');
  }();
  return v;
}

template <int T, bool SC, int NST, int SPL = (T <= 8 ? 2 : 1)>
static cudaError_t mid_t(SmallArgs& P, cudaStream_t st) {
  // + one 4-row panel of slack: the last tile's rows past s read (and discard) past the last operand
  const size_t smem = ((size_t)NST * (SC ? 3 : 2) * P.s * P.s + 4 * (size_t)P.s) * sizeof(double);
  {
    cudaError_t e = smem_attr((const void*)gemm_mid_kernel<T, SC, NST, SPL>, 220 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int per_sm = std::max(1, (int)((225 * 1024) / (smem + 1024)));
  const int grid = (int)std::min<long long>(P.batch, (long long)per_sm * num_sms());
  gemm_mid_kernel<T, SC, NST, SPL><<<grid, 32 * T * SPL, smem, st>>>(P);
  return cudaGetLastError();
}

static cudaError_t mid_launch(SmallArgs& P, cudaStream_t st) {
  const int s = P.s;
  if (s <= 64) {
    switch ((s + 7) / 8) {
      case 4: return mid_t<4, true, 2>(P, st);
      case 5: return mid_t<5, true, 2>(P, st);
      case 6: return mid_t<6, true, 2>(P, st);
      case 7: return mid_t<7, true, 2>(P, st);
      case 8: return mid_t<8, true, 2>(P, st);
    }
  } else if (s <= 80) {
    switch ((s + 7) / 8) {
      case 9: return mid_t<9, false, 2>(P, st);
      case 10: return mid_t<10, false, 2>(P, st);
    }
  } else if (midk_on() && s <= 96) {
    // (13-14 warps are capped at 128 registers and spill the C prefetch: measured
    // 0.76-0.93x there, so s = 100..112 stay on the single-stage kernel)
    switch ((s + 7) / 8) {
      case 11: return midk_t<11>(P, st);
      case 12: return midk_t<12>(P, st);
    }
  } else {
    switch ((s + 7) / 8) {
      case 11: return mid_t<11, false, 1>(P, st);
      case 12: return mid_t<12, false, 1>(P, st);
      case 13: return mid_t<13, false, 1>(P, st);
      case 14: return mid_t<14, false, 1, 2>(P, st);  // two warps per row tile: measured +6-8 % (T = 13: -4 %)
    }
  }
  return cudaErrorInvalidValue;
}

template <int T>
static cudaError_t small_t(SmallArgs& P, cudaStream_t st) {
  const size_t smem = 2 * 3 * (size_t)P.G * P.s * P.s * sizeof(double);
  {
    cudaError_t e = smem_attr((const void*)gemm_small_kernel<T>, 110 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int grid = (int)std::min<long long>(P.nchunks, 2LL * num_sms());
  gemm_small_kernel<T><<<grid, 32 * SM_WARPS, smem, st>>>(P);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Column-major NN, square packed problems (m = n = k = lda = ldb = ldc = s <= 64,
// stride s*s): config 1's shape.  One problem per CTA iteration on a 2-stage
// ring (one CTA per SM: 2 x 104 KB at s = 64); A, B and C arrive as ONE 2-D
// TMA tensor copy each whose box is 4 rows taller than the problem (the rows
// past s are the out-of-bounds zero fill), which gives the column stride
// s + 4 = 4 mod 16 doubles: conflict-free fragment loads for both operands.
// D is formed over C in shared memory and leaves as one tensor store.
#ifndef CM_PAD
#define CM_PAD 4  // box rows past s (out-of-bounds zero fill): column stride s + 4 = 4 mod 16
#endif
struct CmArgs {
  CUtensorMap ta, tb, tc, td;
  double alpha, beta;
  long long batch;
  int s;
};

// Warp blocks: warp w owns RI x RJ tiles of 8x8 (row tiles I0..I0+RI-1, column
// tiles J0..J0+RJ-1) — RI + RJ fragment loads feed RI * RJ independent DMMA
// chains per k step, and the next step's fragments are loaded under the
// current step's DMMAs (register double buffer).
template <int T> struct CmShape;
template <> struct CmShape<4> { static constexpr int RI = 1, RJ = 2; };
template <> struct CmShape<5> { static constexpr int RI = 1, RJ = 5; };
template <> struct CmShape<6> { static constexpr int RI = 1, RJ = 3; };
template <> struct CmShape<7> { static constexpr int RI = 1, RJ = 7; };
template <> struct CmShape<8> { static constexpr int RI = 2, RJ = 4; };
template <int T> __host__ __device__ constexpr int cm_warps() { return (T / CmShape<T>::RI) * (T / CmShape<T>::RJ); }

template <int T>
__global__ void __launch_bounds__(32 * cm_warps<T>()) gemm_cm_kernel(const __grid_constant__ CmArgs P) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ __align__(8) uint64_t full[2];
  constexpr int RI = CmShape<T>::RI, RJ = CmShape<T>::RJ, NWR = T / RI;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int s = P.s, S = s + CM_PAD, ops = S * s;  // doubles per staged operand
  const bool use_c = P.beta != 0.0;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t base = smem_u32(sm);
  auto slot_addr = [&](int slot) { return base + 8u * (uint32_t)(slot * 3 * ops); };
  auto tma3 = [&](uint32_t dst, const CUtensorMap* m, int prob, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(0), "r"(0), "r"(prob), "r"(smem_u32(bar))
        : "memory");
  };
  auto issue = [&](long long prob, int slot) {
    const uint32_t bytes = 8u * (uint32_t)ops;
    const uint32_t a = slot_addr(slot);
    mbar_arrive_expect_tx(&full[slot], use_c ? 3 * bytes : 2 * bytes);
    tma3(a, &P.ta, (int)prob, &full[slot]);
    tma3(a + 8u * ops, &P.tb, (int)prob, &full[slot]);
    if (use_c) tma3(a + 16u * ops, &P.tc, (int)prob, &full[slot]);
  };
  const int I0 = (warp % NWR) * RI, J0 = (warp / NWR) * RJ;
  int it = 0;
  long long prob = blockIdx.x;
  if (tid == 0 && prob < P.batch) issue(prob, 0);
  for (; prob < P.batch; prob += gridDim.x, ++it) {
    const int slot = it & 1;
    const long long next = prob + gridDim.x;
    if (tid == 0) {
      bulk_wait_read0();  // the other slot's store (previous problem) has left shared memory
      if (next < P.batch) issue(next, slot ^ 1);
    }
    mbar_wait(&full[slot], (it >> 1) & 1);
    const uint32_t A = slot_addr(slot), B = A + 8u * ops, C = B + 8u * ops;
    // A(8I+g, l+t) at column l+t, row 8I+g; B(l+t, 8J+g) at column 8J+g, row l+t
    const uint32_t fa0 = A + 8u * (t * S + 8 * I0 + g), fb0 = B + 8u * ((8 * J0 + g) * S + t);
    double acc[RI][RJ][2];
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
      for (int j = 0; j < RJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double a0[RI], b0[RJ], a1[RI], b1[RJ];
    auto load = [&](int l0, double (&fa)[RI], double (&fb)[RJ]) {
#pragma unroll
      for (int i = 0; i < RI; ++i) fa[i] = lds64(fa0 + 8u * (l0 * S + 8 * i));
#pragma unroll
      for (int j = 0; j < RJ; ++j) fb[j] = lds64(fb0 + 8u * (l0 + 8 * S * j));
    };
    auto mma = [&](const double (&fa)[RI], const double (&fb)[RJ]) {
#pragma unroll
      for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < RJ; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    };
    // s % 8 == 0: every tile is inside the problem, s / 4 k steps (even)
    load(0, a0, b0);
    int l0 = 0;
    for (; l0 + 8 <= s; l0 += 8) {
      load(l0 + 4, a1, b1);
      mma(a0, b0);
      if (l0 + 8 < s) load(l0 + 8, a0, b0);
      mma(a1, b1);
    }
    if (l0 < s) mma(a0, b0);  // (s % 8 == 4: not reached on this path)
    __syncwarp();
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
      for (int j = 0; j < RJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 8 * (I0 + i) + g, c = 8 * (J0 + j) + 2 * t + e;
          const uint32_t off = C + 8u * (c * S + r);
          sts64(off, use_c ? fma(P.alpha, acc[i][j][e], P.beta * lds64(off)) : P.alpha * acc[i][j][e]);
        }
    fence_proxy_async();  // every writer fences before the barrier that precedes the async-proxy store
    __syncthreads();
    if (tid == 0) {
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                       reinterpret_cast<uint64_t>(&P.td)),
                   "r"(0), "r"(0), "r"((int)prob), "r"(C)
                   : "memory");
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_read0();
}

static PFN_cuTensorMapEncodeTiled_v12000 small_encode_fn() {
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

bool gemm_cm_ok(int s, const double* a, const double* b, const double* c, long long sa, long long sb,
                long long sc, int lda, int ldb, int ldc) {
  static const bool off = [] {
    const char* e = getenv("PBGPU_GEMM_CM");
    return e && e[0] == '0';
  }();
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const long long ss = (long long)s * s;
  return !off && s >= 32 && s <= 64 && s % 8 == 0 && lda == s && ldb == s && ldc == s && sa == ss && sb == ss &&
         sc == ss && al(a) && al(b) && al(c) && small_encode_fn() != nullptr;
}

cudaError_t gemm_cm_launch(int s, double alpha, const double* a, const double* b, double beta, double* c,
                           long long batch, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  CmArgs P;
  memset(&P, 0, sizeof(P));
  P.alpha = alpha; P.beta = beta; P.batch = batch; P.s = s;
  auto enc = small_encode_fn();
  cuuint64_t dims[3] = {(cuuint64_t)s, (cuuint64_t)s, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)s * 8, (cuuint64_t)s * s * 8};
  cuuint32_t box[3] = {(cuuint32_t)(s + CM_PAD), (cuuint32_t)s, 1u};
  cuuint32_t es[3] = {1, 1, 1};
  const double* ptrs[4] = {a, b, c, c};
  CUtensorMap* maps[4] = {&P.ta, &P.tb, &P.tc, &P.td};
  for (int i = 0; i < 4; ++i)
    if (enc(maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptrs[i]), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  const size_t smem = (size_t)2 * 3 * (s + CM_PAD) * s * sizeof(double);
  const int per_sm = std::max(1, (int)((225 * 1024) / (smem + 1024)));
  const int grid = (int)std::min<long long>(batch, (long long)per_sm * num_sms());
#define PB_CM(TV)                                                                                        \
  case TV: {                                                                                             \
    {                                                                                                    \
      cudaError_t e = smem_attr((const void*)gemm_cm_kernel<TV>, 220 * 1024);                            \
      if (e != cudaSuccess) return e;                                                                    \
    }                                                                                                    \
    gemm_cm_kernel<TV><<<grid, 32 * cm_warps<TV>(), smem, st>>>(P);                                      \
    return cudaGetLastError();                                                                           \
  }
  switch (s / 8) {
    PB_CM(4) PB_CM(5) PB_CM(6) PB_CM(7) PB_CM(8)
  }
#undef PB_CM
  return cudaErrorInvalidValue;
}

bool gemm_small_ok(int s, const double* a, const double* b, const double* c, const double* d, long long sa,
                   long long sb, long long sc, long long sd, int cna, int cnb, int cnc, int cnd) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const long long ss = (long long)s * s;
  static const int mid_hi = [] {  // PBGPU_GEMM_MID_HI: largest order on gemm_mid_kernel (tuning)
    const char* e = getenv("PBGPU_GEMM_MID_HI");
    return e ? atoi(e) : 112;
  }();
  return s > 0 && s <= std::min(mid_hi, 112) && s % 4 == 0 && sa == ss && sb == ss && sc == ss && sd == ss && cna == s &&
         cnb == s && cnc == s && cnd == s && al(a) && al(b) && al(c) && al(d);
}

cudaError_t gemm_small_launch(int s, double alpha, const double* a, const double* b, double beta,
                              const double* c, double* d, long long batch, cudaStream_t st) {
  SmallArgs P;
  P.a = a; P.b = b; P.c = c; P.d = d;
  P.alpha = alpha; P.beta = beta;
  P.batch = batch;
  P.s = s;
  // chunk: <= 16 KB per operand; two stages of A, B, C = 96 KB, two CTAs per SM
  P.G = std::max(1, 2048 / (s * s));
  P.nchunks = (int)((batch + P.G - 1) / P.G);
  if (s == 4) {
    gemm_tiny4_kernel<<<(unsigned)((batch + 32 * kTinyWarps - 1) / (32 * kTinyWarps)), 32 * kTinyWarps, 0, st>>>(P);
    return cudaGetLastError();
  }
  if (s >= 28) return mid_launch(P, st);  // measured: ahead of the chunked kernel from s = 28
  switch ((s + 7) / 8) {
    case 1: return small_t<1>(P, st);
    case 2: return small_t<2>(P, st);
    case 3: return small_t<3>(P, st);
    case 4: return small_t<4>(P, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace pbg
