// Small column-major dgemm, m, n <= 32 (any k, lda/ldb/ldc, all four trans
// pairs): one warp per problem (sm_100a).
//
// The small-n branch of the size switch for the column-major BLAS entry — the
// analogue of the reference's variant D / kernel_gemm_ccc (gemm.hpp:190-204,
// 360-400; micro_kernel.hpp:500-515), which skips packing when the whole
// problem is a register tile or two.  On the GPU the engine's 64x64 CTA tile
// would spend >= 75 % of a work item on padding at n <= 32 (>= 94 % at n <= 16);
// here a warp owns a problem:
//   * op(A) and op(B) are staged k-chunk by k-chunk (32 columns) into the warp's
//     own shared-memory slices with coalesced global loads — A as k-major rows
//     As[l][i] (stride 8 MT + 4), B as Bs[j][l] (stride 36), both strides = 4 mod
//     16 doubles, so DMMA fragment loads are conflict-free;
//   * up to 4 x 4 tiles of 8x8 accumulate on DMMA m8n8k4 as the transposed
//     product C^T = op(B)^T op(A)^T: a lane then owns rows 2t, 2t+1 of one
//     column of each tile, so beta*C and D move as 16-byte pairs when ldc and the
//     base allow (8-byte accesses otherwise);
//   * rows / columns past m, n and k are staged as zeros and masked at the
//     store; beta == 0 never reads C (NaN-safe, micro_kernel.hpp:266-268).
// No block-level barrier: warps are independent, latency hides across the 12-16
// resident warps of an SM.
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace pbg {

struct CmSmallArgs {
  const double* a;
  const double* b;
  double* c;
  long long sa, sb, sc;
  int lda, ldb, ldc;
  int m, n, k, ta, tb;
  double alpha, beta;
  long long batch;
  int vec;   // 16-byte C accesses allowed
  int uplo;  // 0 full, 1 lower (i >= j), 2 upper (i <= j): entries outside are neither read nor written (dsyrk)
};

constexpr int kCmsWarps = 4;

// registers capped so that shared memory, not the register file, bounds residency (3 CTAs at MT = 4)
template <int MT>
__global__ void __launch_bounds__(32 * kCmsWarps, MT >= 3 ? 3 : (MT == 2 ? 5 : 9)) gemm_cmsmall_kernel(const __grid_constant__ CmSmallArgs P) {
  constexpr int MR = 8 * MT;      // rows / columns covered (m, n <= MR)
  constexpr int SA = MR + 4;      // As[l][i]: stride between k-rows
  constexpr int SB = 36;          // Bs[j][l]: stride between columns of op(B)
  constexpr int WSZ = 32 * SA + MR * SB;  // doubles per warp
  constexpr int LPP = 32 / MR;    // staging: k-columns (A) / columns (B) per pass
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* As = sm + (size_t)warp * WSZ;
  double* Bs = As + 32 * SA;
  const uint32_t as32 = smem_u32(As), bs32 = smem_u32(Bs);
  const int m = P.m, n = P.n, k = P.k;
  const bool use_c = P.beta != 0.0;
  const int si = lane % MR, sl = lane / MR;  // staging coordinates (lanes >= LPP * MR idle)
  const bool son = sl < LPP;

  for (long long p = (long long)blockIdx.x * kCmsWarps + warp; p < P.batch; p += (long long)gridDim.x * kCmsWarps) {
    const double* a = P.a + p * P.sa;
    const double* b = P.b + p * P.sb;
    double* c = P.c + p * P.sc;
    double acc[MT][MT][2];  // [J][I]: C rows 8I + 2t, +1 of column 8J + g
#pragma unroll
    for (int J = 0; J < MT; ++J)
#pragma unroll
      for (int I = 0; I < MT; ++I) acc[J][I][0] = acc[J][I][1] = 0.0;

    for (int l0 = 0; l0 < k; l0 += 32) {
      const int kc = min(32, k - l0);
      const int kc4 = (kc + 3) & ~3;
      __syncwarp();  // the previous chunk's fragments are consumed
      // ---- stage op(A)(i, l0 + l) -> As[l][i] and op(B)(l0 + l, j) -> Bs[j][l] ----
      // x = the operand's tile index (i of op(A), j of op(B)), xs / ls = destination strides.
      // Stored with x contiguous (A 'n', B 't'): lanes = (x, a few k-columns per pass);
      // stored with l contiguous (A 't', B 'n'): lanes along l, one x per pass.
      // Every global load of a pass is issued before the first shared-memory store
      // (fixed trip counts, predicated): the warp keeps up to 32 loads in flight.
      auto stage = [&](const double* src, int ld, bool x_contig, int xvalid, double* dst, int xs, int ls) {
        if (x_contig) {
          constexpr int NPASS = (32 + LPP - 1) / LPP;
          double v[NPASS];
#pragma unroll
          for (int q = 0; q < NPASS; ++q) {
            const int l = sl + q * LPP;
            v[q] = 0.0;
            if (son && si < xvalid && l < kc) v[q] = ldg_stream(src + si + (long long)(l0 + l) * ld);
          }
#pragma unroll
          for (int q = 0; q < NPASS; ++q) {
            const int l = sl + q * LPP;
            if (son && l < kc4) dst[si * xs + l * ls] = v[q];
          }
        } else {
          double v[MR];
#pragma unroll
          for (int x = 0; x < MR; ++x) {
            v[x] = 0.0;
            if (x < xvalid && lane < kc) v[x] = ldg_stream(src + l0 + lane + (long long)x * ld);
          }
#pragma unroll
          for (int x = 0; x < MR; ++x)
            if (lane < kc4) dst[x * xs + lane * ls] = v[x];
        }
      };
      stage(a, P.lda, P.ta == 0, m, As, 1, SA);
      stage(b, P.ldb, P.tb != 0, n, Bs, SB, 1);
      __syncwarp();
      // ---- DMMA: acc[J][I] += op(B)^T tile J x op(A)^T tile I ----
      const int ksteps = kc4 >> 2;
      for (int ks = 0; ks < ksteps; ++ks) {
        double af[MT], bf[MT];
#pragma unroll
        for (int I = 0; I < MT; ++I) af[I] = lds64(as32 + 8u * (uint32_t)((4 * ks + t) * SA + 8 * I + g));
#pragma unroll
        for (int J = 0; J < MT; ++J) bf[J] = lds64(bs32 + 8u * (uint32_t)((8 * J + g) * SB + 4 * ks + t));
#pragma unroll
        for (int J = 0; J < MT; ++J)
#pragma unroll
          for (int I = 0; I < MT; ++I) dmma(acc[J][I][0], acc[J][I][1], bf[J], af[I]);
      }
    }
    // ---- epilogue: d = alpha * acc + beta * c on the valid part ----
    // every C load first, then the stores: a store to C between two loads would pin
    // the loads in program order (they may alias) and serialise MT*MT DRAM round trips
    double cv[MT][MT][2];
#pragma unroll
    for (int J = 0; J < MT; ++J)
#pragma unroll
      for (int I = 0; I < MT; ++I) {
        const int i = 8 * I + 2 * t, j = 8 * J + g;
        cv[J][I][0] = cv[J][I][1] = 0.0;
        if (!use_c || j >= n || i >= m) continue;
        const double* cp = c + i + (long long)j * P.ldc;
        const bool in0 = P.uplo == 0 || (P.uplo == 1 ? i >= j : i <= j);
        const bool in1 = P.uplo == 0 || (P.uplo == 1 ? i + 1 >= j : i + 1 <= j);
        if (!(in0 && in1)) {  // the pair straddles the diagonal (or lies outside): element-wise
          if (in0) cv[J][I][0] = cp[0];
          if (in1 && i + 1 < m) cv[J][I][1] = cp[1];
          continue;
        }
        if (P.vec && i + 1 < m) {
          const double2 v = *reinterpret_cast<const double2*>(cp);
          cv[J][I][0] = v.x;
          cv[J][I][1] = v.y;
        } else {
          cv[J][I][0] = cp[0];
          if (i + 1 < m) cv[J][I][1] = cp[1];
        }
      }
#pragma unroll
    for (int J = 0; J < MT; ++J)
#pragma unroll
      for (int I = 0; I < MT; ++I) {
        const int i = 8 * I + 2 * t, j = 8 * J + g;
        if (j >= n || i >= m) continue;
        double* cp = c + i + (long long)j * P.ldc;
        const bool two = i + 1 < m;
        const double r0 = use_c ? fma(P.alpha, acc[J][I][0], P.beta * cv[J][I][0]) : acc[J][I][0] * P.alpha;
        const double r1 = use_c ? fma(P.alpha, acc[J][I][1], P.beta * cv[J][I][1]) : acc[J][I][1] * P.alpha;
        const bool in0 = P.uplo == 0 || (P.uplo == 1 ? i >= j : i <= j);
        const bool in1 = P.uplo == 0 || (P.uplo == 1 ? i + 1 >= j : i + 1 <= j);
        if (!(in0 && in1)) {
          if (in0) cp[0] = r0;
          if (in1 && two) cp[1] = r1;
          continue;
        }
        if (P.vec && two) {
          *reinterpret_cast<double2*>(cp) = make_double2(r0, r1);
        } else {
          cp[0] = r0;
          if (two) cp[1] = r1;
        }
      }
  }
}

template <int MT>
static cudaError_t cmsmall_t(const CmSmallArgs& P, cudaStream_t s) {
  constexpr int MR = 8 * MT;
  const size_t smem = (size_t)kCmsWarps * (32 * (MR + 4) + MR * 36) * sizeof(double);
  cudaError_t e = smem_attr((const void*)gemm_cmsmall_kernel<MT>, (int)smem, true);
  if (e != cudaSuccess) return e;
  // persistent grid = exactly the CTAs the device holds at once (a larger grid would run a
  // second, nearly empty wave: problems are dealt to CTAs by a fixed stride); the occupancy
  // query is cached per device
  static std::atomic<int> resident[64];
  int dev = 0;
  cudaGetDevice(&dev);
  dev = dev >= 0 && dev < 64 ? dev : 0;
  int per_sm = resident[dev].load(std::memory_order_relaxed);
  if (per_sm <= 0) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemm_cmsmall_kernel<MT>, 32 * kCmsWarps, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    resident[dev].store(per_sm, std::memory_order_relaxed);
  }
  const long long want = (P.batch + kCmsWarps - 1) / kCmsWarps;
  const long long cap = (long long)num_sms() * per_sm;
  gemm_cmsmall_kernel<MT><<<(unsigned)(want < cap ? want : cap), 32 * kCmsWarps, smem, s>>>(P);
  return cudaGetLastError();
}

bool gemm_cmsmall_ok(int m, int n) {
  static const bool off = [] {
    const char* e = getenv("PBGPU_GEMM_CMSMALL");
    return e && e[0] == '0';
  }();
  return !off && m >= 1 && n >= 1 && m <= 32 && n <= 32;
}

cudaError_t gemm_cmsmall_launch(int ta, int tb, int m, int n, int k, double alpha, const double* a, int lda,
                                long long sa, const double* b, int ldb, long long sb, double beta, double* c,
                                int ldc, long long sc, int uplo, long long batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  CmSmallArgs P{a, b, c, sa, sb, sc, lda, ldb, ldc, m, n, k, ta, tb, alpha, beta, batch, 0, uplo};
  P.vec = (reinterpret_cast<uintptr_t>(c) & 15) == 0 && ldc % 2 == 0 && sc % 2 == 0;
  const int mx = m > n ? m : n;
  if (mx <= 8) return cmsmall_t<1>(P, s);
  if (mx <= 16) return cmsmall_t<2>(P, s);
  if (mx <= 24) return cmsmall_t<3>(P, s);
  return cmsmall_t<4>(P, s);
}

}  // namespace pbg
