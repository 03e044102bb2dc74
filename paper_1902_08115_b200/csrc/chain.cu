// Fused panel-major syrk+potrf (syrk_potrf_nd) and the variable-size
// Riccati-like chain of config 5 (dsyrk -> dpotrf -> dtrsm), plus the batched
// small kernels they need (the per-class info scatter).
//
//   syrk_potrf_nd (level3.hpp:533-575): n <= 160 runs in ONE kernel — the
//   pipelined CTA Cholesky with the prologue S = C + A B^T on the tensor cores
//   and the LowerZero band store; larger n: gemm engine (lower S in D) ->
//   blocked panel-major potrf in place (band zeros by its diagonal blocks).
//
//   chain (pb_chain_vbatched): problems are split on the host by order.
//   n <= 160: variable-batch kernels straight on the caller's buffers
//     column-major: fused syrk+potrf (n > 32; syrk -> potrf_reg below) -> trsm X L^T = B
//     panel-major : fused syrk+potrf (prologue)  -> trsm_rltn
//   n > 160: per distinct order, the strided kernels (engine syrk, blocked
//   potrf, trsm_rlt) run on the caller's buffers through per-problem offsets.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <vector>

#include "common.cuh"
#include "launch.h"

namespace pbg {

// ------------------------------------------------------------------ small kernels
// Square n x n problems: ws[q] <- base + offs[q] (all of it) / base + offs[q] <- ws[q] (lower triangle)
__global__ void gather_kernel(const double* base, const long long* offs, double* ws, int n) {
  const int q = blockIdx.y;
  const long long nn = (long long)n * n;
  const double* s = base + offs[q];
  double* d = ws + (long long)q * nn;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nn; e += (long long)gridDim.x * blockDim.x)
    d[e] = s[e];
}
__global__ void scatter_lower_kernel(const double* ws, double* base, const long long* offs, int n) {
  const int q = blockIdx.y;
  const long long nn = (long long)n * n;
  const double* s = ws + (long long)q * nn;
  double* d = base + offs[q];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nn; e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / n), i = (int)(e - (long long)j * n);
    if (i >= j) d[e] = s[e];
  }
}
static dim3 grid2(long long work, int batch) {
  return dim3((unsigned)std::max<long long>(1, std::min<long long>((work + 255) / 256, 64)), (unsigned)batch);
}
__global__ void scatter_info_kernel(const int* src, const int* idx, int* info, int count) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < count; q += gridDim.x * blockDim.x) info[idx[q]] = src[q];
}


// ------------------------------------------------------------------ syrk_potrf_nd
cudaError_t syrk_potrf_launch(const SyrkPotrfLaunch& L, cudaStream_t s) {
  if (L.batch <= 0 || L.n <= 0) return cudaSuccess;
  // fused (S formed in the Cholesky kernel's prologue) up to n = 112 or k < 16;
  // above, the tile engine forms S first (measured: n = 128, k = 64 0.96 ->
  // 0.82 ms; n = 160, k = 160 1.70 -> 1.07 ms; the prologue wins at n <= 96).
  // On a numerical failure the engine path leaves S (not the caller's D) in the
  // entries outside the reference's partial write set, as the blocked n > 160 path.
  static const int fused_nmax = [] {
    const char* e = getenv("PBGPU_SYRK_POTRF_FUSED_NMAX");
    return e ? atoi(e) : 112;
  }();
  const bool fused_ok = L.n <= 160 && !L.offs && (L.n <= fused_nmax || L.k < 16) &&
                        (L.k == 0 || (L.cna == L.cnb && L.sa == L.sb));
  if (fused_ok)
    return syrk_potrf_cta_launch(L.d, L.sd, nullptr, nullptr, L.cnd, L.c, L.sc, L.cnc, L.k ? L.a : nullptr,
                                 L.k ? L.b : nullptr, L.sa, L.k, L.cna, L.n, 1, 1, L.info, L.batch, s);
  // Large n: lower S = C + A B^T into D (gemm engine), factor a column-major copy, pack back.
  cudaError_t e;
  GemmLaunch g;
  g.out_pm = 1;
  g.lay_a = L_PMX;
  g.lay_b = L_PMX;
  g.a.base = L.a; g.a.stride = L.sa; g.a.ld = L.cna;
  g.a.bulk = ((reinterpret_cast<uintptr_t>(L.a) & 15) == 0) && (L.offs ? L.offs_even != 0 : L.sa % 2 == 0);
  g.b.base = L.b; g.b.stride = L.sb; g.b.ld = L.cnb;
  g.b.bulk = ((reinterpret_cast<uintptr_t>(L.b) & 15) == 0) && (L.offs ? L.offs_even != 0 : L.sb % 2 == 0);
  g.o.c = L.c; g.o.d = L.d; g.o.sc = L.sc; g.o.sd = L.sd; g.o.ldc = L.cnc; g.o.ldd = L.cnd;
  g.o.vec = ((reinterpret_cast<uintptr_t>(L.c) & 15) == 0) && ((reinterpret_cast<uintptr_t>(L.d) & 15) == 0) &&
            (L.offs ? L.offs_even != 0 : (L.sc % 2 == 0 && L.sd % 2 == 0));  // pm pairs (i, i + 1), i even
  g.a.offs = g.b.offs = g.o.offs = L.offs;
  g.m = g.n = L.n;
  g.k = L.k;
  g.alpha = 1.0;
  g.beta = 1.0;
  g.uplo = 1;
  g.batch = L.batch;
  if (L.k > 0) e = gemm_launch(g, s);
  else e = scale_launch(1, g.o, L.n, L.n, 1.0, 1, L.batch, s);
  if (e != cudaSuccess) return e;
  // factor D in place, panel-major, with the LowerZero band zeros
  PotrfLaunch P;
  P.a = L.d; P.stride = L.sd; P.lda = L.cnd; P.n = L.n; P.pm = 1; P.zero_fill = 1;
  P.offs = L.offs; P.offs_even = L.offs_even;
  P.info = L.info; P.batch = L.batch;
  return potrf_launch(P, s);
}

// ------------------------------------------------------------------ chain (cfg 5)
// PBGPU_CHAIN_UNFUSED=1: column-major small orders as syrk -> potrf launches (A/B only)
static bool chain_unfused() {
  static const bool v = [] {
    const char* e = getenv("PBGPU_CHAIN_UNFUSED");
    return e && e[0] == '1';
  }();
  return v;
}

// PBGPU_CHAIN_CM_INPLACE=0: column-major large orders through the strided workspace (A/B only)
static bool cm_inplace_on() {
  static const bool v = [] {
    const char* e = getenv("PBGPU_CHAIN_CM_INPLACE");
    return !(e && e[0] == '0');
  }();
  return v;
}

// PBGPU_CHAIN_SYRK=fused: small orders form S in the Cholesky kernel's prologue (A/B only)
static bool chain_engine_syrk() {
  static const bool v = [] {
    const char* e = getenv("PBGPU_CHAIN_SYRK");
    return !(e && e[0] == 'f');
  }();
  return v;
}

// PBGPU_CHAIN_ENGINE_FROM=n: classes above n use the engine syrk (tuning)
static int chain_engine_from() {
  static const int v = [] {
    const char* e = getenv("PBGPU_CHAIN_ENGINE_FROM");
    return e ? atoi(e) : 32;
  }();
  return v;
}

// The order classes are independent problems: they are issued round-robin on a
// few side streams (forked from / joined to the caller's stream with events), so
// the tail of one class's launches overlaps the next class's instead of draining
// the GPU ~250 times per call.  PBGPU_CHAIN_STREAMS = 1 keeps one stream (A/B).
constexpr int kChainStreams = 4;
struct ChainPool {
  cudaStream_t st[kChainStreams] = {};
  cudaEvent_t done[kChainStreams] = {};
  cudaEvent_t fork = nullptr;
  bool ready = false;
};
static ChainPool* chain_pool() {
  static thread_local ChainPool pools[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  ChainPool& P = pools[dev];
  if (!P.ready) {
    for (int i = 0; i < kChainStreams; ++i) {
      if (cudaStreamCreateWithFlags(&P.st[i], cudaStreamNonBlocking) != cudaSuccess) return nullptr;
      if (cudaEventCreateWithFlags(&P.done[i], cudaEventDisableTiming) != cudaSuccess) return nullptr;
    }
    if (cudaEventCreateWithFlags(&P.fork, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    P.ready = true;
  }
  return &P;
}
static int chain_streams() {
  static const int v = [] {
    const char* e = getenv("PBGPU_CHAIN_STREAMS");
    const int n = e ? atoi(e) : kChainStreams;
    return n < 1 ? 1 : (n > kChainStreams ? kChainStreams : n);
  }();
  return v;
}

cudaError_t chain_launch(const ChainLaunch& L, cudaStream_t s0) {
  if (L.batch <= 0) return cudaSuccess;
  mempool_keep();
  cudaError_t e;
  cudaStream_t s = s0;  // the stream of the current class (a side stream after the fork)
  // The split by order is planned on the host: from the caller's host copies of
  // n / offset when given (no synchronisation), else from a device -> host copy.
  std::vector<int> nv(L.batch);
  std::vector<long long> ov(L.batch);
  if (L.n_host && L.offset_host) {
    std::copy(L.n_host, L.n_host + L.batch, nv.begin());
    std::copy(L.offset_host, L.offset_host + L.batch, ov.begin());
  } else {
    if ((e = cudaMemcpyAsync(nv.data(), L.n, sizeof(int) * L.batch, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    if ((e = cudaMemcpyAsync(ov.data(), L.offset, sizeof(long long) * L.batch, cudaMemcpyDeviceToHost, s)) !=
        cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  }
  std::vector<int> small;
  std::map<int, std::vector<int>> big;
  int nsmall_max = 0;
  for (int p = 0; p < L.batch; ++p) {
    if (nv[p] <= 160) {
      small.push_back(p);
      nsmall_max = std::max(nsmall_max, nv[p]);
    } else {
      big[nv[p]].push_back(p);
    }
  }
  ChainPool* pool = chain_streams() > 1 ? chain_pool() : nullptr;
  const int nstreams = pool ? chain_streams() : 1;
  int next_stream = 0;
  bool forked = false;
  auto fork = [&]() -> cudaError_t {  // side streams start after everything queued on s0 so far
    if (!pool || forked) return cudaSuccess;
    cudaError_t fe = cudaEventRecord(pool->fork, s0);
    for (int i = 0; i < nstreams && fe == cudaSuccess; ++i) fe = cudaStreamWaitEvent(pool->st[i], pool->fork, 0);
    forked = fe == cudaSuccess;
    return fe;
  };
  auto class_stream = [&]() -> cudaStream_t {
    if (!pool) return s0;
    cudaStream_t cs = pool->st[next_stream];
    next_stream = (next_stream + 1) % nstreams;
    return cs;
  };
  auto join = [&]() -> cudaError_t {  // s0 continues after every side stream
    if (!pool || !forked) return cudaSuccess;
    cudaError_t je = cudaSuccess;
    for (int i = 0; i < nstreams && je == cudaSuccess; ++i) {
      je = cudaEventRecord(pool->done[i], pool->st[i]);
      if (je == cudaSuccess) je = cudaStreamWaitEvent(s0, pool->done[i], 0);
    }
    forked = false;
    return je;
  };
  // Small orders: sorted by order and launched per 8-column class, so every
  // launch is sized (shared memory, warps, unrolling) for its own problems.
  std::sort(small.begin(), small.end(), [&](int x, int y) { return nv[x] < nv[y]; });
  const size_t nsm = small.size();
  int *d_idx = nullptr, *d_n = nullptr, *d_info = nullptr;
  long long* d_off = nullptr;
  std::vector<long long> so(nsm);
  std::vector<int> sn(nsm);
  if (nsm) {
    for (size_t q = 0; q < nsm; ++q) {
      so[q] = ov[small[q]];
      sn[q] = nv[small[q]];
    }
    if ((e = cudaMallocAsync(&d_idx, sizeof(int) * nsm, s)) != cudaSuccess ||
        (e = cudaMallocAsync(&d_n, sizeof(int) * nsm, s)) != cudaSuccess ||
        (e = cudaMallocAsync(&d_info, sizeof(int) * nsm, s)) != cudaSuccess ||
        (e = cudaMallocAsync(&d_off, sizeof(long long) * nsm, s)) != cudaSuccess)
      return e;
    cudaMemcpyAsync(d_idx, small.data(), sizeof(int) * nsm, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_n, sn.data(), sizeof(int) * nsm, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_off, so.data(), sizeof(long long) * nsm, cudaMemcpyHostToDevice, s);
  }
  // column-major large orders factor in a strided workspace (A gathered, S = C + A A^T,
  // then L): one per side stream, sized for the largest class that stream will see and
  // allocated here on the caller's stream — large stream-ordered allocations issued
  // concurrently from several streams made the pool serialise or grow (cm 32 -> 49 ms)
  double* ws_stream[kChainStreams] = {};
  // 16-byte aligned column-major problems take the panel-major route below: in
  // place on the caller's buffers through the offsets (tensor maps with offset
  // dimensions in the engine), no workspace, gather or scatter
  bool cm_inplace = !L.pm && cm_inplace_on() && (reinterpret_cast<uintptr_t>(L.A) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(L.C) & 15) == 0;
  for (auto& kv : big) {
    if (!cm_inplace) break;
    cm_inplace = kv.first % 2 == 0;
    for (int q : kv.second) cm_inplace = cm_inplace && ov[q] % 2 == 0;
  }
  if (!L.pm && !cm_inplace && !big.empty()) {
    size_t need[kChainStreams] = {};
    int k = 0;
    for (auto it = big.rbegin(); it != big.rend(); ++it, k = (k + 1) % nstreams)
      need[k] = std::max(need[k], (size_t)2 * it->first * it->first * it->second.size());
    for (int i = 0; i < nstreams; ++i)
      if (need[i] && (e = cudaMallocAsync(&ws_stream[i], sizeof(double) * need[i], s0)) != cudaSuccess) return e;
  }
  if ((e = fork()) != cudaSuccess) return e;
  // large orders, per distinct n: the syrk, the blocked Cholesky and the solve
  // run straight on the caller's buffers through per-problem offsets (the
  // class's members), so nothing is gathered or scattered
  for (auto it = big.rbegin(); it != big.rend(); ++it) {  // largest orders first
    auto& kv = *it;
    const int stream_slot = next_stream;
    s = class_stream();
    const int n = kv.first, cnt = (int)kv.second.size();
    int *d_i = nullptr, *w_info = nullptr;
    long long* d_o = nullptr;
    if ((e = cudaMallocAsync(&d_i, sizeof(int) * cnt, s)) != cudaSuccess ||
        (e = cudaMallocAsync(&w_info, sizeof(int) * cnt, s)) != cudaSuccess ||
        (e = cudaMallocAsync(&d_o, sizeof(long long) * cnt, s)) != cudaSuccess)
      return e;
    std::vector<long long> ob(cnt);
    bool even = true;
    for (int q = 0; q < cnt; ++q) {
      ob[q] = ov[kv.second[q]];
      even = even && (ob[q] % 2 == 0);
    }
    cudaMemcpyAsync(d_i, kv.second.data(), sizeof(int) * cnt, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_o, ob.data(), sizeof(long long) * cnt, cudaMemcpyHostToDevice, s);
    double* wc = nullptr;  // column-major: the factor's workspace (S = C + A A^T, then L)
    double* wa = nullptr;
    if (cm_inplace) {
      GemmLaunch g;  // dsyrk('l','n') in place: C += A A^T (lower)
      g.lay_a = g.lay_b = L_MNC;
      g.a.base = g.b.base = L.A; g.a.offs = g.b.offs = d_o; g.a.ld = g.b.ld = n; g.a.bulk = g.b.bulk = 1;
      g.o.c = L.C; g.o.d = L.C; g.o.offs = d_o; g.o.ldc = g.o.ldd = n; g.o.vec = 1;
      g.m = g.n = g.k = n;
      g.alpha = 1.0; g.beta = 1.0; g.uplo = 1; g.batch = cnt;
      e = gemm_launch(g, s);
      if (e == cudaSuccess) {
        PotrfLaunch P;
        P.a = L.C; P.offs = d_o; P.offs_even = 1; P.lda = n; P.n = n; P.info = w_info; P.batch = cnt;
        e = potrf_launch(P, s);
      }
    } else if (!L.pm) {
      // column-major: A streams straight from the caller's buffer through the
      // engine's offset tensor maps (16-byte aligned problems; otherwise it is
      // gathered into the strided workspace first), S = C + A A^T lands in a
      // strided workspace (C read through the offsets), is factored there, and
      // only L's lower triangle goes back to C
      const long long nn = (long long)n * n;
      wa = ws_stream[pool ? stream_slot : 0];
      wc = wa + nn * cnt;
      GemmLaunch g;  // dsyrk('l','n'): S = C + A A^T
      g.lay_a = g.lay_b = L_MNC;
      if (even && n % 2 == 0 && (reinterpret_cast<uintptr_t>(L.A) & 15) == 0) {
        g.a.base = g.b.base = L.A; g.a.offs = g.b.offs = d_o; g.a.ld = g.b.ld = n; g.a.bulk = g.b.bulk = 1;
      } else {
        gather_kernel<<<grid2(nn, cnt), 256, 0, s>>>(L.A, d_o, wa, n);
        g.a.base = g.b.base = wa; g.a.stride = g.b.stride = nn; g.a.ld = g.b.ld = n; g.a.bulk = g.b.bulk = 1;
      }
      g.o.c = L.C; g.o.offs_c = d_o; g.o.d = wc; g.o.sd = nn; g.o.ldc = g.o.ldd = n;
      g.o.vec = even && n % 2 == 0 && (reinterpret_cast<uintptr_t>(L.C) & 15) == 0;
      g.m = g.n = g.k = n;
      g.alpha = 1.0; g.beta = 1.0; g.uplo = 1; g.batch = cnt;
      e = gemm_launch(g, s);
      if (e == cudaSuccess) {
        PotrfLaunch P;
        P.a = wc; P.stride = nn; P.lda = n; P.n = n; P.info = w_info; P.batch = cnt;
        e = potrf_launch(P, s);
      }
    } else {
      SyrkPotrfLaunch S;
      S.a = S.b = L.A; S.c = L.C; S.d = L.C;
      S.offs = d_o;
      S.offs_even = even && (reinterpret_cast<uintptr_t>(L.A) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(L.C) & 15) == 0;
      S.cna = S.cnb = S.cnc = S.cnd = n;
      S.n = S.k = n;
      S.info = w_info;
      S.batch = cnt;
      e = syrk_potrf_launch(S, s);
    }
    if (e == cudaSuccess) {
      TrsmLaunch T;
      T.pm = L.pm;
      T.lower = 1; T.trans = 1; T.unit = 0;
      T.mm = T.nn = n;
      T.alpha = 1.0;
      const bool in_c = L.pm || cm_inplace;
      T.a = in_c ? L.C : wc; T.offs_a = in_c ? d_o : nullptr; T.sa = (long long)n * n; T.lda = n;
      T.b = L.B; T.ldb = n;
      T.d = L.B; T.ldd = n;
      T.offs_b = d_o;
      T.info = w_info;
      T.skip_nonzero = 1;
      T.batch = cnt;
      e = trsm_launch(T, s);
    }
    if (e == cudaSuccess && !L.pm && !cm_inplace) {
      scatter_lower_kernel<<<grid2((long long)n * n, cnt), 256, 0, s>>>(wc, L.C, d_o, n);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
      scatter_info_kernel<<<std::max(1, (cnt + 255) / 256), 256, 0, s>>>(w_info, d_i, L.info, cnt);
      e = cudaGetLastError();
    }
    cudaFreeAsync(d_i, s);
    cudaFreeAsync(d_o, s);
    cudaFreeAsync(w_info, s);
    if (e != cudaSuccess) return e;
  }
  // small orders after the large ones (the longest work first), on the same side streams
  if (nsm) {
    for (size_t b0 = 0; b0 < nsm && e == cudaSuccess;) {
      s = class_stream();
      const int cls = (sn[b0] + 7) / 8;
      size_t b1 = b0;
      while (b1 < nsm && (sn[b1] + 7) / 8 == cls) ++b1;
      const int bs = (int)(b1 - b0), nmax = sn[b1 - 1];
      int* bn = d_n + b0;
      int* binfo = d_info + b0;
      long long* boff = d_off + b0;
      if (nmax > chain_engine_from() && chain_engine_syrk()) {
        // S = C + A A^T per distinct order on the tile engine (per-problem offsets,
        // bulk-copied operands), then the Cholesky of the class without a prologue
        for (size_t c0 = b0; c0 < b1 && e == cudaSuccess;) {
          size_t c1 = c0;
          while (c1 < b1 && sn[c1] == sn[c0]) ++c1;
          const int n = sn[c0];
          bool even = n % 2 == 0;
          for (size_t q = c0; q < c1; ++q) even = even && so[q] % 2 == 0;
          GemmLaunch g;
          g.lay_a = g.lay_b = L.pm ? L_PMX : L_MNC;
          g.out_pm = L.pm;
          g.a.base = g.b.base = L.A; g.a.ld = g.b.ld = n; g.a.offs = g.b.offs = d_off + c0;
          g.a.bulk = g.b.bulk = even && (reinterpret_cast<uintptr_t>(L.A) & 15) == 0;
          g.o.c = L.C; g.o.d = L.C; g.o.ldc = g.o.ldd = n; g.o.offs = d_off + c0;
          g.o.vec = even && (reinterpret_cast<uintptr_t>(L.C) & 15) == 0;
          g.m = g.n = g.k = n;
          g.alpha = 1.0; g.beta = 1.0; g.uplo = 1; g.batch = (int)(c1 - c0);
          e = gemm_launch(g, s);
          c0 = c1;
        }
        if (e == cudaSuccess)
          e = potrf_cta_launch(L.C, 0, boff, bn, 0, nmax, 0, L.pm, L.pm, binfo, 0, 0, bs, s);
      } else if (!L.pm && (nmax <= 32 || chain_unfused())) {
        // register-resident Cholesky for the smallest orders: syrk first, then potrf_reg
        e = syrk_lower_cta_launch(L.C, boff, bn, L.A, nmax, 0, binfo, bs, s);
        if (e == cudaSuccess) e = potrf_cta_launch(L.C, 0, boff, bn, 0, nmax, 0, 0, 0, binfo, 0, 0, bs, s);
      } else if (!L.pm) {
        // one kernel: S = C + A A^T (lower) formed in shared memory, factored there, written once
        e = syrk_potrf_cta_launch(L.C, 0, boff, bn, 0, L.C, 0, 0, L.A, L.A, 0, 1, 0, nmax, 0, 0, binfo, bs, s);
      } else {
        e = syrk_potrf_cta_launch(L.C, 0, boff, bn, 0, L.C, 0, 0, L.A, L.A, 0, 1, 0, nmax, 1, 1, binfo, bs, s);
      }
      if (e == cudaSuccess) {
        TrsmLaunch T;
        T.pm = L.pm;
        T.lower = 1; T.trans = 1; T.unit = 0;
        T.mm = T.nn = nmax;
        T.alpha = 1.0;
        T.a = L.C; T.b = L.B; T.d = L.B;
        T.nvec = bn; T.offs = boff;
        T.info = binfo;
        T.skip_nonzero = 1;
        T.batch = bs;
        e = trsm_launch(T, s);
      }
      b0 = b1;
    }
  }
  if (e != cudaSuccess) return e;
  s = s0;
  if ((e = join()) != cudaSuccess) return e;
  for (int i = 0; i < kChainStreams; ++i)
    if (ws_stream[i]) cudaFreeAsync(ws_stream[i], s0);
  if (nsm) {
    if (e == cudaSuccess) {
      scatter_info_kernel<<<std::max(1, (int)((nsm + 255) / 256)), 256, 0, s>>>(d_info, d_idx, L.info, (int)nsm);
      e = cudaGetLastError();
    }
    cudaFreeAsync(d_idx, s);
    cudaFreeAsync(d_n, s);
    cudaFreeAsync(d_info, s);
    cudaFreeAsync(d_off, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace pbg
