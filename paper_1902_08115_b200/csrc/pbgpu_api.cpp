// Host side of the drop-in boundary (include/pbgpu.h).
//
// Mirrors the reference's adapters (blas.hpp:73-215) and native panel
// entry points (level3.hpp:360-575): identical argument validation order,
// argument positions, messages, LAPACK/BLAS info conventions and quick
// returns — all decided on the host before anything is launched.  The
// arithmetic then runs in the sm_100a kernels (gemm.cu, potrf.cu, getrf.cu,
// trsm.cu, chain.cu); there is no CPU compute path.  Host-memory calls are
// staged through the GPU in chunks on two streams so H2D, compute and D2H of
// consecutive chunks overlap.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "launch.h"
#include "pbgpu.h"

using namespace pbg;

namespace {

// ------------------------------------------------------------ result plumbing
int finish(pb_result* res, int info, long long flops) {
  if (res) {
    res->info = info;
    res->error_index = 0;
    res->routine = nullptr;
    res->message = nullptr;
    res->flops = info == 0 ? flops : 0;
  }
  return info;
}
// Invalid argument: BlasCallError{routine, index, message} (blas.hpp:44-52).
int fail(pb_result* res, const char* routine, int index, int info, const char* msg) {
  if (res) {
    res->info = info;
    res->error_index = index;
    res->routine = routine;
    res->message = msg;
    res->flops = 0;
  }
  return info;
}
// Engine Status failure (no argument report).
int status(pb_result* res, int info, const char* msg) {
  if (res) {
    res->info = info;
    res->error_index = 0;
    res->routine = nullptr;
    res->message = msg;
    res->flops = 0;
  }
  return info;
}
// Numerical failure of a factorization: the reference still reports the
// flop count (factor.hpp:93, 222-223 set flops after the failure status).
int numerical(pb_result* res, int info, const char* msg, long long flops) {
  status(res, info, msg);
  if (res) res->flops = flops;
  return info;
}
int cuda_fail(pb_result* res, const char* routine, cudaError_t e) {
  cudaGetLastError();
  if (res) {
    res->info = PB_INFO_CUDA_ERROR;
    res->error_index = 0;
    res->routine = routine;
    res->message = cudaGetErrorString(e);
    res->flops = 0;
  }
  return PB_INFO_CUDA_ERROR;
}

int parse_trans(char c) {  // mat_view.hpp:26-32
  switch (c) {
    case 'n': case 'N': return 0;
    case 't': case 'T': case 'c': case 'C': return 1;
  }
  return -1;
}
int parse_uplo(char c) {  // 1 = Lower
  switch (c) {
    case 'l': case 'L': return 1;
    case 'u': case 'U': return 0;
  }
  return -1;
}
int parse_side(char c) {  // 1 = Left
  switch (c) {
    case 'l': case 'L': return 1;
    case 'r': case 'R': return 0;
  }
  return -1;
}
int parse_diag(char c) {  // 1 = Unit
  switch (c) {
    case 'n': case 'N': return 0;
    case 'u': case 'U': return 1;
  }
  return -1;
}

bool device_ok() {
  static int count = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
    cudaGetLastError();
  });
  return count > 0;
}

// ------------------------------------------------------------ memory kinds
enum Kind { K_NONE, K_DEVICE, K_HOST };
Kind kind_of(const void* p) {
  if (!p) return K_NONE;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return K_HOST;
  }
  return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) ? K_DEVICE : K_HOST;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// True when a column-major output region has no gaps (padding rows or
// inter-problem slack) that a host round trip would have to preserve.
bool dense(int rows, int ld, long long stride, int cols, int batch) {
  return ld == rows && (batch == 1 || stride == (long long)ld * cols);
}

// One operand of a batched call: problem p occupies
// [p*stride, p*stride + extent) elements of `ptr`.
struct Operand {
  void* ptr = nullptr;
  size_t esize = 8;
  long long stride = 0;
  long long extent = 0;
  bool in = true, out = false;
};

// Per-thread staging resources for host-pointer calls (per device).
// Host-pointer staging state: per calling thread AND per device (a thread that
// drives several GPUs keeps one set of streams and buffers on each).
struct Stager {
  int device = -1;
  cudaStream_t st[2] = {nullptr, nullptr};
  std::vector<void*> bufs[2];
  std::vector<size_t> caps[2];
  ~Stager() {
    // Process teardown may already have destroyed the context: ignore errors.
    int cur = -1;
    cudaGetDevice(&cur);
    if (device >= 0) cudaSetDevice(device);
    for (int s = 0; s < 2; ++s) {
      for (void* b : bufs[s]) cudaFree(b);
      if (st[s]) cudaStreamDestroy(st[s]);
    }
    if (cur >= 0) cudaSetDevice(cur);
    cudaGetLastError();
  }
  cudaError_t ensure(int dev, size_t nops) {
    device = dev;
    for (int s = 0; s < 2; ++s) {
      if (!st[s]) {
        cudaError_t e = cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
      }
      if (bufs[s].size() < nops) {
        bufs[s].resize(nops, nullptr);
        caps[s].resize(nops, 0);
      }
    }
    return cudaSuccess;
  }
  cudaError_t buf(int s, size_t i, size_t bytes, void** out) {
    if (caps[s][i] < bytes) {
      if (bufs[s][i]) cudaFree(bufs[s][i]);
      bufs[s][i] = nullptr;
      caps[s][i] = 0;
      size_t want = std::max(bytes, (size_t)1 << 20);
      cudaError_t e = cudaMalloc(&bufs[s][i], want);
      if (e != cudaSuccess) return e;
      caps[s][i] = want;
    }
    *out = bufs[s][i];
    return cudaSuccess;
  }
};
thread_local std::map<int, Stager> g_stagers;  // device -> this thread's staging state

size_t region_bytes(const Operand& o, long long nb) {
  if (nb <= 0 || o.extent <= 0) return 0;
  return (size_t)((nb - 1) * o.stride + o.extent) * o.esize;
}

// Runs launch(ptrs, nb, stream) over the batch.  Device operands run in one
// launch on the caller's stream; host operands are staged in chunks.
//
// `result` names the operand holding the routine's result: under
// PBGPU_MUTATE=eps (fault injection, the analogue of PANELBLAS_MUTATE,
// gemm.hpp:126-127) element (0, 0) of every problem's result is perturbed
// by eps after the launch, so the parity harness can be shown to go red.
template <class F>
int run_batched(const char* routine, std::vector<Operand> ops, int batch, pb_stream stream,
                pb_result* res, int result, F&& launch) {
  const double eps = mutation_epsilon();
  auto run = [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
    cudaError_t e = launch(p, nb, s);
    if (e == cudaSuccess && eps != 0.0 && result >= 0 && p[result])
      e = mutate_launch((double*)p[result], ops[result].stride, nullptr, nb, eps, s);
    return e;
  };
  if (!device_ok()) return status(res, PB_INFO_NO_DEVICE, "no CUDA device: pbgpu has no CPU path");
  int ndev = 0, nhost = 0;
  for (auto& o : ops) {
    Kind k = kind_of(o.ptr);
    if (k == K_DEVICE) ++ndev;
    if (k == K_HOST) ++nhost;
  }
  if (ndev && nhost) return status(res, PB_INFO_CUDA_ERROR, "mixed host and device pointers in one call");
  std::vector<void*> ptrs(ops.size());
  if (!nhost) {
    for (size_t i = 0; i < ops.size(); ++i) ptrs[i] = ops[i].ptr;
    cudaError_t e = run(ptrs, batch, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(res, routine, e);
    return 0;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  Stager& S = g_stagers[dev];
  cudaError_t e = S.ensure(dev, ops.size());
  if (e != cudaSuccess) return cuda_fail(res, routine, e);
  size_t per = 0;
  for (auto& o : ops) per += (size_t)std::max<long long>(o.stride, o.extent) * o.esize;
  const size_t target = (size_t)48 << 20;
  long long chunk = std::max<long long>(1, std::min<long long>(batch, (long long)(target / std::max<size_t>(per, 1))));
  int nchunks = (int)((batch + chunk - 1) / chunk);
  // Do not start before earlier work on the caller's stream (NULL: the legacy
  // default stream, which the non-blocking staging streams do not wait for)
  // has finished: it may still be writing the host buffers.
  e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(res, routine, e);
  for (int c = 0; c < nchunks; ++c) {
    int s = c & 1;
    long long p0 = (long long)c * chunk, nb = std::min<long long>(chunk, batch - p0);
    for (size_t i = 0; i < ops.size(); ++i) {
      const Operand& o = ops[i];
      if (!o.ptr) { ptrs[i] = nullptr; continue; }
      size_t bytes = region_bytes(o, nb);
      void* d = nullptr;
      e = S.buf(s, i, bytes, &d);
      if (e != cudaSuccess) return cuda_fail(res, routine, e);
      ptrs[i] = d;
      if (o.in && bytes) {
        e = cudaMemcpyAsync(d, (char*)o.ptr + (size_t)(p0 * o.stride) * o.esize, bytes,
                            cudaMemcpyHostToDevice, S.st[s]);
        if (e != cudaSuccess) return cuda_fail(res, routine, e);
      }
    }
    e = run(ptrs, (int)nb, S.st[s]);
    if (e != cudaSuccess) return cuda_fail(res, routine, e);
    for (size_t i = 0; i < ops.size(); ++i) {
      const Operand& o = ops[i];
      if (!o.ptr || !o.out) continue;
      size_t bytes = region_bytes(o, nb);
      if (!bytes) continue;
      e = cudaMemcpyAsync((char*)o.ptr + (size_t)(p0 * o.stride) * o.esize, ptrs[i], bytes,
                          cudaMemcpyDeviceToHost, S.st[s]);
      if (e != cudaSuccess) return cuda_fail(res, routine, e);
    }
  }
  for (int s = 0; s < 2; ++s) {
    e = cudaStreamSynchronize(S.st[s]);
    if (e != cudaSuccess) return cuda_fail(res, routine, e);
  }
  return 0;
}

long long cm_extent(int rows, int cols, int ld) {  // ld*(cols-1) + rows
  if (rows <= 0 || cols <= 0) return 0;
  return (long long)ld * (cols - 1) + rows;
}
long long pm_extent(const pb_dmat& d) {
  if (d.m <= 0 || d.n <= 0) return 0;
  return (long long)d.pm * d.cn;
}

// Single-problem host calls report numerical info through a scratch cell of
// the same memory kind as the matrix.
struct InfoCell {
  int host = 0;
  int* dev = nullptr;
};

// ------------------------------------------------------------ gemm helpers
OpDesc cm_side(const void* base, long long stride, int ld, int trans_contig_x, int xdim, int k) {
  // trans_contig_x: 1 when x is the contiguous index (L_MNC), 0 when l is (L_KC).
  OpDesc d;
  d.base = (const double*)base;
  d.stride = stride;
  d.ld = ld;
  (void)trans_contig_x; (void)xdim; (void)k;
  // TMA tensor maps need 16-byte aligned base and byte strides.
  d.bulk = aligned16(base) && (stride % 2 == 0) && (ld % 2 == 0);
  return d;
}

}  // namespace

extern "C" {

int pb_version(void) { return 100; }

int pb_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

double pb_probe_dmma_tflops(void) { return device_ok() ? probe_dmma_tflops() : 0.0; }

// ============================================================== dgemm family
static int dgemm_impl(const char* routine, bool batched, char transa, char transb, int m, int n,
                      int k, double alpha, const double* a, int lda, long long sa, const double* b,
                      int ldb, long long sb, double beta, double* c, int ldc, long long sc,
                      int batch, pb_stream stream, pb_result* res) {
  // blas.hpp:77-91: validation in Fortran argument order.
  int ta = parse_trans(transa);
  if (ta < 0) return fail(res, routine, 1, 1, "transa is not one of n, t, c");
  int tb = parse_trans(transb);
  if (tb < 0) return fail(res, routine, 2, 2, "transb is not one of n, t, c");
  if (m < 0) return fail(res, routine, 3, 3, "m is negative");
  if (n < 0) return fail(res, routine, 4, 4, "n is negative");
  if (k < 0) return fail(res, routine, 5, 5, "k is negative");
  int nrowa = ta == 0 ? m : k;
  int nrowb = tb == 0 ? k : n;
  if (lda < std::max(1, nrowa)) return fail(res, routine, 8, 8, "lda is smaller than the rows of op(a)");
  if (ldb < std::max(1, nrowb)) return fail(res, routine, 10, 10, "ldb is smaller than the rows of op(b)");
  if (ldc < std::max(1, m)) return fail(res, routine, 13, 13, "ldc is smaller than m");
  if (batched) {
    if (batch < 0) return fail(res, routine, 14, 14, "batch is negative");
    if (sa < 0 || sb < 0 || sc < 0) return fail(res, routine, 15, 15, "a stride is negative");
  }
  // blas.hpp:93-95 quick returns.
  if (m == 0 || n == 0 || batch == 0) return finish(res, 0, 0);
  if ((alpha == 0.0 || k == 0) && beta == 1.0) return finish(res, 0, 0);
  const bool scale_only = alpha == 0.0 || k == 0;  // gemm.hpp:443
  long long flops = scale_only ? 0 : 2LL * m * n * k * batch;

  std::vector<Operand> ops(3);
  ops[0] = {(void*)a, 8, sa, scale_only ? 0 : cm_extent(nrowa, ta == 0 ? k : m, lda), true, false};
  ops[1] = {(void*)b, 8, sb, scale_only ? 0 : cm_extent(nrowb, tb == 0 ? n : k, ldb), true, false};
  ops[2] = {(void*)c, 8, sc, cm_extent(m, n, ldc), beta != 0.0 || !dense(m, ldc, sc, n, batch), true};
  if (scale_only) ops[0].ptr = ops[1].ptr = nullptr;
  int rc = run_batched(routine, ops, batch, stream, res, 2,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         OutDesc o;
                         o.c = (const double*)p[2];
                         o.d = (double*)p[2];
                         o.sc = o.sd = sc;
                         o.ldc = o.ldd = ldc;
                         o.vec = aligned16(p[2]) && sc % 2 == 0 && ldc % 2 == 0;
                         if (scale_only) return scale_launch(0, o, m, n, beta, 0, nb, s);
                         // size switch (gemm.hpp:190-204): square packed NN problems up to 64
                         if (ta == 0 && tb == 0 && m == n && n == k &&
                             gemm_cm_ok(m, (const double*)p[0], (const double*)p[1], o.c, sa, sb, sc, lda, ldb, ldc))
                           return gemm_cm_launch(m, alpha, (const double*)p[0], (const double*)p[1], beta, o.d, nb, s);
                         // small-n branch (variant D's role): a warp per problem, no 64x64 tile padding
                         if (gemm_cmsmall_ok(m, n))
                           return gemm_cmsmall_launch(ta != 0, tb != 0, m, n, k, alpha, (const double*)p[0], lda, sa,
                                                      (const double*)p[1], ldb, sb, beta, o.d, ldc, sc, 0, nb, s);
                         GemmLaunch g;
                         // M side: op(A)(i, l); N side: op(B)(l, j) as (x = j, l).
                         g.lay_a = ta == 0 ? L_MNC : L_KC;
                         g.lay_b = tb == 0 ? L_KC : L_MNC;
                         g.a = cm_side(p[0], sa, lda, ta == 0, m, k);
                         g.b = cm_side(p[1], sb, ldb, tb == 1, n, k);
                         g.o = o;
                         g.m = m; g.n = n; g.k = k;
                         g.alpha = alpha; g.beta = beta;
                         g.batch = nb;
                         return gemm_launch(g, s);
                       });
  if (rc) return rc;
  return finish(res, 0, flops);
}

int pb_dgemm(char transa, char transb, int m, int n, int k, double alpha, const double* a, int lda,
             const double* b, int ldb, double beta, double* c, int ldc, pb_result* res) {
  return dgemm_impl("dgemm", false, transa, transb, m, n, k, alpha, a, lda, 0, b, ldb, 0, beta, c,
                    ldc, 0, 1, nullptr, res);
}

int pb_dgemm_batched(char transa, char transb, int m, int n, int k, double alpha, const double* a,
                     int lda, long long stride_a, const double* b, int ldb, long long stride_b,
                     double beta, double* c, int ldc, long long stride_c, int batch,
                     pb_stream stream, pb_result* res) {
  return dgemm_impl("dgemm", true, transa, transb, m, n, k, alpha, a, lda, stride_a, b, ldb,
                    stride_b, beta, c, ldc, stride_c, batch, stream, res);
}

// ============================================================== dsyrk family
static int dsyrk_impl(bool batched, char uplo, char trans, int n, int k, double alpha,
                      const double* a, int lda, long long sa, double beta, double* c, int ldc,
                      long long sc, int batch, pb_stream stream, pb_result* res) {
  const char* routine = "dsyrk";
  // blas.hpp:107-118
  int lo = parse_uplo(uplo);
  if (lo < 0) return fail(res, routine, 1, 1, "uplo is not one of u, l");
  int tr = parse_trans(trans);
  if (tr < 0) return fail(res, routine, 2, 2, "trans is not one of n, t, c");
  if (n < 0) return fail(res, routine, 3, 3, "n is negative");
  if (k < 0) return fail(res, routine, 4, 4, "k is negative");
  int nrowa = tr == 0 ? n : k;
  if (lda < std::max(1, nrowa)) return fail(res, routine, 7, 7, "lda is smaller than the rows of op(a)");
  if (ldc < std::max(1, n)) return fail(res, routine, 10, 10, "ldc is smaller than n");
  if (batched) {
    if (batch < 0) return fail(res, routine, 11, 11, "batch is negative");
    if (sa < 0 || sc < 0) return fail(res, routine, 12, 12, "a stride is negative");
  }
  if (n == 0 || batch == 0) return finish(res, 0, 0);
  if ((alpha == 0.0 || k == 0) && beta == 1.0) return finish(res, 0, 0);
  const bool scale_only = alpha == 0.0 || k == 0;  // level3.hpp:232-235
  long long flops = scale_only ? 0 : (long long)n * n * k * batch;
  std::vector<Operand> ops(2);
  ops[0] = {(void*)a, 8, sa, scale_only ? 0 : cm_extent(nrowa, tr == 0 ? k : n, lda), true, false};
  ops[1] = {(void*)c, 8, sc, cm_extent(n, n, ldc), true, true};
  if (scale_only) ops[0].ptr = nullptr;
  int rc = run_batched(routine, ops, batch, stream, res, 1,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         OutDesc o;
                         o.c = (const double*)p[1];
                         o.d = (double*)p[1];
                         o.sc = o.sd = sc;
                         o.ldc = o.ldd = ldc;
                         o.vec = aligned16(p[1]) && sc % 2 == 0 && ldc % 2 == 0;
                         int up = lo ? 1 : 2;
                         if (scale_only) return scale_launch(0, o, n, n, beta, up, nb, s);
                         // small-n branch: C = alpha op(A) op(A)^T + beta C on a warp per problem
                         if (gemm_cmsmall_ok(n, n))
                           return gemm_cmsmall_launch(tr != 0, tr == 0, n, n, k, alpha, (const double*)p[0], lda, sa,
                                                      (const double*)p[0], lda, sa, beta, o.d, ldc, sc, up, nb, s);
                         GemmLaunch g;
                         g.lay_a = g.lay_b = tr == 0 ? L_MNC : L_KC;
                         g.a = g.b = cm_side(p[0], sa, lda, tr == 0, n, k);
                         g.o = o;
                         g.m = g.n = n; g.k = k;
                         g.alpha = alpha; g.beta = beta;
                         g.uplo = up;
                         g.batch = nb;
                         return gemm_launch(g, s);
                       });
  if (rc) return rc;
  return finish(res, 0, flops);
}

int pb_dsyrk(char uplo, char trans, int n, int k, double alpha, const double* a, int lda,
             double beta, double* c, int ldc, pb_result* res) {
  return dsyrk_impl(false, uplo, trans, n, k, alpha, a, lda, 0, beta, c, ldc, 0, 1, nullptr, res);
}
int pb_dsyrk_batched(char uplo, char trans, int n, int k, double alpha, const double* a, int lda,
                     long long stride_a, double beta, double* c, int ldc, long long stride_c,
                     int batch, pb_stream stream, pb_result* res) {
  return dsyrk_impl(true, uplo, trans, n, k, alpha, a, lda, stride_a, beta, c, ldc, stride_c,
                    batch, stream, res);
}

// ============================================================== dtrsm family
static int dtrsm_impl(bool batched, char side, char uplo, char transa, char diag, int m, int n,
                      double alpha, const double* a, int lda, long long sa, double* b, int ldb,
                      long long sb, int* info, int batch, pb_stream stream, pb_result* res) {
  const char* routine = "dtrsm";
  // blas.hpp:139-157 (trimul_adapter)
  int sd = parse_side(side);
  if (sd < 0) return fail(res, routine, 1, 1, "side is not one of l, r");
  int lo = parse_uplo(uplo);
  if (lo < 0) return fail(res, routine, 2, 2, "uplo is not one of u, l");
  int tr = parse_trans(transa);
  if (tr < 0) return fail(res, routine, 3, 3, "transa is not one of n, t, c");
  int un = parse_diag(diag);
  if (un < 0) return fail(res, routine, 4, 4, "diag is not one of u, n");
  if (m < 0) return fail(res, routine, 5, 5, "m is negative");
  if (n < 0) return fail(res, routine, 6, 6, "n is negative");
  int nrowa = sd ? m : n;
  if (lda < std::max(1, nrowa)) return fail(res, routine, 9, 9, "lda is smaller than the triangle order");
  if (ldb < std::max(1, m)) return fail(res, routine, 11, 11, "ldb is smaller than m");
  if (batched) {
    if (batch < 0) return fail(res, routine, 12, 12, "batch is negative");
    if (sa < 0 || sb < 0) return fail(res, routine, 13, 13, "a stride is negative");
  }
  if (m == 0 || n == 0 || batch == 0) {
    if (batched && info && batch > 0 && kind_of(info) == K_HOST) std::fill(info, info + batch, 0);
    if (batched && info && batch > 0 && kind_of(info) == K_DEVICE)
      cudaMemsetAsync(info, 0, sizeof(int) * batch, (cudaStream_t)stream);
    return finish(res, 0, 0);
  }
  // Single calls report the zero-diagonal failure as the return value; the
  // batched form reports it per problem.
  InfoCell cell;
  int* infop = info;
  bool single = !batched;
  if (single) infop = &cell.host;
  long long flops = alpha == 0.0 ? 0 : (sd ? (long long)n * m * m : (long long)m * n * n) * batch;
  std::vector<Operand> ops(3);
  ops[0] = {(void*)a, 8, sa, alpha == 0.0 ? 0 : cm_extent(nrowa, nrowa, lda), true, false};
  if (alpha == 0.0) ops[0].ptr = nullptr;
  ops[1] = {(void*)b, 8, sb, cm_extent(m, n, ldb), alpha != 0.0 || !dense(m, ldb, sb, n, batch), true};
  ops[2] = {(void*)infop, 4, 1, 1, false, true};
  if (single && kind_of(b) == K_DEVICE) {
    if (cudaMalloc(&cell.dev, sizeof(int)) != cudaSuccess) return cuda_fail(res, routine, cudaGetLastError());
    ops[2].ptr = cell.dev;
  }
  int rc = run_batched(routine, ops, batch, stream, res, 1,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         if (alpha == 0.0) {  // level3.hpp:291: zeros, a never read
                           OutDesc o;
                           o.c = o.d = (double*)p[1];
                           o.sc = o.sd = sb;
                           o.ldc = o.ldd = ldb;
                           cudaError_t e = scale_launch(0, o, m, n, 0.0, 0, nb, s);
                           if (e != cudaSuccess) return e;
                           return cudaMemsetAsync(p[2], 0, sizeof(int) * nb, s);
                         }
                         TrsmLaunch L;
                         L.pm = 0;
                         L.twin = sd;
                         L.lower = lo;
                         L.trans = sd ? !tr : tr;  // Left = transposed right-side problem
                         L.unit = un;
                         L.mm = sd ? n : m;
                         L.nn = sd ? m : n;
                         L.alpha = alpha;
                         L.a = (const double*)p[0]; L.sa = sa; L.lda = lda;
                         L.b = (const double*)p[1]; L.sb = sb; L.ldb = ldb;
                         L.d = (double*)p[1]; L.sd = sb; L.ldd = ldb;
                         L.info = (int*)p[2];
                         L.batch = nb;
                         return trsm_launch(L, s);
                       });
  int single_info = 0;
  if (cell.dev) {
    if (!rc) cudaMemcpy(&single_info, cell.dev, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(cell.dev);
  } else if (single) {
    single_info = cell.host;
  }
  if (rc) return rc;
  if (single && single_info) return status(res, single_info, "triangular factor has an exactly zero diagonal");
  return finish(res, 0, flops);
}

int pb_dtrsm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
             const double* a, int lda, double* b, int ldb, pb_result* res) {
  return dtrsm_impl(false, side, uplo, transa, diag, m, n, alpha, a, lda, 0, b, ldb, 0, nullptr, 1,
                    nullptr, res);
}
int pb_dtrsm_batched(char side, char uplo, char transa, char diag, int m, int n, double alpha,
                     const double* a, int lda, long long stride_a, double* b, int ldb,
                     long long stride_b, int* info, int batch, pb_stream stream, pb_result* res) {
  return dtrsm_impl(true, side, uplo, transa, diag, m, n, alpha, a, lda, stride_a, b, ldb, stride_b,
                    info, batch, stream, res);
}

// ============================================================== dpotrf
static int dpotrf_impl(bool batched, char uplo, int n, double* a, int lda, long long sa, int* info,
                       int batch, pb_stream stream, pb_result* res) {
  const char* routine = "dpotrf";
  // blas.hpp:192-198: LAPACK convention, info = -index.
  int lo = parse_uplo(uplo);
  if (lo < 0) return fail(res, routine, 1, -1, "uplo is not one of u, l");
  if (n < 0) return fail(res, routine, 2, -2, "n is negative");
  if (lda < std::max(1, n)) return fail(res, routine, 4, -4, "lda is smaller than n");
  if (batched) {
    if (batch < 0) return fail(res, routine, 5, -5, "batch is negative");
    if (sa < 0) return fail(res, routine, 6, -6, "a stride is negative");
    if (!info && n > 0 && batch > 0) return fail(res, routine, 7, -7, "info is null");
  }
  long long flops = (long long)n * n * n / 3 * batch;  // factor.hpp:93
  if (n == 0 || batch == 0) {
    if (batched && info && batch > 0) {
      if (kind_of(info) == K_DEVICE) cudaMemsetAsync(info, 0, sizeof(int) * batch, (cudaStream_t)stream);
      else std::fill(info, info + batch, 0);
    }
    return finish(res, 0, 0);
  }
  InfoCell cell;
  int* infop = batched ? info : &cell.host;
  std::vector<Operand> ops(2);
  ops[0] = {(void*)a, 8, sa, cm_extent(n, n, lda), true, true};
  ops[1] = {(void*)infop, 4, 1, 1, false, true};
  if (!batched && kind_of(a) == K_DEVICE) {
    if (cudaMalloc(&cell.dev, sizeof(int)) != cudaSuccess) return cuda_fail(res, routine, cudaGetLastError());
    ops[1].ptr = cell.dev;
  }
  int rc = run_batched(routine, ops, batch, stream, res, 0,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         PotrfLaunch L;
                         L.a = (double*)p[0]; L.stride = sa; L.lda = lda; L.n = n;
                         L.upper = !lo;
                         L.info = (int*)p[1];
                         L.batch = nb;
                         return potrf_launch(L, s);
                       });
  int single_info = 0;
  if (cell.dev) {
    if (!rc) cudaMemcpy(&single_info, cell.dev, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(cell.dev);
  } else if (!batched) {
    single_info = cell.host;
  }
  if (rc) return rc;
  if (!batched && single_info) return numerical(res, single_info, "matrix is not positive definite", flops);
  return finish(res, 0, flops);
}

int pb_dpotrf(char uplo, int n, double* a, int lda, pb_result* res) {
  return dpotrf_impl(false, uplo, n, a, lda, 0, nullptr, 1, nullptr, res);
}
int pb_dpotrf_batched(char uplo, int n, double* a, int lda, long long stride_a, int* info,
                      int batch, pb_stream stream, pb_result* res) {
  return dpotrf_impl(true, uplo, n, a, lda, stride_a, info, batch, stream, res);
}

// ============================================================== dgetrf
static int dgetrf_impl(bool batched, int m, int n, double* a, int lda, long long sa, int* ipiv,
                       long long sp, int* info, int batch, pb_stream stream, pb_result* res) {
  const char* routine = "dgetrf";
  // blas.hpp:206-211
  if (m < 0) return fail(res, routine, 1, -1, "m is negative");
  if (n < 0) return fail(res, routine, 2, -2, "n is negative");
  if (lda < std::max(1, m)) return fail(res, routine, 4, -4, "lda is smaller than m");
  int minmn = std::min(m, n);
  if (batched) {
    if (batch < 0) return fail(res, routine, 7, -7, "batch is negative");
    if (sa < 0 || sp < minmn) return fail(res, routine, 8, -8, "a stride is negative or ipiv stride below min(m, n)");
    if (!ipiv && minmn > 0 && batch > 0) return fail(res, routine, 9, -9, "ipiv is null");
    if (!info && minmn > 0 && batch > 0) return fail(res, routine, 10, -10, "info is null");
  }
  // BlasResult.flops of the reference (factor.hpp:222-223): n^2 m - n^3/3
  long long flops = ((long long)n * n * m - (long long)n * n * n / 3) * batch;
  if (minmn == 0 || batch == 0) {
    if (batched && info && batch > 0) {
      if (kind_of(info) == K_DEVICE) cudaMemsetAsync(info, 0, sizeof(int) * batch, (cudaStream_t)stream);
      else std::fill(info, info + batch, 0);
    }
    return finish(res, 0, 0);
  }
  InfoCell cell;
  int* infop = batched ? info : &cell.host;
  std::vector<Operand> ops(3);
  ops[0] = {(void*)a, 8, sa, cm_extent(m, n, lda), true, true};
  // ipiv rows with gaps (stride > min(m, n)) are staged in too, so the
  // entries between problems survive the host round trip
  ops[1] = {(void*)ipiv, 4, batched ? sp : minmn, minmn, batched && sp != minmn, true};
  ops[2] = {(void*)infop, 4, 1, 1, false, true};
  if (!batched && kind_of(a) == K_DEVICE) {
    if (cudaMalloc(&cell.dev, sizeof(int)) != cudaSuccess) return cuda_fail(res, routine, cudaGetLastError());
    ops[2].ptr = cell.dev;
  }
  long long spv = batched ? sp : minmn;
  int rc = run_batched(routine, ops, batch, stream, res, 0,
                       [&](const std::vector<void*>& pt, int nb, cudaStream_t s) -> cudaError_t {
                         GetrfLaunch L;
                         L.a = (double*)pt[0]; L.stride = sa; L.lda = lda; L.m = m; L.n = n;
                         L.ipiv = (int*)pt[1]; L.stride_ipiv = spv;
                         L.info = (int*)pt[2];
                         L.batch = nb;
                         return getrf_launch(L, s);
                       });
  int single_info = 0;
  if (cell.dev) {
    if (!rc) cudaMemcpy(&single_info, cell.dev, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(cell.dev);
  } else if (!batched) {
    single_info = cell.host;
  }
  if (rc) return rc;
  if (!batched && single_info) return numerical(res, single_info, "factor has an exactly zero pivot", flops);
  return finish(res, 0, flops);
}

int pb_dgetrf(int m, int n, double* a, int lda, int* ipiv, pb_result* res) {
  return dgetrf_impl(false, m, n, a, lda, 0, ipiv, 0, nullptr, 1, nullptr, res);
}
int pb_dgetrf_batched(int m, int n, double* a, int lda, long long stride_a, int* ipiv,
                      long long stride_ipiv, int* info, int batch, pb_stream stream,
                      pb_result* res) {
  return dgetrf_impl(true, m, n, a, lda, stride_a, ipiv, stride_ipiv, info, batch, stream, res);
}

// ============================================================== panel-major
static bool panel_ok(const pb_dmat& r, int m, int n) {  // level3.hpp:327-333
  return r.data != nullptr && r.ps == 4 && r.m == m && r.n == n;
}
static OpDesc pm_side(const void* base, long long stride, int cn) {
  OpDesc d;
  d.base = (const double*)base;
  d.stride = stride;
  d.ld = cn;
  d.bulk = aligned16(base) && stride % 2 == 0;
  return d;
}

static int gemm_nd_impl(bool batched, char transa, char transb, int m, int n, int k, double alpha,
                        pb_dmat a, long long sa, pb_dmat b, long long sb, double beta, pb_dmat c,
                        long long sc, pb_dmat d, long long sd, int batch, pb_stream stream,
                        pb_result* res) {
  int ta = parse_trans(transa), tb = parse_trans(transb);
  if (ta != 0) return status(res, PB_INFO_UNSUPPORTED, "native gemm requires untransposed a");
  if (tb < 0) return status(res, PB_INFO_UNSUPPORTED, "transb is not one of n, t, c");
  if (m < 0) return status(res, -4, "m < 0");
  if (n < 0) return status(res, -5, "n < 0");
  if (k < 0) return status(res, -6, "k < 0");
  int bm = tb == 0 ? k : n, bn = tb == 0 ? n : k;
  if (!panel_ok(a, m, k)) return status(res, -8, "a panel mismatch");
  if (!panel_ok(b, bm, bn)) return status(res, -9, "b panel mismatch");
  if (!panel_ok(c, m, n)) return status(res, -11, "c panel mismatch");
  if (!panel_ok(d, m, n)) return status(res, -12, "d panel mismatch");
  if (batched && batch < 0) return status(res, -17, "batch is negative");
  if (m == 0 || n == 0 || batch == 0) return finish(res, 0, 0);
  const bool scale_only = alpha == 0.0 || k == 0;
  long long flops = scale_only ? 0 : 2LL * m * n * k * batch;
  const bool alias = c.data == d.data && sc == sd;
  std::vector<Operand> ops(4);
  ops[0] = {(void*)a.data, 8, sa, scale_only ? 0 : pm_extent(a), true, false};
  ops[1] = {(void*)b.data, 8, sb, scale_only ? 0 : pm_extent(b), true, false};
  ops[2] = {(void*)c.data, 8, sc, pm_extent(c), beta != 0.0, false};
  ops[3] = {(void*)d.data, 8, sd, pm_extent(d), true, true};  // pad lanes must survive the round trip
  if (scale_only) ops[0].ptr = ops[1].ptr = nullptr;
  if (alias || beta == 0.0) ops[2].ptr = nullptr;
  int rc = run_batched("gemm_nd", ops, batch, stream, res, 3,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         OutDesc o;
                         o.d = (double*)p[3];
                         o.c = alias ? (const double*)p[3] : (p[2] ? (const double*)p[2] : o.d);
                         o.sc = sc; o.sd = sd;
                         o.ldc = c.cn; o.ldd = d.cn;
                         o.vec = aligned16(o.c) && aligned16(o.d) && sc % 2 == 0 && sd % 2 == 0;
                         if (scale_only) return scale_launch(1, o, m, n, beta, 0, nb, s);
                         // size switch (gemm.hpp:190-204): tiny square NT problems stream in chunks
                         if (tb == 1 && m == n && n == k && !alias &&
                             gemm_small_ok(m, (const double*)p[0], (const double*)p[1], o.c, o.d, sa, sb, sc, sd,
                                           a.cn, b.cn, c.cn, d.cn))
                           return gemm_small_launch(m, alpha, (const double*)p[0], (const double*)p[1], beta, o.c,
                                                    o.d, nb, s);
                         GemmLaunch g;
                         g.out_pm = 1;
                         g.lay_a = L_PMX;
                         g.lay_b = tb == 1 ? L_PMX : L_PML;
                         g.a = pm_side(p[0], sa, a.cn);
                         g.b = pm_side(p[1], sb, b.cn);
                         g.o = o;
                         g.m = m; g.n = n; g.k = k;
                         g.alpha = alpha; g.beta = beta;
                         g.batch = nb;
                         return gemm_launch(g, s);
                       });
  if (rc) return rc;
  return finish(res, 0, flops);
}

int pb_gemm_nd(char transa, char transb, int m, int n, int k, double alpha, pb_dmat a, pb_dmat b,
               double beta, pb_dmat c, pb_dmat d, pb_result* res) {
  return gemm_nd_impl(false, transa, transb, m, n, k, alpha, a, 0, b, 0, beta, c, 0, d, 0, 1,
                      nullptr, res);
}
int pb_gemm_nd_batched(char transa, char transb, int m, int n, int k, double alpha, pb_dmat a,
                       long long stride_a, pb_dmat b, long long stride_b, double beta, pb_dmat c,
                       long long stride_c, pb_dmat d, long long stride_d, int batch,
                       pb_stream stream, pb_result* res) {
  return gemm_nd_impl(true, transa, transb, m, n, k, alpha, a, stride_a, b, stride_b, beta, c,
                      stride_c, d, stride_d, batch, stream, res);
}

static int syrk_nd_impl(bool batched, int n, int k, double alpha, pb_dmat a, long long sa,
                        double beta, pb_dmat c, long long sc, pb_dmat d, long long sd, int batch,
                        pb_stream stream, pb_result* res) {
  if (n < 0) return status(res, -2, "n < 0");
  if (k < 0) return status(res, -3, "k < 0");
  if (!panel_ok(a, n, k)) return status(res, -5, "a panel mismatch");
  if (!panel_ok(c, n, n)) return status(res, -7, "c panel mismatch");
  if (!panel_ok(d, n, n)) return status(res, -8, "d panel mismatch");
  if (batched && batch < 0) return status(res, -12, "batch is negative");
  if (n == 0 || batch == 0) return finish(res, 0, 0);
  const bool scale_only = alpha == 0.0 || k == 0;
  long long flops = scale_only ? 0 : (long long)n * n * k * batch;
  const bool alias = c.data == d.data && sc == sd;
  std::vector<Operand> ops(3);
  ops[0] = {(void*)a.data, 8, sa, scale_only ? 0 : pm_extent(a), true, false};
  ops[1] = {(void*)c.data, 8, sc, pm_extent(c), beta != 0.0, false};
  ops[2] = {(void*)d.data, 8, sd, pm_extent(d), true, true};
  if (scale_only) ops[0].ptr = nullptr;
  if (alias || beta == 0.0) ops[1].ptr = nullptr;
  int rc = run_batched("syrk_nd", ops, batch, stream, res, 2,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         OutDesc o;
                         o.d = (double*)p[2];
                         o.c = alias ? (const double*)p[2] : (p[1] ? (const double*)p[1] : o.d);
                         o.sc = sc; o.sd = sd;
                         o.ldc = c.cn; o.ldd = d.cn;
                         o.vec = aligned16(o.c) && aligned16(o.d) && sc % 2 == 0 && sd % 2 == 0;
                         if (scale_only) return scale_launch(1, o, n, n, beta, 1, nb, s);
                         GemmLaunch g;
                         g.out_pm = 1;
                         g.lay_a = g.lay_b = L_PMX;
                         g.a = g.b = pm_side(p[0], sa, a.cn);
                         g.o = o;
                         g.m = g.n = n; g.k = k;
                         g.alpha = alpha; g.beta = beta;
                         g.uplo = 1;
                         g.batch = nb;
                         return gemm_launch(g, s);
                       });
  if (rc) return rc;
  return finish(res, 0, flops);
}

int pb_syrk_nd(int n, int k, double alpha, pb_dmat a, double beta, pb_dmat c, pb_dmat d,
               pb_result* res) {
  return syrk_nd_impl(false, n, k, alpha, a, 0, beta, c, 0, d, 0, 1, nullptr, res);
}
int pb_syrk_nd_batched(int n, int k, double alpha, pb_dmat a, long long stride_a, double beta,
                       pb_dmat c, long long stride_c, pb_dmat d, long long stride_d, int batch,
                       pb_stream stream, pb_result* res) {
  return syrk_nd_impl(true, n, k, alpha, a, stride_a, beta, c, stride_c, d, stride_d, batch, stream,
                      res);
}

static int trsm_rltn_nd_impl(bool batched, int m, int n, double alpha, pb_dmat a, long long sa,
                             pb_dmat b, long long sb, pb_dmat d, long long sd, int* info, int batch,
                             pb_stream stream, pb_result* res) {
  if (m < 0) return status(res, -2, "m < 0");
  if (n < 0) return status(res, -3, "n < 0");
  if (!panel_ok(a, n, n)) return status(res, -5, "a panel mismatch");
  if (!panel_ok(b, m, n)) return status(res, -6, "b panel mismatch");
  if (!panel_ok(d, m, n)) return status(res, -7, "d panel mismatch");
  if (batched && batch < 0) return status(res, -12, "batch is negative");
  if (m == 0 || n == 0 || batch == 0) {
    if (batched && info && batch > 0) {
      if (kind_of(info) == K_DEVICE) cudaMemsetAsync(info, 0, sizeof(int) * batch, (cudaStream_t)stream);
      else std::fill(info, info + batch, 0);
    }
    return finish(res, 0, 0);
  }
  InfoCell cell;
  int* infop = batched ? info : &cell.host;
  const bool alias = b.data == d.data && sb == sd;
  std::vector<Operand> ops(4);
  ops[0] = {(void*)a.data, 8, sa, pm_extent(a), true, false};
  ops[1] = {(void*)b.data, 8, sb, pm_extent(b), alpha != 0.0, false};
  ops[2] = {(void*)d.data, 8, sd, pm_extent(d), true, true};
  ops[3] = {(void*)infop, 4, 1, 1, false, true};
  if (alias) ops[1].ptr = nullptr;
  if (!batched && kind_of(d.data) == K_DEVICE) {
    if (cudaMalloc(&cell.dev, sizeof(int)) != cudaSuccess) return cuda_fail(res, "trsm_rltn_nd", cudaGetLastError());
    ops[3].ptr = cell.dev;
  }
  int rc = run_batched("trsm_rltn_nd", ops, batch, stream, res, 2,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         TrsmLaunch L;
                         L.pm = 1;
                         L.lower = 1; L.trans = 1; L.unit = 0;
                         L.mm = m; L.nn = n;
                         L.alpha = alpha;
                         L.a = (const double*)p[0]; L.sa = sa; L.lda = a.cn;
                         L.d = (double*)p[2]; L.sd = sd; L.ldd = d.cn;
                         L.b = alias ? L.d : (const double*)p[1]; L.sb = sb; L.ldb = b.cn;
                         L.info = (int*)p[3];
                         L.batch = nb;
                         if (alpha == 0.0) return trsm_nd_zero_launch(L, s);  // level3.hpp:493-504
                         return trsm_launch(L, s);
                       });
  int single_info = 0;
  if (cell.dev) {
    if (!rc) cudaMemcpy(&single_info, cell.dev, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(cell.dev);
  } else if (!batched) {
    single_info = cell.host;
  }
  if (rc) return rc;
  if (!batched && single_info) return status(res, single_info, "triangular factor has an exactly zero diagonal");
  return finish(res, 0, alpha == 0.0 ? 0 : (long long)m * n * n * batch);
}

int pb_trsm_rltn_nd(int m, int n, double alpha, pb_dmat a, pb_dmat b, pb_dmat d, pb_result* res) {
  return trsm_rltn_nd_impl(false, m, n, alpha, a, 0, b, 0, d, 0, nullptr, 1, nullptr, res);
}
int pb_trsm_rltn_nd_batched(int m, int n, double alpha, pb_dmat a, long long stride_a, pb_dmat b,
                            long long stride_b, pb_dmat d, long long stride_d, int* info,
                            int batch, pb_stream stream, pb_result* res) {
  return trsm_rltn_nd_impl(true, m, n, alpha, a, stride_a, b, stride_b, d, stride_d, info, batch,
                           stream, res);
}

static int syrk_potrf_nd_impl(bool batched, int n, int k, pb_dmat a, long long sa, pb_dmat b,
                              long long sb, pb_dmat c, long long sc, pb_dmat d, long long sd,
                              int* info, int batch, pb_stream stream, pb_result* res) {
  if (n < 0) return status(res, -2, "n < 0");
  if (k < 0) return status(res, -3, "k < 0");
  if (!panel_ok(a, n, k)) return status(res, -4, "a panel mismatch");
  if (!panel_ok(b, n, k)) return status(res, -5, "b panel mismatch");
  if (!panel_ok(c, n, n)) return status(res, -6, "c panel mismatch");
  if (!panel_ok(d, n, n)) return status(res, -7, "d panel mismatch");
  if (batched && batch < 0) return status(res, -13, "batch is negative");
  if (batched && !info && n > 0 && batch > 0) return status(res, -14, "info is null");
  if (n == 0 || batch == 0) {
    if (batched && info && batch > 0) {
      if (kind_of(info) == K_DEVICE) cudaMemsetAsync(info, 0, sizeof(int) * batch, (cudaStream_t)stream);
      else std::fill(info, info + batch, 0);
    }
    return finish(res, 0, 0);
  }
  InfoCell cell;
  int* infop = batched ? info : &cell.host;
  const bool alias = c.data == d.data && sc == sd;
  std::vector<Operand> ops(5);
  ops[0] = {(void*)a.data, 8, sa, k ? pm_extent(a) : 0, true, false};
  ops[1] = {(void*)b.data, 8, sb, k ? pm_extent(b) : 0, true, false};
  ops[2] = {(void*)c.data, 8, sc, pm_extent(c), true, false};
  ops[3] = {(void*)d.data, 8, sd, pm_extent(d), true, true};
  ops[4] = {(void*)infop, 4, 1, 1, false, true};
  if (!k) ops[0].ptr = ops[1].ptr = nullptr;
  if (alias) ops[2].ptr = nullptr;
  if (!batched && kind_of(d.data) == K_DEVICE) {
    if (cudaMalloc(&cell.dev, sizeof(int)) != cudaSuccess) return cuda_fail(res, "syrk_potrf_nd", cudaGetLastError());
    ops[4].ptr = cell.dev;
  }
  int rc = run_batched("syrk_potrf_nd", ops, batch, stream, res, 3,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         SyrkPotrfLaunch L;
                         L.a = (const double*)p[0]; L.sa = sa; L.cna = a.cn;
                         L.b = (const double*)p[1]; L.sb = sb; L.cnb = b.cn;
                         L.d = (double*)p[3]; L.sd = sd; L.cnd = d.cn;
                         L.c = alias ? L.d : (const double*)p[2]; L.sc = sc; L.cnc = c.cn;
                         L.n = n; L.k = k;
                         L.info = (int*)p[4];
                         L.batch = nb;
                         return syrk_potrf_launch(L, s);
                       });
  int single_info = 0;
  if (cell.dev) {
    if (!rc) cudaMemcpy(&single_info, cell.dev, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(cell.dev);
  } else if (!batched) {
    single_info = cell.host;
  }
  if (rc) return rc;
  if (!batched && single_info) return status(res, single_info, "updated matrix is not positive definite");
  return finish(res, 0, ((long long)n * n * n / 3 + (long long)n * n * k) * batch);  // level3.hpp:572-573
}

int pb_syrk_potrf_nd(int n, int k, pb_dmat a, pb_dmat b, pb_dmat c, pb_dmat d, pb_result* res) {
  return syrk_potrf_nd_impl(false, n, k, a, 0, b, 0, c, 0, d, 0, nullptr, 1, nullptr, res);
}
int pb_syrk_potrf_nd_batched(int n, int k, pb_dmat a, long long stride_a, pb_dmat b,
                             long long stride_b, pb_dmat c, long long stride_c, pb_dmat d,
                             long long stride_d, int* info, int batch, pb_stream stream,
                             pb_result* res) {
  return syrk_potrf_nd_impl(true, n, k, a, stride_a, b, stride_b, c, stride_c, d, stride_d, info,
                            batch, stream, res);
}

// ============================================================== chain (cfg 5)
int pb_chain_vbatched(char layout, const int* n, const long long* offset, double* A, double* C,
                      double* B, int* info, int batch, int max_n, pb_stream stream,
                      pb_result* res) {
  const char* routine = "chain";
  int pm;
  if (layout == 'C' || layout == 'c') pm = 0;
  else if (layout == 'P' || layout == 'p') pm = 1;
  else return fail(res, routine, 1, 1, "layout is not one of C, P");
  if (batch < 0) return fail(res, routine, 9, 9, "batch is negative");
  if (max_n < 0) return fail(res, routine, 10, 10, "max_n is negative");
  if (batch == 0) return finish(res, 0, 0);
  if (!device_ok()) return status(res, PB_INFO_NO_DEVICE, "no CUDA device: pbgpu has no CPU path");
  // Memory kinds: everything on the device (asynchronous; the split by order costs
  // one device -> host copy of n / offset), n / offset on the host with the
  // matrices on the device (asynchronous, no synchronisation), or everything on
  // the host (staged through the device; returns when done).
  const Kind kd = kind_of(A);
  if (kd == K_NONE || kind_of(C) != kd || kind_of(B) != kd || kind_of(info) != kd)
    return status(res, PB_INFO_UNSUPPORTED, "A, C, B and info must be all device or all host pointers");
  const Kind kn = kind_of(n);
  if (kn == K_NONE || kind_of(offset) != kn || (kd == K_HOST && kn != K_HOST))
    return status(res, PB_INFO_UNSUPPORTED, "n and offset must share one memory kind (host with host matrices)");
  cudaStream_t s = (cudaStream_t)stream;
  if (kd == K_HOST) cudaStreamSynchronize(s);  // earlier work on the caller's stream (ADVICE: host calls)
  mempool_keep();
  ChainLaunch L;
  L.pm = pm;
  L.batch = batch; L.max_n = max_n;
  std::vector<void*> scratch;
  auto dalloc = [&](size_t bytes) -> void* {
    void* q = nullptr;
    if (cudaMallocAsync(&q, std::max<size_t>(bytes, 16), s) != cudaSuccess) return nullptr;
    scratch.push_back(q);
    return q;
  };
  cudaError_t e = cudaSuccess;
  long long extent = 0;  // doubles spanned by the matrices (host matrices only)
  if (kn == K_HOST) {
    for (int p = 0; p < batch; ++p) {
      if (n[p] < 0 || n[p] > max_n) return fail(res, routine, 2, 2, "n[p] is negative or above max_n");
      if (offset[p] < 0) return fail(res, routine, 3, 3, "offset[p] is negative");
      extent = std::max(extent, offset[p] + (long long)n[p] * n[p]);
    }
    int* dn = (int*)dalloc(sizeof(int) * batch);
    long long* doff = (long long*)dalloc(sizeof(long long) * batch);
    if (!dn || !doff) e = cudaErrorMemoryAllocation;
    if (e == cudaSuccess) e = cudaMemcpyAsync(dn, n, sizeof(int) * batch, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(doff, offset, sizeof(long long) * batch, cudaMemcpyHostToDevice, s);
    L.n = dn; L.offset = doff;
    L.n_host = n; L.offset_host = offset;
  } else {
    L.n = n; L.offset = offset;
  }
  double *dA = A, *dC = C, *dB = B;
  int* dinfo = info;
  if (e == cudaSuccess && kd == K_HOST) {
    const size_t bytes = sizeof(double) * (size_t)extent;
    dA = (double*)dalloc(bytes); dC = (double*)dalloc(bytes); dB = (double*)dalloc(bytes);
    dinfo = (int*)dalloc(sizeof(int) * batch);
    if (!dA || !dC || !dB || !dinfo) e = cudaErrorMemoryAllocation;
    if (e == cudaSuccess) e = cudaMemcpyAsync(dA, A, bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dC, C, bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dB, B, bytes, cudaMemcpyHostToDevice, s);
  }
  L.A = dA; L.C = dC; L.B = dB;
  L.info = dinfo;
  if (e == cudaSuccess) e = chain_launch(L, s);
  if (e == cudaSuccess && mutation_epsilon() != 0.0)
    e = mutate_launch(dB, 0, L.offset, batch, mutation_epsilon(), s);
  if (e == cudaSuccess && kd == K_HOST) {
    const size_t bytes = sizeof(double) * (size_t)extent;
    e = cudaMemcpyAsync(C, dC, bytes, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(B, dB, bytes, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(info, dinfo, sizeof(int) * batch, cudaMemcpyDeviceToHost, s);
  }
  for (void* q : scratch) cudaFreeAsync(q, s);
  if (e == cudaSuccess && kd == K_HOST) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(res, routine, e);
  return finish(res, 0, 0);
}


// ============================================================== dtrmm
// blas.hpp:166-176: the trimul adapter shared with dtrsm (blas.hpp:132-162),
// same validation order and positions; level3.hpp:250-275 underneath.
static int dtrmm_impl(bool batched, char side, char uplo, char transa, char diag, int m, int n,
                      double alpha, const double* a, int lda, long long sa, double* b, int ldb,
                      long long sb, int batch, pb_stream stream, pb_result* res) {
  const char* routine = "dtrmm";
  int sd = parse_side(side);
  if (sd < 0) return fail(res, routine, 1, 1, "side is not one of l, r");
  int lo = parse_uplo(uplo);
  if (lo < 0) return fail(res, routine, 2, 2, "uplo is not one of u, l");
  int tr = parse_trans(transa);
  if (tr < 0) return fail(res, routine, 3, 3, "transa is not one of n, t, c");
  int un = parse_diag(diag);
  if (un < 0) return fail(res, routine, 4, 4, "diag is not one of u, n");
  if (m < 0) return fail(res, routine, 5, 5, "m is negative");
  if (n < 0) return fail(res, routine, 6, 6, "n is negative");
  int nrowa = sd ? m : n;
  if (lda < std::max(1, nrowa)) return fail(res, routine, 9, 9, "lda is smaller than the triangle order");
  if (ldb < std::max(1, m)) return fail(res, routine, 11, 11, "ldb is smaller than m");
  if (batched) {
    if (batch < 0) return fail(res, routine, 12, 12, "batch is negative");
    if (sa < 0 || sb < 0) return fail(res, routine, 13, 13, "a stride is negative");
  }
  if (m == 0 || n == 0 || batch == 0) return finish(res, 0, 0);
  const long long flops = alpha == 0.0 ? 0 : (sd ? (long long)n * m * m : (long long)m * n * n) * batch;
  std::vector<Operand> ops(2);
  ops[0] = {(void*)a, 8, sa, alpha == 0.0 ? 0 : cm_extent(nrowa, nrowa, lda), true, false};
  if (alpha == 0.0) ops[0].ptr = nullptr;
  ops[1] = {(void*)b, 8, sb, cm_extent(m, n, ldb), alpha != 0.0 || !dense(m, ldb, sb, n, batch), true};
  int rc = run_batched(routine, ops, batch, stream, res, 1,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         if (alpha == 0.0) {  // level3.hpp:261: scale_only, zeros, a never read
                           OutDesc o;
                           o.c = o.d = (double*)p[1];
                           o.sc = o.sd = sb;
                           o.ldc = o.ldd = ldb;
                           return scale_launch(0, o, m, n, 0.0, 0, nb, s);
                         }
                         TrsmLaunch L;
                         L.pm = 0;
                         L.twin = sd;
                         L.lower = lo;
                         L.trans = sd ? !tr : tr;  // Left = transposed right-side problem (level3.hpp:263-265)
                         L.unit = un;
                         L.mm = sd ? n : m;
                         L.nn = sd ? m : n;
                         L.alpha = alpha;
                         L.a = (const double*)p[0]; L.sa = sa; L.lda = lda;
                         L.b = (const double*)p[1]; L.sb = sb; L.ldb = ldb;
                         L.d = (double*)p[1]; L.sd = sb; L.ldd = ldb;
                         L.batch = nb;
                         return trmm_launch(L, s);
                       });
  if (rc) return rc;
  return finish(res, 0, flops);
}

int pb_dtrmm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
             const double* a, int lda, double* b, int ldb, pb_result* res) {
  return dtrmm_impl(false, side, uplo, transa, diag, m, n, alpha, a, lda, 0, b, ldb, 0, 1, nullptr, res);
}
int pb_dtrmm_batched(char side, char uplo, char transa, char diag, int m, int n, double alpha,
                     const double* a, int lda, long long stride_a, double* b, int ldb,
                     long long stride_b, int batch, pb_stream stream, pb_result* res) {
  return dtrmm_impl(true, side, uplo, transa, diag, m, n, alpha, a, lda, stride_a, b, ldb, stride_b,
                    batch, stream, res);
}

// ============================================================== trmm_rlnn_nd
// level3.hpp:446-479: d <- alpha * b * a, a lower non-unit untransposed; b may alias d.
static int trmm_rlnn_nd_impl(bool batched, int m, int n, double alpha, pb_dmat a, long long sa,
                             pb_dmat b, long long sb, pb_dmat d, long long sd, int batch,
                             pb_stream stream, pb_result* res) {
  if (m < 0) return status(res, -2, "m < 0");
  if (n < 0) return status(res, -3, "n < 0");
  if (!panel_ok(a, n, n)) return status(res, -5, "a panel mismatch");
  if (!panel_ok(b, m, n)) return status(res, -6, "b panel mismatch");
  if (!panel_ok(d, m, n)) return status(res, -7, "d panel mismatch");
  if (batched && batch < 0) return status(res, -11, "batch is negative");
  if (m == 0 || n == 0 || batch == 0) return finish(res, 0, 0);
  const bool alias = b.data == d.data && sb == sd;
  std::vector<Operand> ops(3);
  ops[0] = {(void*)a.data, 8, sa, alpha == 0.0 ? 0 : pm_extent(a), true, false};
  ops[1] = {(void*)b.data, 8, sb, pm_extent(b), alpha != 0.0, false};
  ops[2] = {(void*)d.data, 8, sd, pm_extent(d), true, true};  // pad lanes survive the round trip
  if (alpha == 0.0) ops[0].ptr = ops[1].ptr = nullptr;
  if (alias) ops[1].ptr = nullptr;
  int rc = run_batched("trmm_rlnn_nd", ops, batch, stream, res, 2,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         if (alpha == 0.0) {  // scale_tiles_nd(beta = 0): +0, b never read
                           OutDesc o;
                           o.c = o.d = (double*)p[2];
                           o.sc = o.sd = sd;
                           o.ldc = o.ldd = d.cn;
                           return scale_launch(1, o, m, n, 0.0, 0, nb, s);
                         }
                         TrsmLaunch L;
                         L.pm = 1;
                         L.lower = 1; L.trans = 0; L.unit = 0;
                         L.mm = m; L.nn = n;
                         L.alpha = alpha;
                         L.a = (const double*)p[0]; L.sa = sa; L.lda = a.cn;
                         L.d = (double*)p[2]; L.sd = sd; L.ldd = d.cn;
                         L.b = alias ? L.d : (const double*)p[1]; L.sb = sb; L.ldb = b.cn;
                         L.batch = nb;
                         return trmm_launch(L, s);
                       });
  if (rc) return rc;
  return finish(res, 0, alpha == 0.0 ? 0 : (long long)m * n * n * batch);
}

int pb_trmm_rlnn_nd(int m, int n, double alpha, pb_dmat a, pb_dmat b, pb_dmat d, pb_result* res) {
  return trmm_rlnn_nd_impl(false, m, n, alpha, a, 0, b, 0, d, 0, 1, nullptr, res);
}
int pb_trmm_rlnn_nd_batched(int m, int n, double alpha, pb_dmat a, long long stride_a, pb_dmat b,
                            long long stride_b, pb_dmat d, long long stride_d, int batch,
                            pb_stream stream, pb_result* res) {
  return trmm_rlnn_nd_impl(true, m, n, alpha, a, stride_a, b, stride_b, d, stride_d, batch, stream, res);
}

// ============================================================== pack / unpack
// panel_mat.hpp:45-48
long long pb_memsize(int m, int n, int ps) {
  if (m <= 0 || n <= 0 || ps <= 0) return 0;
  return (long long)((m + ps - 1) / ps * ps) * ((n + ps - 1) / ps * ps) * (long long)sizeof(double);
}

static bool dmat_shape_ok(const pb_dmat& d) {
  return d.data && d.ps > 0 && d.m >= 0 && d.n >= 0 && d.pm == (d.m + d.ps - 1) / d.ps * d.ps &&
         d.cn == (d.n + d.ps - 1) / d.ps * d.ps;
}

// panel_mat.hpp:141-160: d <- packed op(a); op(a) is d.m x d.n; pad lanes untouched.
static int pack_impl(bool batched, char trans, const double* a, int lda, long long sa, pb_dmat d,
                     long long sd, int batch, pb_stream stream, pb_result* res) {
  const char* routine = "pack_from_colmajor";
  int tr = parse_trans(trans);
  if (tr < 0) return fail(res, routine, 1, 1, "trans is not one of n, t, c");
  if (!dmat_shape_ok(d)) return fail(res, routine, 4, 4, "destination is not a consistent panel descriptor");
  const int rows = tr ? d.n : d.m, cols = tr ? d.m : d.n;
  if (lda < std::max(1, rows)) return fail(res, routine, 3, 3, "lda is smaller than the rows of a");
  if (batched) {
    if (batch < 0) return fail(res, routine, 6, 6, "batch is negative");
    if (sa < 0 || sd < 0) return fail(res, routine, 7, 7, "a stride is negative");
  }
  if (d.m == 0 || d.n == 0 || batch == 0) return finish(res, 0, 0);
  std::vector<Operand> ops(2);
  ops[0] = {(void*)a, 8, sa, cm_extent(rows, cols, lda), true, false};
  ops[1] = {(void*)d.data, 8, sd, (long long)d.pm * d.cn, true, true};  // pad lanes survive
  int rc = run_batched(routine, ops, batch, stream, res, -1,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         return pack_launch(tr, d.m, d.n, (const double*)p[0], lda, sa, (double*)p[1], d.ps,
                                            d.cn, sd, nb, s);
                       });
  if (rc) return rc;
  return finish(res, 0, 0);
}

// panel_mat.hpp:164-171: a <- unpacked s; only the m x n interior is read.
static int unpack_impl(bool batched, pb_dmat src, long long ss, double* a, int lda, long long sa,
                       int batch, pb_stream stream, pb_result* res) {
  const char* routine = "unpack_to_colmajor";
  if (!dmat_shape_ok(src)) return fail(res, routine, 1, 1, "source is not a consistent panel descriptor");
  if (lda < std::max(1, src.m)) return fail(res, routine, 3, 3, "lda is smaller than m");
  if (batched) {
    if (batch < 0) return fail(res, routine, 5, 5, "batch is negative");
    if (ss < 0 || sa < 0) return fail(res, routine, 6, 6, "a stride is negative");
  }
  if (src.m == 0 || src.n == 0 || batch == 0) return finish(res, 0, 0);
  std::vector<Operand> ops(2);
  ops[0] = {(void*)src.data, 8, ss, (long long)src.pm * src.cn, true, false};
  ops[1] = {(void*)a, 8, sa, cm_extent(src.m, src.n, lda), !dense(src.m, lda, sa, src.n, batch), true};
  int rc = run_batched(routine, ops, batch, stream, res, -1,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         return unpack_launch(src.m, src.n, (const double*)p[0], src.ps, src.cn, ss,
                                              (double*)p[1], lda, sa, nb, s);
                       });
  if (rc) return rc;
  return finish(res, 0, 0);
}

int pb_pack(char trans, const double* a, int lda, pb_dmat d, pb_result* res) {
  return pack_impl(false, trans, a, lda, 0, d, 0, 1, nullptr, res);
}
int pb_pack_batched(char trans, const double* a, int lda, long long stride_a, pb_dmat d,
                    long long stride_d, int batch, pb_stream stream, pb_result* res) {
  return pack_impl(true, trans, a, lda, stride_a, d, stride_d, batch, stream, res);
}
int pb_unpack(pb_dmat s, double* a, int lda, pb_result* res) {
  return unpack_impl(false, s, 0, a, lda, 0, 1, nullptr, res);
}
int pb_unpack_batched(pb_dmat s, long long stride_s, double* a, int lda, long long stride_a, int batch,
                      pb_stream stream, pb_result* res) {
  return unpack_impl(true, s, stride_s, a, lda, stride_a, batch, stream, res);
}

// ============================================================== Riccati
// riccati.hpp:257-373 (RiccatiFusedWork), 402-512 (riccati_run, FusedNative):
// a batch of independent OCPs with the same (nx, nu, N).
int pb_riccati_nd_batched(int nx, int nu, int N, pb_dmat m0, long long stride_m0, pb_dmat q,
                          long long stride_q, pb_dmat g, long long stride_g, pb_dmat f,
                          long long stride_f, pb_dmat lterm, long long stride_lterm, int* info,
                          int* stage, int batch, pb_stream stream, pb_result* res) {
  const char* routine = "riccati";
  // riccati.hpp:50-52 / 409-412: nx >= 1, nu >= 0, N >= 1 (info -1)
  if (nx < 1 || nu < 0 || N < 1) return status(res, -1, "dims must satisfy nx >= 1, nu >= 0, N >= 1");
  const int nt = nx + nu;
  if (!panel_ok(m0, nt, nt)) return status(res, -4, "m0 panel mismatch");
  if (!panel_ok(q, nx, nx)) return status(res, -6, "q panel mismatch");
  if (!panel_ok(g, nt, nx)) return status(res, -8, "g panel mismatch");
  if (!panel_ok(f, nt, nt)) return status(res, -10, "f panel mismatch");
  const long long f_len = (long long)f.pm * f.cn;
  if (stride_f < f_len * N) return status(res, -11, "f stride below N stage factors");
  if (lterm.data && !panel_ok(lterm, nx, nx)) return status(res, -12, "lterm panel mismatch");
  if (batch < 0) return status(res, -16, "batch is negative");
  if (!info && batch > 0) return status(res, -14, "info is null");
  if (batch == 0) return finish(res, 0, 0);
  std::vector<Operand> ops(7);
  ops[0] = {(void*)m0.data, 8, stride_m0, pm_extent(m0), true, false};
  ops[1] = {(void*)q.data, 8, stride_q, pm_extent(q), true, false};
  ops[2] = {(void*)g.data, 8, stride_g, pm_extent(g), true, false};
  ops[3] = {(void*)f.data, 8, stride_f, f_len * N, false, true};
  ops[4] = {(void*)lterm.data, 8, stride_lterm, lterm.data ? pm_extent(lterm) : 0, true, true};
  ops[5] = {(void*)info, 4, 1, 1, false, true};
  ops[6] = {(void*)stage, 4, 1, 1, false, true};
  int rc = run_batched(routine, ops, batch, stream, res, 3,
                       [&](const std::vector<void*>& p, int nb, cudaStream_t s) -> cudaError_t {
                         RiccatiLaunch R;
                         R.nx = nx; R.nu = nu; R.N = N;
                         R.m0 = (const double*)p[0]; R.sm0 = stride_m0; R.cnm0 = m0.cn;
                         R.q = (const double*)p[1]; R.sq = stride_q; R.cnq = q.cn;
                         R.g = (const double*)p[2]; R.sg = stride_g; R.cng = g.cn;
                         R.f = (double*)p[3]; R.sf = stride_f; R.cnf = f.cn;
                         R.lterm = (double*)p[4]; R.sl = stride_lterm; R.cnl = lterm.cn;
                         R.info = (int*)p[5];
                         R.stage = (int*)p[6];
                         R.batch = nb;
                         return riccati_launch(R, s);
                       });
  if (rc) return rc;
  // flops of the horizon (level3.hpp:479 trmm m n^2; syrk_potrf_nd n^3/3 + n^2 k, :572-573)
  const long long per_stage = (long long)nt * nx * nx + (long long)nt * nt * nt / 3 + (long long)nt * nt * nx;
  return finish(res, 0, ((long long)nx * nx * nx / 3 + N * per_stage) * batch);
}

}  // extern "C"
