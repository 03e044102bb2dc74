// Batched layout kernels of the drop-in boundary: column-major <-> panel-major
// (pack_from_colmajor / unpack_to_colmajor, panel_mat.hpp:141-171; memsize
// 45-48), and the PBGPU_MUTATE fault-injection pass.
//
// Both directions iterate in DESTINATION order, so every store is coalesced
// and every 32-byte read sector is used whole when ps = 4 (a panel column is
// ps consecutive doubles of one source column).  Pad lanes of a panel-major
// destination are never written (panel_mat.hpp:8-12).  HBM-bound: algorithmic
// bytes 16 m n per problem.
#include <cstdlib>

#include "launch.h"

namespace pbg {

__global__ void pack_kernel(int trans, int m, int n, const double* __restrict__ a, int lda, long long sa,
                            double* __restrict__ d, int ps, int cn, long long sd, long long pm_cn) {
  const long long p = blockIdx.y;
  const double* src = a + p * sa;
  double* dst = d + p * sd;
  const long long pw = (long long)ps * cn;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < pm_cn; q += (long long)gridDim.x * blockDim.x) {
    const long long P = q / pw, rem = q - P * pw;
    const int j = (int)(rem / ps), i = (int)(P * ps + rem % ps);
    if (i >= m || j >= n) continue;
    dst[q] = trans ? src[(long long)j + (long long)i * lda] : src[(long long)i + (long long)j * lda];
  }
}

__global__ void unpack_kernel(int m, int n, const double* __restrict__ s, int ps, int cn, long long ss,
                              double* __restrict__ a, int lda, long long sa) {
  const long long p = blockIdx.y;
  const double* src = s + p * ss;
  double* dst = a + p * sa;
  const long long mn = (long long)m * n;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < mn; q += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(q / m), i = (int)(q - (long long)j * m);
    dst[(long long)i + (long long)j * lda] = src[(long long)(i / ps) * ps * cn + (long long)j * ps + i % ps];
  }
}

static dim3 lgrid(long long work, int batch) {
  long long bx = (work + 255) / 256;
  // enough CTAs to cover the SMs several times over even for small batches
  const long long want = (8LL * num_sms() + batch - 1) / batch;
  bx = bx < want ? bx : want;
  return dim3((unsigned)(bx < 1 ? 1 : bx), (unsigned)batch);
}

cudaError_t pack_launch(int trans, int m, int n, const double* a, int lda, long long sa, double* d, int ps, int cn,
                        long long sd, int batch, cudaStream_t s) {
  if (batch <= 0 || m <= 0 || n <= 0) return cudaSuccess;
  const long long pm = (long long)((m + ps - 1) / ps) * ps;
  const long long work = pm * cn;
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = batch - b0 < 65535 ? batch - b0 : 65535;
    pack_kernel<<<lgrid(work, nb), 256, 0, s>>>(trans, m, n, a + (long long)b0 * sa, lda, sa, d + (long long)b0 * sd,
                                                ps, cn, sd, work);
  }
  return cudaGetLastError();
}

cudaError_t unpack_launch(int m, int n, const double* src, int ps, int cn, long long ss, double* a, int lda,
                          long long sa, int batch, cudaStream_t s) {
  if (batch <= 0 || m <= 0 || n <= 0) return cudaSuccess;
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = batch - b0 < 65535 ? batch - b0 : 65535;
    unpack_kernel<<<lgrid((long long)m * n, nb), 256, 0, s>>>(m, n, src + (long long)b0 * ss, ps, cn, ss,
                                                             a + (long long)b0 * sa, lda, sa);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- PBGPU_MUTATE
double mutation_epsilon() {
  static const double eps = [] {
    const char* e = getenv("PBGPU_MUTATE");
    return e ? atof(e) : 0.0;
  }();
  return eps;
}

__global__ void mutate_kernel(double* d, long long sd, const long long* offs, int batch, double eps) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < batch) d[offs ? offs[p] : (long long)p * sd] += eps;
}

cudaError_t mutate_launch(double* d, long long sd, const long long* offs, int batch, double eps, cudaStream_t s) {
  if (batch <= 0 || eps == 0.0 || !d) return cudaSuccess;
  mutate_kernel<<<(batch + 255) / 256, 256, 0, s>>>(d, sd, offs, batch, eps);
  return cudaGetLastError();
}

}  // namespace pbg
