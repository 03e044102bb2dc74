// Live FP64 tensor-core peak probe (DMMA m8n8k4, 4 warps/SM x 8 independent
// chains).  bench.py uses it as the measured FP64 roofline denominator, since
// MEASURED_PEAKS.json carries no FP64 figure (profiles/r01_fp64_peak.txt).
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace pbg {

__global__ void dmma_probe_kernel(double* out, int iters) {
  double acc[8][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < 8; ++c) { acc[c][0] = c; acc[c][1] = -c; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int c = 0; c < 8; ++c) dmma(acc[c][0], acc[c][1], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

double probe_dmma_tflops() {
  double* out = nullptr;
  if (cudaMalloc(&out, 8) != cudaSuccess) return 0.0;
  const int sms = num_sms(), iters = 20000, blocks = sms * 2, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_probe_kernel<<<blocks, threads>>>(out, iters);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    dmma_probe_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  double flops = 512.0 * 8 * iters * (double)blocks * (threads / 32);
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace pbg
