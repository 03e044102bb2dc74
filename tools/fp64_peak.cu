// FP64 throughput microbenchmark for the roofline denominator (DMMA m8n8k4 and DFMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double acc[CHAINS][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { acc[c][0] = c; acc[c][1] = -c; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double acc[CHAINS];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
float timeit(K kern, int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 20000;
  for (int wpb : {4, 8, 16}) for (int bps : {1, 2, 4}) {
    int threads = 32 * wpb, blocks = sms * bps;
    float ms = timeit(dmma_loop<8>, blocks, threads, iters, out);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * wpb);
    printf("DMMA chains=8 warps/blk=%d blk/SM=%d : %.2f TFLOP/s\n", wpb, bps, flops / ms / 1e9);
  }
  for (int wpb : {4, 8, 16}) for (int bps : {1, 2, 4}) {
    int threads = 32 * wpb, blocks = sms * bps;
    float ms = timeit(dfma_loop<8>, blocks, threads, iters, out);
    double flops = 2.0 * 8.0 * iters * (blocks * threads);
    printf("DFMA chains=8 warps/blk=%d blk/SM=%d : %.2f TFLOP/s\n", wpb, bps, flops / ms / 1e9);
  }
  // single-warp latency probe: 1 chain
  {
    float ms = timeit(dmma_loop<1>, 1, 32, iters, out);
    printf("DMMA dependent-chain latency: %.1f ns/op\n", ms * 1e6 / iters);
    ms = timeit(dfma_loop<1>, 1, 32, iters, out);
    printf("DFMA dependent-chain latency: %.1f ns/op\n", ms * 1e6 / iters);
    ms = timeit(dmma_loop<4>, sms, 32, iters, out);
    printf("DMMA 1 warp/SM 4 chains: %.2f TFLOP/s\n", 2.0*256*4.0*iters*sms/ms/1e9);
    ms = timeit(dmma_loop<8>, sms, 32, iters, out);
    printf("DMMA 1 warp/SM 8 chains: %.2f TFLOP/s\n", 2.0*256*8.0*iters*sms/ms/1e9);
    ms = timeit(dmma_loop<8>, sms, 128, iters, out);
    printf("DMMA 4 warp/SM 8 chains: %.2f TFLOP/s\n", 2.0*256*8.0*iters*sms*4/ms/1e9);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms=%d clock_khz=%d\n", sms, clk);
  return 0;
}
