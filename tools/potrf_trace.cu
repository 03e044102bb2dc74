// Phase timing of potrf_cta_kernel: builds the kernel with PB_TRACE, factors a
// batch of SPD matrices and prints the average clock64 cycles per phase.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1902_08115_b200/csrc \
//      tools/potrf_trace.cu -o tools/potrf_trace
#define PB_TRACE 1
#include "../paper_1902_08115_b200/csrc/potrf_cta.cu"
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

namespace pbg {

}

__global__ void make_spd(double* a, int n, int batch) {
  long long p = blockIdx.x;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int r = e % n, c = e / n;
    double v = 0.0;
    for (int l = 0; l < n; ++l) {
      double br = sin(0.37 * (p + 1) * (r + 1) + 0.11 * l), bc = sin(0.37 * (p + 1) * (c + 1) + 0.11 * l);
      v += br * bc;
    }
    a[p * n * n + e] = v + (r == c ? n : 0.0);
  }
}

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 64;
  int batch = argc > 2 ? atoi(argv[2]) : 8192;
  double *a, *a0;
  int* info;
  cudaMalloc(&a, sizeof(double) * n * n * batch);
  cudaMalloc(&a0, sizeof(double) * n * n * batch);
  cudaMalloc(&info, sizeof(int) * batch);
  make_spd<<<batch, 256>>>(a0, n, batch);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(a, a0, sizeof(double) * n * n * batch, cudaMemcpyDeviceToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    pbg::potrf_cta_launch(a, (long long)n * n, nullptr, nullptr, n, n, 0, 0, 0, info, 0, 0, batch, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d: %.4f ms (%s)\n", rep, ms, cudaGetErrorString(cudaGetLastError()));
  }
  {  // residual ||L L^T - A||_F / ||A||_F on a few problems
    std::vector<double> L((size_t)n * n), A((size_t)n * n);
    std::vector<int> inf(batch);
    cudaMemcpy(inf.data(), info, sizeof(int) * batch, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < batch; ++i) bad += inf[i] != 0;
    double worst = 0.0;
    const int probes[4] = {0, 1, batch / 2, batch - 1};
    for (int q = 0; q < 4; ++q) {
      const size_t o = (size_t)probes[q] * n * n;
      cudaMemcpy(L.data(), a + o, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
      cudaMemcpy(A.data(), a0 + o, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
      double num = 0.0, den = 0.0;
      for (int c = 0; c < n; ++c)
        for (int r = c; r < n; ++r) {
          double v = 0.0;
          for (int l = 0; l <= c; ++l) v += L[r + (size_t)l * n] * L[c + (size_t)l * n];
          const double d = v - A[r + (size_t)c * n];
          num += d * d;
          den += A[r + (size_t)c * n] * A[r + (size_t)c * n];
        }
      worst = std::max(worst, std::sqrt(num / den));
    }
    printf("check: nonzero info %d, worst residual %.3e\n", bad, worst);
  }
  std::vector<long long> tr(256 * 64);
  cudaMemcpyFromSymbol(tr.data(), pbg::pb_trace, sizeof(long long) * tr.size());
  const int T = (n + 7) / 8;
  double acc[64] = {0};
  int cnt = 0;
  const int sampled = (batch + 31) / 32 < 256 ? (batch + 31) / 32 : 256;
  for (int b = 0; b < sampled; ++b) {
    const long long* t = &tr[b * 64];
    for (int s = 1; s < 64; ++s) acc[s] += (double)(t[s] - t[0]);
    ++cnt;
  }
  printf("n=%d: cycles since CTA start (avg of %d CTAs)\n", n, cnt);
  printf("  staged      %8.0f\n", acc[1] / cnt);
  for (int k = 0; k < T; ++k)
    printf("  panel %2d: start %8.0f  factored %8.0f  (factor %6.0f)  update warp ready for it %8.0f\n", k,
           acc[4 + 2 * k] / cnt, acc[5 + 2 * k] / cnt, (acc[5 + 2 * k] - acc[4 + 2 * k]) / cnt,
           k + 1 < 24 ? acc[40 + k + 1] / cnt : 0.0);
  printf("  all done    %8.0f\n  written     %8.0f\n", acc[2] / cnt, acc[3] / cnt);
  return 0;
}
