// Phase timing of getrf_sq_kernel (PB_SQ_TRACE): average clock64 cycles per phase under full load.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1902_08115_b200/csrc \
//      tools/getrf_trace.cu paper_1902_08115_b200/csrc/runtime.cpp -o tools/getrf_trace
#define PB_SQ_TRACE 1
#include "../paper_1902_08115_b200/csrc/getrf_sq.cu"
#include <cstdio>
#include <vector>

__global__ void fill(double* a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = (i + 0x9e3779b97f4a7c15ull) * 0xbf58476d1ce4e5b9ull;
    z ^= z >> 31; z *= 0x94d049bb133111ebull; z ^= z >> 29;
    a[i] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 48, batch = argc > 2 ? atoi(argv[2]) : 8192;
  double *a, *a0; int *ipiv, *info;
  const long long tot = (long long)n * n * batch;
  cudaMalloc(&a, 8 * tot); cudaMalloc(&a0, 8 * tot); cudaMalloc(&ipiv, 4ll * n * batch); cudaMalloc(&info, 4 * batch);
  fill<<<1024, 256>>>(a0, tot);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(a, a0, 8 * tot, cudaMemcpyDeviceToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = pbg::getrf_sq_launch(a, (long long)n * n, n, n, ipiv, n, info, 0, 0, 0, batch, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d: %.4f ms (%s / %s)\n", rep, ms, cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<long long> tr(128 * 128);
  cudaMemcpyFromSymbol(tr.data(), pbg::sq_trace, 8 * tr.size());
  const int T = n / 8, sampled = (batch + 63) / 64 < 128 ? (batch + 63) / 64 : 128;
  std::vector<double> acc(128, 0.0);
  for (int b = 0; b < sampled; ++b)
    for (int s = 1; s < 128; ++s) acc[s] += (double)(tr[b * 128 + s] - tr[b * 128]) / sampled;
  printf("n=%d: cycles since CTA start (avg of %d CTAs)\n", n, sampled);
  for (int k = 0; k < T; ++k)
    printf("  block %2d: panel start %8.0f  end %8.0f (%6.0f)   look-ahead done %8.0f   rest done %8.0f\n", k,
           acc[4 * k + 4], acc[4 * k + 5], acc[4 * k + 5] - acc[4 * k + 4], k + 1 < T ? acc[4 * k + 6] : 0.0,
           k + 1 < T ? acc[4 * k + 7] : 0.0);
  printf("  written %8.0f\n", acc[1]);
  return 0;
}
