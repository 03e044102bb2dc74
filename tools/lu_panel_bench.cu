// Cycles of one sq_panel<T,1> call (8 columns, 32 rows) for one warp alone on its SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1902_08115_b200/csrc tools/lu_panel_bench.cu paper_1902_08115_b200/csrc/runtime.cpp -o tools/lu_panel_bench
#include "../paper_1902_08115_b200/csrc/getrf_sq.cu"
#include <cstdio>
using namespace pbg;

template <int T>
__global__ void bench(long long* out, int reps, int c0) {
  constexpr int N = 8 * T, S = sq_stride(T);
  extern __shared__ __align__(16) double sm[];
  __shared__ int piv_all[N];
  __shared__ __align__(16) double scr[2][12];
  __shared__ int mv[20];
  const int lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < S * N; e += blockDim.x) {
    unsigned z = (unsigned)e * 2654435761u;
    z ^= z >> 15;
    sm[e] = (double)(z & 0xffffff) / 16777216.0 - 0.5;
  }
  __syncthreads();
  const uint32_t sbase = smem_u32(sm), scr0 = smem_u32(&scr[0][0]);
  int fz = 0;
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    fz = sq_panel<T, 1>(sbase, c0, lane, scr0, piv_all, mv, nullptr, fz);
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x] = (t1 - t0) / reps + (fz > 1000000);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 148);
  constexpr int T = 12;
  const size_t smem = (size_t)sq_stride(T) * 8 * T * 8;
  cudaFuncSetAttribute(bench<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int c0 : {64, 88}) {
    bench<T><<<148, 32, smem>>>(d, 50, c0);
    cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("sq_panel<12,1> c0=%d (rows %d): %lld cycles per 8-column block alone (%s)\n", c0, 96 - c0, h[0],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
