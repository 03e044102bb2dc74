// Microbenchmark: per-warp staging of a 32 KB problem into shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE, int WPC>
__global__ void k(const double* __restrict__ a, double* out, int batch, int per) {
  extern __shared__ __align__(16) double sm[];
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long p = (long long)blockIdx.x * WPC + w;
  if (p >= batch) return;
  double* s = sm + w * per;
  const double* g = a + p * per;
  if (MODE == 0) {  // cp.async 16B, all issued then wait
    for (int e = lane * 2; e < per; e += 64)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(s + e)), "l"(g + e) : "memory");
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  } else if (MODE == 1) {  // LDG.128 -> STS, 8 at a time
    for (int e0 = lane * 2; e0 < per; e0 += 64 * 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) if (e0 + u * 64 < per) v[u] = *(const double2*)(g + e0 + u * 64);
#pragma unroll
      for (int u = 0; u < 8; ++u) if (e0 + u * 64 < per) *(double2*)(s + e0 + u * 64) = v[u];
    }
  } else if (MODE == 2) {  // one TMA bulk copy
    __shared__ __align__(8) uint64_t bar[WPC];
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[w])));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar[w])), "r"(per * 8) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(su32(s)), "l"(g), "r"(per * 8), "r"(su32(&bar[w])) : "memory");
    }
    __syncwarp();
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n selp.u32 %0,1,0,q;\n}\n" : "=r"(ok) : "r"(su32(&bar[w])) : "memory");
  } else if (MODE == 3) {  // cp.async 8B .ca, all issued
    for (int e = lane; e < per; e += 32)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(su32(s + e)), "l"(g + e) : "memory");
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  __syncwarp();
  // write back: STS->STG.128
  double* o = out + p * per;
  for (int e = lane * 2; e < per; e += 64) *(double2*)(o + e) = *(double2*)(s + e);
}
template <int MODE, int WPC>
void run(const double* a, double* out, int batch, int per, const char* name) {
  size_t smem = (size_t)WPC * per * 8;
  cudaFuncSetAttribute(k<MODE, WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = (batch + WPC - 1) / WPC;
  k<MODE, WPC><<<grid, 32 * WPC, smem>>>(a, out, batch, per);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<MODE, WPC><<<grid, 32 * WPC, smem>>>(a, out, batch, per);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
  printf("%-28s WPC=%d per=%d: %.4f ms  %.0f GB/s (r+w)  err=%s\n", name, WPC, per, ms, 2.0 * batch * per * 8 / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int batch = 8192;
  for (int per : {2080, 4096}) {
    double *a, *o; cudaMalloc(&a, (size_t)batch * per * 8); cudaMalloc(&o, (size_t)batch * per * 8);
    cudaMemset(a, 0, (size_t)batch * per * 8);
    run<0, 2>(a, o, batch, per, "cp.async16 wpc2");
    run<0, 4>(a, o, batch, per, "cp.async16 wpc4");
    run<1, 2>(a, o, batch, per, "ldg128->sts wpc2");
    run<1, 4>(a, o, batch, per, "ldg128->sts wpc4");
    run<2, 2>(a, o, batch, per, "tma bulk wpc2");
    run<2, 4>(a, o, batch, per, "tma bulk wpc4");
    run<3, 2>(a, o, batch, per, "cp.async8 wpc2");
    cudaFree(a); cudaFree(o);
  }
}
