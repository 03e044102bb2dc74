// Dependent-chain latencies (cycles per op) of FP64 ops on sm_100a, one warp.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001, z = 0.9999999;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x = fma(x, y, z);
  }
  t1 = clock64(); cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x = x * y;
  }
  t1 = clock64(); cyc[1] = t1 - t0;
  // rsqrt chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x = rsqrt(x) + 0.5;
  }
  t1 = clock64(); cyc[2] = t1 - t0;
  // float rsqrt + 2 Newton steps in double
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double r = (double)rsqrtf((float)x);
      double h = x * r;
      double e = fma(-h, r, 1.0);
      r = fma(r * 0.5, e, r) ;
      h = x * r; e = fma(-h, r, 1.0);
      r = fma(r * 0.5, e, r);
      x = r + 0.5;
    }
  }
  t1 = clock64(); cyc[3] = t1 - t0;
  // sqrt chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x = sqrt(x) + 0.5;
  }
  t1 = clock64(); cyc[4] = t1 - t0;
  // 1/x chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x = 1.0 / x + 0.5;
  }
  t1 = clock64(); cyc[5] = t1 - t0;
  // shfl chain
  double s = x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s = __shfl_sync(0xffffffffu, s, (threadIdx.x + 1) & 31);
  }
  t1 = clock64(); cyc[6] = t1 - t0;
  // dadd chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x = x + y;
  }
  t1 = clock64(); cyc[7] = t1 - t0;
  // DMMA chain (accumulator dependent)
  double d0 = 0, d1 = 0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d0), "+d"(d1) : "d"(y), "d"(z));
  }
  t1 = clock64(); cyc[8] = t1 - t0;
  // 8 independent DMMA chains (throughput, one warp)
  double e[8][2] = {};
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(e[j][0]), "+d"(e[j][1]) : "d"(y), "d"(z));
  }
  t1 = clock64(); cyc[9] = t1 - t0;
  double acc = 0; for (int j = 0; j < 8; ++j) acc += e[j][0] + e[j][1];
  // rsqrt_nb chain (rsqrt.approx.ftz.f64 + one third-order Newton step, common.cuh)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double yy;
      asm("rsqrt.approx.ftz.f64 %0, %1;\n" : "=d"(yy) : "d"(x));
      const double ee = fma(-x, yy * yy, 1.0);
      const double cc = fma(ee, 0.375, 0.5);
      x = fma(cc, yy * ee, yy) + 0.5;
    }
  }
  t1 = clock64(); cyc[10] = t1 - t0;
  // shared-memory load chain (pointer chase through a 32-entry ring)
  __shared__ int ring[64];
  ring[threadIdx.x] = (threadIdx.x + 1) & 31;
  __syncwarp();
  int pidx = threadIdx.x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) pidx = ((volatile int*)ring)[pidx];
  }
  t1 = clock64(); cyc[11] = t1 - t0;
  acc += pidx;
  // redux.sync (CREDUX) chain: max over the warp feeding the next input
  unsigned ru = threadIdx.x * 2654435761u;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) ru = __reduce_max_sync(0xffffffffu, ru) ^ (threadIdx.x + j);
  }
  t1 = clock64(); cyc[12] = t1 - t0;
  // ballot chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) ru = __ballot_sync(0xffffffffu, (ru >> (threadIdx.x & 7)) & 1) + threadIdx.x + j;
  }
  t1 = clock64(); cyc[13] = t1 - t0;
  // sts.128 -> syncwarp -> lds.128 round trip (one lane publishes, all read)
  __shared__ __align__(16) double rb[2][4];
  double rx = x, ry = x + 1.0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (threadIdx.x == ((i + j) & 31)) asm volatile("st.shared.v2.f64 [%0], {%1,%2};\n" ::"r"((unsigned)__cvta_generic_to_shared(&rb[j & 1][0])), "d"(rx), "d"(ry) : "memory");
      __syncwarp();
      asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(rx), "=d"(ry) : "r"((unsigned)__cvta_generic_to_shared(&rb[j & 1][0])) : "memory");
      rx += 1.0;
    }
  }
  t1 = clock64(); cyc[14] = t1 - t0;
  // __drcp_rn chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x = __drcp_rn(x) + 0.5;
  }
  t1 = clock64(); cyc[15] = t1 - t0;
  acc += ru + rx + ry;
  out[threadIdx.x] = x + s + d0 + d1 + acc;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 32); cudaMallocManaged(&c, 8 * 16);
  k<<<1, 32>>>(o, c, 1.5); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.5); cudaDeviceSynchronize();
  const char* nm[] = {"dfma", "dmul", "rsqrt(double)", "rsqrtf+2NR", "sqrt(double)", "1/x", "shfl", "dadd", "dmma dep", "dmma 8 indep", "rsqrt_nb", "lds chain", "redux.max (CREDUX)", "ballot", "sts128+syncwarp+lds128 (+dadd)", "__drcp_rn (+dadd)"};
  for (int i = 0; i < 16; ++i) printf("%-32s %6.1f cycles/op\n", nm[i], c[i] / 2048.0);
}
