// Cycles per call of panel-factorization variants (one warp alone on its SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1902_08115_b200/csrc tools/panel_bench.cu -o tools/panel_bench
#include "../paper_1902_08115_b200/csrc/potrf_cta.cu"
#include <cstdio>
namespace pbg { int num_sms() { return 148; } }
using namespace pbg;

// V0: D chain only (no rows)
__device__ __forceinline__ int chain_only(uint32_t pan, int RS) {
  double D[8][8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int i = c & ~1; i < 8; i += 2) {
      double2 v;
      asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(pan + 8u * (c * RS + i)));
      D[i][c] = v.x;
      D[i + 1][c] = v.y;
    }
  int f = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double piv = D[c][c];
    if (f == 0 && piv <= 0.0) f = c + 1;
    const double inv = rsqrt_nb(piv);
    D[c][c] = piv * inv;
#pragma unroll
    for (int i = c + 1; i < 8; ++i) D[i][c] *= inv;
#pragma unroll
    for (int c2 = c + 1; c2 < 8; ++c2)
#pragma unroll
      for (int i = c2; i < 8; ++i) D[i][c2] -= D[i][c] * D[c2][c];
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) sts64(pan + 8u * (c * RS + (threadIdx.x & 7)), D[7][c]);
  return f;
}

// V2: rows deferred by one column (software pipelined)
template <int R>
__device__ __forceinline__ int piped(uint32_t pan, int RS, int rows, int lane) {
  double x[R][8];
  double D[8][8];
  double invs[8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int i = c & ~1; i < 8; i += 2) {
      double2 v;
      asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(pan + 8u * (c * RS + i)));
      D[i][c] = v.x;
      D[i + 1][c] = v.y;
    }
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[q][c] = lds64(pan + 8u * (c * RS + lane + 32 * q));
  int f = 0;
#pragma unroll
  for (int c = 0; c <= 8; ++c) {
    if (c < 8) {
      const double piv = D[c][c];
      if (f == 0 && piv <= 0.0) f = c + 1;
      const double inv = rsqrt_nb(piv);
      invs[c] = inv;
      D[c][c] = piv * inv;
#pragma unroll
      for (int i = c + 1; i < 8; ++i) D[i][c] *= inv;
#pragma unroll
      for (int c2 = c + 1; c2 < 8; ++c2)
#pragma unroll
        for (int i = c2; i < 8; ++i) D[i][c2] -= D[i][c] * D[c2][c];
    }
    if (c > 0) {
      const int cp = c - 1;
#pragma unroll
      for (int q = 0; q < R; ++q) x[q][cp] *= invs[cp];
#pragma unroll
      for (int c2 = cp + 1; c2 < 8; ++c2)
#pragma unroll
        for (int q = 0; q < R; ++q) x[q][c2] -= x[q][cp] * D[c2][cp];
    }
  }
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      sts64_if(pan + 8u * (c * RS + lane + 32 * q), x[q][c], lane + 32 * q < rows);
  return f;
}

// V3: all 8 columns of D first (chain), then rows against the finished L11 (TRSM by substitution)
template <int R>
__device__ __forceinline__ int chol_then_trsm(uint32_t pan, int RS, int rows, int lane) {
  double x[R][8];
  double D[8][8];
  double invs[8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int i = c & ~1; i < 8; i += 2) {
      double2 v;
      asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(pan + 8u * (c * RS + i)));
      D[i][c] = v.x;
      D[i + 1][c] = v.y;
    }
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[q][c] = (lane + 32 * q < rows) ? lds64(pan + 8u * (c * RS + lane + 32 * q)) : 0.0;
  int f = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double piv = D[c][c];
    if (f == 0 && piv <= 0.0) f = c + 1;
    const double inv = rsqrt_nb(piv);
    invs[c] = inv;
    D[c][c] = piv * inv;
#pragma unroll
    for (int i = c + 1; i < 8; ++i) D[i][c] *= inv;
#pragma unroll
    for (int c2 = c + 1; c2 < 8; ++c2)
#pragma unroll
      for (int i = c2; i < 8; ++i) D[i][c2] -= D[i][c] * D[c2][c];
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
#pragma unroll
    for (int q = 0; q < R; ++q) x[q][c] *= invs[c];
#pragma unroll
    for (int c2 = c + 1; c2 < 8; ++c2)
#pragma unroll
      for (int q = 0; q < R; ++q) x[q][c2] -= x[q][c] * D[c2][c];
  }
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (lane + 32 * q < rows) sts64(pan + 8u * (c * RS + lane + 32 * q), x[q][c]);
  return f;
}


// V4: rows only, the diagonal block's column broadcast by shuffles (no redundant D)
template <int R>
__device__ __forceinline__ int shfl_panel(uint32_t pan, int RS, int rows, int lane) {
  const unsigned FULL = 0xffffffffu;
  double x[R][8];
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[q][c] = lds64(pan + 8u * (c * RS + lane + 32 * q));
  int f = 0;
  bool special = false;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double piv = __shfl_sync(FULL, x[0][c], c);
    if (f == 0 && piv <= 0.0) f = c + 1;
    special |= f == 0 && rsqrt_special(piv);
    const double inv = rsqrt_nb(piv);
#pragma unroll
    for (int q = 0; q < R; ++q) x[q][c] *= inv;
    // lanes c+1..7 hold L(c2, c) in x[0][c]
#pragma unroll
    for (int c2 = c + 1; c2 < 8; ++c2) {
      const double l = __shfl_sync(FULL, x[0][c], c2);
#pragma unroll
      for (int q = 0; q < R; ++q) x[q][c2] -= x[q][c] * l;
    }
  }
  if (lane < 8) {}  // diagonal: x[0][lane] = piv * inv already (x * inv with x == piv)
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c) sts64_if(pan + 8u * (c * RS + lane + 32 * q), x[q][c], lane + 32 * q < rows);
  return f + special;
}

template <int R, int V>
__global__ void bench(long long* cyc, double* sink, int T) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31;
  const int RS = 8 * T + 4, rows = 8 * T;
  for (int e = threadIdx.x; e < 8 * RS; e += blockDim.x) {
    const int c = e / RS, r = e % RS;
    sm[e] = (r == c) ? 100.0 : 0.01 * ((r * 7 + c * 3) % 11);
  }
  __syncthreads();
  const uint32_t pan = smem_u32(sm);
  int f = 0;
  long long t0 = clock64();
  for (int it = 0; it < 64; ++it) {
    if (V == 0) f += chain_only(pan, RS);
    if (V == 1) f += cta_factor_panel<R>(pan, RS, rows, lane, 0, 1 << 20);
    if (V == 2) f += piped<R>(pan, RS, rows, lane);
    if (V == 3) f += shfl_panel<R>(pan, RS, rows, lane);
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x] = (t1 - t0) / 64;
  sink[threadIdx.x] = sm[threadIdx.x] + f;
}

template <int R>
void run(int T) {
  long long* c;
  double* s;
  cudaMallocManaged(&c, 8 * 1024);
  cudaMalloc(&s, 8 * 1024);
  size_t smem = (8 * (8 * T + 4) + 8 * T + 32) * 8;
  long long r[4];
  for (int rep = 0; rep < 2; ++rep) {
    bench<R, 0><<<1, 32, smem>>>(c, s, T); cudaDeviceSynchronize(); r[0] = c[0];
    bench<R, 1><<<1, 32, smem>>>(c, s, T); cudaDeviceSynchronize(); r[1] = c[0];
    bench<R, 2><<<1, 32, smem>>>(c, s, T); cudaDeviceSynchronize(); r[2] = c[0];
    bench<R, 3><<<1, 32, smem>>>(c, s, T); cudaDeviceSynchronize(); r[3] = c[0];
  }
  printf("T=%2d R=%d: chain-only %lld  current %lld  piped %lld  shfl %lld  (%s)\n", T, R, r[0], r[1], r[2],
         r[3], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<1>(4);
  run<2>(8);
  run<3>(12);
  run<4>(16);
}
