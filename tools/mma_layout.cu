// Verifies the assumed per-lane fragment layouts of the f64 mma shapes m16n8k4/k8/k16 on sm_100a.
//   g = lane>>2, t = lane&3
//   A (16 x K, row):   a[i] = A[g + 8*(i%2)][t + 4*(i/2)]      i < K/2
//   B (K x 8, col):    b[i] = B[t + 4*i][g]                     i < K/4
//   C/D (16 x 8):      d[0],d[1] = D[g][2t], D[g][2t+1]; d[2],d[3] = D[g+8][2t], D[g+8][2t+1]
#include <cstdio>
#include <cmath>
template <int K>
__global__ void run(const double* A, const double* B, double* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[K / 2], b[K / 4], d[4];
  for (int i = 0; i < K / 2; ++i) a[i] = A[(g + 8 * (i % 2)) * K + t + 4 * (i / 2)];
  for (int i = 0; i < K / 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  for (int i = 0; i < 4; ++i) d[i] = 0.0;
  if constexpr (K == 4)
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  if constexpr (K == 8)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  if constexpr (K == 16)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  D[g * 8 + 2 * t] = d[0];
  D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2];
  D[(g + 8) * 8 + 2 * t + 1] = d[3];
}
template <int K>
int check() {
  double hA[16 * K], hB[K * 8], hD[128];
  for (int i = 0; i < 16 * K; ++i) hA[i] = (i * 37 % 101) * 0.01 - 0.3;
  for (int i = 0; i < K * 8; ++i) hB[i] = (i * 53 % 97) * 0.02 - 0.9;
  double *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  run<K><<<1, 32>>>(A, B, D);
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += hA[m * K + k] * hB[k * 8 + n];
      err = fmax(err, fabs(s - hD[m * 8 + n]));
    }
  printf("m16n8k%d: max err %.3e (%s)\n", K, err, cudaGetErrorString(cudaGetLastError()));
  return err < 1e-12 ? 0 : 1;
}
int main() { return check<4>() | check<8>() | check<16>(); }
