#include <cstdio>
#include <cmath>
__global__ void k(const double* x, double* y, int n) {
  int i = threadIdx.x;
  if (i < n) { double v = x[i]; y[3*i] = rsqrt(v); y[3*i+1] = 1.0/sqrt(v); y[3*i+2] = v * rsqrt(v); }
}
int main() {
  double h[6] = {ldexp(1.0,-1040), ldexp(1.0,-1030), ldexp(1.0,-1073), 4.0, INFINITY, ldexp(3.0,-1050)};
  double *d, *o; cudaMalloc(&d, 6*8); cudaMalloc(&o, 18*8);
  cudaMemcpy(d, h, 48, cudaMemcpyHostToDevice);
  k<<<1,32>>>(d, o, 6);
  double r[18]; cudaMemcpy(r, o, 18*8, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 6; ++i) printf("x=%a rsqrt=%a 1/sqrt=%a x*rsqrt=%a\n", h[i], r[3*i], r[3*i+1], r[3*i+2]);
}
