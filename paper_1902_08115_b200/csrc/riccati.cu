// Batched factorized backward Riccati recursion (the paper's application,
// PAPER.md:787-817): many independent optimal-control problems (OCPs), each
// running the packed stage loop of RiccatiFusedWork (riccati.hpp:257-373)
// over its horizon, as riccati_run's FusedNative path does for one OCP
// (riccati.hpp:402-512).
//
// Stage s (s = N-1 .. 0) of every OCP of the batch runs as three batched
// launches; the stages themselves are sequential (calL_s needs calL_{s+1}):
//   C_s    = G * calL_{s+1}                 trmm_rlnn_nd  (trmm.cu, DMMA)
//   F_s    = chol(M0 + C_s C_s^T)           syrk_potrf_nd (potrf_cta.cu fused prologue)
//   calL_s = trailing nx x nx block of F_s  (copy below, strict upper kept zero)
// The terminal factor calL_N = chol(Q) is syrk_potrf_nd with k = 0
// (riccati.hpp:297-303), so no factor ever leaves panel storage.
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace pbg {

__device__ __forceinline__ long long rc_poff(int i, int j, int cn) {
  return (long long)(i >> 2) * 4 * cn + (long long)j * 4 + (i & 3);
}

// calL (nx x nx, cn = cnl) <- lower part of F(nu.., nu..) (F nt x nt, cn = cnf);
// strictly-upper entries are written as 0 (RiccatiFusedWork::call_ keeps them zero).
__global__ void riccati_trailing_kernel(const double* F, long long sf, int cnf, double* Lc, long long sl, int cnl,
                                        int nu, int nx) {
  const long long p = blockIdx.y;
  const double* f = F + p * sf;
  double* l = Lc + p * sl;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nx * nx; e += gridDim.x * blockDim.x) {
    const int j = e / nx, i = e - j * nx;
    l[rc_poff(i, j, cnl)] = i >= j ? f[rc_poff(nu + i, nu + j, cnf)] : 0.0;
  }
}

// First failure wins: info[p] / stage[p] keep the earliest (highest) stage's report.
__global__ void riccati_merge_info_kernel(const int* st_info, int* info, int* stage, int s, int batch) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= batch) return;
  if (info[p] == 0 && st_info[p] != 0) {
    info[p] = st_info[p];
    if (stage) stage[p] = s;
  }
}

cudaError_t riccati_launch(const RiccatiLaunch& R, cudaStream_t s) {
  if (R.batch <= 0) return cudaSuccess;
  const int nx = R.nx, nu = R.nu, nt = nx + nu, N = R.N;
  const int cnt = (nt + 3) & ~3, cnx = (nx + 3) & ~3;
  const long long l_len = (long long)cnx * cnx, c_len = (long long)cnt * cnx;
  mempool_keep();
  cudaError_t e;
  double* ws = nullptr;
  int* st_info = nullptr;
  if ((e = cudaMallocAsync(&ws, sizeof(double) * (l_len + c_len) * R.batch, s)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&st_info, sizeof(int) * R.batch, s)) != cudaSuccess) {
    cudaFreeAsync(ws, s);
    return e;
  }
  double* call = ws;                           // calL workspace, problem p at p * l_len
  double* cbuf = ws + l_len * R.batch;         // C = G calL, problem p at p * c_len
  auto done = [&](cudaError_t err) {
    cudaFreeAsync(ws, s);
    cudaFreeAsync(st_info, s);
    return err;
  };
  // zero-filled workspaces and stage factors: strictly-upper tiles are never written
  if ((e = cudaMemsetAsync(ws, 0, sizeof(double) * (l_len + c_len) * R.batch, s)) != cudaSuccess) return done(e);
  if ((e = cudaMemsetAsync(R.info, 0, sizeof(int) * R.batch, s)) != cudaSuccess) return done(e);
  if (R.stage && (e = cudaMemsetAsync(R.stage, 0xff, sizeof(int) * R.batch, s)) != cudaSuccess) return done(e);
  const long long f_len = (long long)R.cnf * R.cnf;
  for (int b = 0; b < R.batch; ++b) {  // (strided: one memset per OCP when the stride has gaps)
    if (R.sf == f_len * N) {
      e = cudaMemsetAsync(R.f, 0, sizeof(double) * f_len * N * R.batch, s);
      break;
    }
    if ((e = cudaMemsetAsync(R.f + (long long)b * R.sf, 0, sizeof(double) * f_len * N, s)) != cudaSuccess) break;
  }
  if (e != cudaSuccess) return done(e);

  // terminal factor calL_N = chol(Q): syrk_potrf_nd(nx, 0, -, -, Q, calL)
  SyrkPotrfLaunch T;
  T.c = R.q; T.sc = R.sq; T.cnc = R.cnq;
  T.d = call; T.sd = l_len; T.cnd = cnx;
  T.n = nx; T.k = 0;
  T.info = st_info;
  T.batch = R.batch;
  if ((e = syrk_potrf_launch(T, s)) != cudaSuccess) return done(e);
  riccati_merge_info_kernel<<<(R.batch + 255) / 256, 256, 0, s>>>(st_info, R.info, R.stage, N, R.batch);
  if ((e = cudaGetLastError()) != cudaSuccess) return done(e);
  if (R.lterm) {
    // lterm <- calL_N (same panel layout, its own stride)
    riccati_trailing_kernel<<<dim3((unsigned)std::max(1, std::min(64, (nx * nx + 255) / 256)), R.batch), 256, 0, s>>>(
        call, l_len, cnx, R.lterm, R.sl, R.cnl, 0, nx);
    if ((e = cudaGetLastError()) != cudaSuccess) return done(e);
  }
  for (int st = N - 1; st >= 0; --st) {
    double* fs = R.f + (long long)st * f_len;
    TrsmLaunch M;  // C = G * calL  (trmm_rlnn_nd: right, lower, no-trans, non-unit)
    M.pm = 1;
    M.lower = 1; M.trans = 0; M.unit = 0;
    M.mm = nt; M.nn = nx;
    M.alpha = 1.0;
    M.a = call; M.sa = l_len; M.lda = cnx;
    M.b = R.g; M.sb = R.sg; M.ldb = R.cng;
    M.d = cbuf; M.sd = c_len; M.ldd = cnx;
    M.batch = R.batch;
    if ((e = trmm_launch(M, s)) != cudaSuccess) return done(e);
    SyrkPotrfLaunch P;  // F_s = chol(M0 + C C^T)
    P.a = cbuf; P.b = cbuf; P.sa = P.sb = c_len; P.cna = P.cnb = cnx;
    P.c = R.m0; P.sc = R.sm0; P.cnc = R.cnm0;
    P.d = fs; P.sd = R.sf; P.cnd = R.cnf;
    P.n = nt; P.k = nx;
    P.info = st_info;
    P.batch = R.batch;
    if ((e = syrk_potrf_launch(P, s)) != cudaSuccess) return done(e);
    riccati_merge_info_kernel<<<(R.batch + 255) / 256, 256, 0, s>>>(st_info, R.info, R.stage, st, R.batch);
    riccati_trailing_kernel<<<dim3((unsigned)std::max(1, std::min(64, (nx * nx + 255) / 256)), R.batch), 256, 0, s>>>(
        fs, R.sf, R.cnf, call, l_len, cnx, nu, nx);
    if ((e = cudaGetLastError()) != cudaSuccess) return done(e);
  }
  return done(cudaSuccess);
}

}  // namespace pbg
