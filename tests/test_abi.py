"""CPU: the C-ABI library loads, exports every symbol include/pbgpu.h declares, and
validates arguments exactly like the reference adapters before touching a device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pbgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(pb):
    lib = ctypes.CDLL(pb.library_path)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(pb.EXPORTED)


def test_shim_header_compiles_against_the_abi(tmp_path):
    """include/pbgpu_panelblas.hpp (reference-shaped C++ API) compiles and links."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "pbgpu_panelblas.hpp"\nint main(){ pbgpu::BlasConfig c; double x[4]={0};\n'
                   ' auto r = pbgpu::dgemm(c, \'x\', \'n\', 1,1,1, 1.0, x,1, x,1, 0.0, x,1);\n'
                   ' return r.info == 1 && r.error && r.error->index == 1 ? 0 : 1; }\n')
    exe = tmp_path / "t"
    import subprocess
    r = subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                        os.path.join(ROOT, "paper_1902_08115_b200", "libpbgpu.so"),
                        f"-Wl,-rpath,{os.path.join(ROOT, 'paper_1902_08115_b200')}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(exe)]).returncode == 0


def check(r, routine, index, info):
    assert r.info == info
    assert r.error is not None and r.error.routine == routine and r.error.index == index


def test_dgemm_validation_order(pb):
    buf = np.zeros(16)
    call = lambda ta, tb, m, n, k, lda, ldb, ldc: pb.dgemm(ta, tb, m, n, k, 1.0, buf, lda, buf, ldb, 0.0, buf, ldc)
    check(call("x", "t", 2, 2, 2, 2, 2, 2), "dgemm", 1, 1)
    check(call("n", "q", 2, 2, 2, 2, 2, 2), "dgemm", 2, 2)
    check(call("n", "n", -1, 2, 2, 2, 2, 2), "dgemm", 3, 3)
    check(call("n", "n", 2, -1, 2, 2, 2, 2), "dgemm", 4, 4)
    check(call("n", "n", 2, 2, -1, 2, 2, 2), "dgemm", 5, 5)
    check(call("n", "n", 2, 2, 2, 1, 2, 2), "dgemm", 8, 8)
    check(call("t", "n", 2, 2, 3, 2, 3, 2), "dgemm", 8, 8)
    check(call("n", "n", 2, 2, 2, 2, 1, 2), "dgemm", 10, 10)
    check(call("n", "t", 2, 3, 2, 2, 2, 2), "dgemm", 10, 10)
    check(call("n", "n", 2, 2, 2, 2, 2, 1), "dgemm", 13, 13)
    check(call("n", "n", 1, 1, 1, 0, 1, 1), "dgemm", 8, 8)
    check(call("x", "q", -1, -1, -1, 0, 0, 0), "dgemm", 1, 1)
    # 'C' parses as transpose; empty shapes quick-return without a device
    assert pb.dgemm("C", "c", 0, 3, 2, 1.0, buf, 2, buf, 3, 0.0, buf, 1).ok()
    assert pb.dgemm("n", "n", 3, 0, 2, 1.0, buf, 3, buf, 2, 0.5, buf, 3).ok()
    assert pb.dgemm("n", "n", 2, 2, 0, 1.0, buf, 2, buf, 1, 1.0, buf, 2).ok()  # k=0, beta=1


def test_dsyrk_trsm_potrf_getrf_validation(pb):
    buf = np.zeros(16)
    s = lambda ul, tr, n, k, lda, ldc: pb.dsyrk(ul, tr, n, k, 1.0, buf, lda, 1.0, buf, ldc)
    check(s("x", "n", 1, 1, 1, 1), "dsyrk", 1, 1)
    check(s("l", "z", 1, 1, 1, 1), "dsyrk", 2, 2)
    check(s("l", "n", -1, 1, 1, 1), "dsyrk", 3, 3)
    check(s("l", "n", 1, -1, 1, 1), "dsyrk", 4, 4)
    check(s("l", "n", 2, 1, 1, 2), "dsyrk", 7, 7)
    check(s("l", "t", 1, 2, 1, 1), "dsyrk", 7, 7)
    check(s("l", "n", 2, 1, 2, 1), "dsyrk", 10, 10)
    t = lambda sd, ul, tr, dg, m, n, lda, ldb: pb.dtrsm(sd, ul, tr, dg, m, n, 1.0, buf, lda, buf, ldb)
    check(t("x", "l", "n", "n", 1, 1, 1, 1), "dtrsm", 1, 1)
    check(t("l", "x", "n", "n", 1, 1, 1, 1), "dtrsm", 2, 2)
    check(t("l", "l", "x", "n", 1, 1, 1, 1), "dtrsm", 3, 3)
    check(t("l", "l", "n", "x", 1, 1, 1, 1), "dtrsm", 4, 4)
    check(t("l", "l", "n", "n", -1, 1, 1, 1), "dtrsm", 5, 5)
    check(t("l", "l", "n", "n", 1, -1, 1, 1), "dtrsm", 6, 6)
    check(t("l", "l", "n", "n", 2, 1, 1, 2), "dtrsm", 9, 9)
    check(t("r", "l", "n", "n", 1, 2, 1, 1), "dtrsm", 9, 9)
    check(t("l", "l", "n", "n", 2, 1, 2, 1), "dtrsm", 11, 11)
    check(t("l", "l", "n", "n", 0, 1, 1, 0), "dtrsm", 11, 11)  # validation precedes the quick return
    check(pb.dpotrf("x", 1, buf, 1), "dpotrf", 1, -1)
    check(pb.dpotrf("l", -1, buf, 1), "dpotrf", 2, -2)
    check(pb.dpotrf("l", 2, buf, 1), "dpotrf", 4, -4)
    ip = np.zeros(4, np.int32)
    check(pb.dgetrf(-1, 1, buf, 1, ip), "dgetrf", 1, -1)
    check(pb.dgetrf(1, -1, buf, 1, ip), "dgetrf", 2, -2)
    check(pb.dgetrf(2, 1, buf, 1, ip), "dgetrf", 4, -4)
    with pytest.raises(pb.ArgError) as e:
        pb.dgemm("x", "n", 1, 1, 1, 1.0, buf, 1, buf, 1, 0.0, buf, 1, cfg=pb.BlasConfig(abort_on_error=True))
    assert e.value.index == 1


def test_panel_validation(pb):
    b = np.zeros(64)
    P = pb.PanelRef
    assert pb.gemm_nd("t", "t", 4, 4, 4, 1.0, P(b, 4, 4), P(b, 4, 4), 0.0, P(b, 4, 4), P(b, 4, 4)).info == pb.INFO_UNSUPPORTED
    assert pb.gemm_nd("n", "t", -1, 4, 4, 1.0, P(b, 4, 4), P(b, 4, 4), 0.0, P(b, 4, 4), P(b, 4, 4)).info == -4
    assert pb.gemm_nd("n", "t", 4, 4, 4, 1.0, P(b, 4, 3), P(b, 4, 4), 0.0, P(b, 4, 4), P(b, 4, 4)).info == -8
    assert pb.gemm_nd("n", "t", 4, 4, 4, 1.0, P(b, 4, 4), P(b, 3, 4), 0.0, P(b, 4, 4), P(b, 4, 4)).info == -9
    assert pb.gemm_nd("n", "t", 4, 4, 4, 1.0, P(b, 4, 4), P(b, 4, 4), 0.0, P(b, 4, 5), P(b, 4, 4)).info == -11
    assert pb.gemm_nd("n", "t", 4, 4, 4, 1.0, P(b, 4, 4), P(b, 4, 4), 0.0, P(b, 4, 4), P(b, 4, 4, ps=8)).info == -12
    assert pb.syrk_nd(4, 2, 1.0, P(b, 4, 3), 1.0, P(b, 4, 4), P(b, 4, 4)).info == -5
    assert pb.trsm_rltn_nd(3, 4, 1.0, P(b, 4, 4), P(b, 3, 5), P(b, 3, 4)).info == -6
    assert pb.syrk_potrf_nd(4, 2, P(b, 4, 2), P(b, 4, 2), P(b, 4, 4), P(b, 4, 3)).info == -7


def test_no_cpu_fallback_without_device(pb):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    a = np.asfortranarray(np.eye(4))
    with pytest.raises(RuntimeError, match="no CUDA device"):
        pb.dgemm("n", "n", 4, 4, 4, 1.0, a, 4, a, 4, 0.0, a.copy(order="F"), 4)


def test_batched_null_info_rejected(pb):
    """Batched factorizations write info[p] per problem: a null info (or ipiv) is an
    argument error reported before anything is launched (extension argument positions)."""
    buf = np.zeros(64)
    r = pb.dpotrf_batched("l", 4, buf, 4, 16, None, 2)
    assert r.info == -7 and r.error.index == 7
    ip = np.zeros(8, np.int32); info = np.zeros(2, np.int32)
    r = pb.dgetrf_batched(4, 4, buf, 4, 16, None, 4, info, 2)
    assert r.info == -9 and r.error.index == 9
    r = pb.dgetrf_batched(4, 4, buf, 4, 16, ip, 4, None, 2)
    assert r.info == -10 and r.error.index == 10
    P = pb.PanelRef
    r = pb.syrk_potrf_nd_batched(4, 0, P(buf, 4, 0), 0, P(buf, 4, 0), 0, P(buf, 4, 4), 16, P(buf, 4, 4), 16, None, 2)
    assert r.info == -14


_SHIM_RUN = r'''
#include "pbgpu_panelblas.hpp"
#include "pb_oracle.h"
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
static double relf(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) { num += (a[i] - b[i]) * (a[i] - b[i]); den += b[i] * b[i]; }
  return std::sqrt(num / (den > 0 ? den : 1));
}
int main() {
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(-1, 1);
  pbgpu::BlasConfig cfg;
  const int n = 48;
  std::vector<double> A(n * n), B(n * n), C(n * n);
  for (auto* v : {&A, &B, &C}) for (auto& x : *v) x = u(rng);
  // dgemm through the reference-shaped signature vs the oracle
  std::vector<double> c1 = C, c2 = C;
  auto r = pbgpu::dgemm(cfg, 'n', 't', n, n, n, 1.5, A.data(), n, B.data(), n, -0.5, c1.data(), n);
  orc_dgemm('n', 't', n, n, n, 1.5, A.data(), n, B.data(), n, -0.5, c2.data(), n);
  if (!r.ok() || relf(c1, c2) > 1e-13 * n || r.flops != 2LL * n * n * n) { std::printf("dgemm\n"); return 1; }
  // dpotrf on an SPD matrix
  std::vector<double> S(n * n, 0.0);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
    for (int l = 0; l < n; ++l) S[i + j * n] += A[i + l * n] * A[j + l * n];
    if (i == j) S[i + j * n] += n;
  }
  std::vector<double> s1 = S, s2 = S;
  r = pbgpu::dpotrf(cfg, 'l', n, s1.data(), n);
  if (r.info != 0 || orc_dpotrf('l', n, s2.data(), n) != 0) { std::printf("dpotrf info\n"); return 2; }
  for (int j = 0; j < n; ++j) for (int i = 0; i < j; ++i) s1[i + j * n] = s2[i + j * n] = 0.0;
  if (relf(s1, s2) > 1e-13 * n) { std::printf("dpotrf\n"); return 3; }
  // dgetrf: pivots bit-exact
  std::vector<double> g1 = A, g2 = A;
  std::vector<int> p1, p2(n);
  r = pbgpu::dgetrf(cfg, n, n, g1.data(), n, p1);
  orc_dgetrf(n, n, g2.data(), n, p2.data());
  if (r.info != 0 || p1 != p2) { std::printf("dgetrf pivots\n"); return 4; }
  // argument error in abort mode throws ArgError with the reference's index
  pbgpu::BlasConfig strict;
  strict.abort_on_error = true;
  try { pbgpu::dpotrf(strict, 'x', n, s1.data(), n); return 5; } catch (const pbgpu::ArgError& e) {
    if (e.index() != 1) return 6;
  }
  std::printf("shim ok\n");
  return 0;
}
'''


@pytest.mark.gpu
def test_shim_compute_calls_match_the_oracle(tmp_path, orc):
    """Compute calls through the reference-shaped C++ signatures (pbgpu_panelblas.hpp) on the
    GPU: dgemm and dpotrf within 1e-13 n of the oracle, dgetrf pivots bit-exact, ArgError."""
    import subprocess
    src = tmp_path / "shim.cpp"
    src.write_text(_SHIM_RUN)
    exe = tmp_path / "shim"
    pkg = os.path.join(ROOT, "paper_1902_08115_b200")
    obuild = os.path.join(ROOT, "oracle", "_build")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
                        os.path.join(ROOT, "oracle"), str(src), "-o", str(exe),
                        os.path.join(pkg, "libpbgpu.so"), os.path.join(obuild, "liboracle.so"),
                        f"-Wl,-rpath,{pkg}:{obuild}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "shim ok" in out.stdout, (out.returncode, out.stdout, out.stderr)
