#!/usr/bin/env python3
"""Generates tests/golden/golden.npz from the REFERENCE itself.

Every expected output here is produced by the reference library compiled from
/root/reference/proj/include (oracle/_ref/libpanelblas_ref.so, see
oracle/Makefile), called through its own BLAS adapters and native panel
routines.  Inputs follow the recipes of the reference's own tests (cited per
case) and its seeded generator (matgen.hpp, std::mt19937_64).  Run here, where
/root/reference exists; the .npz is committed and travels to the GPU box.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import binding as ob  # noqa: E402

R = ob.ref()
out: dict[str, np.ndarray] = {}


def F(a):
    return np.asfortranarray(np.array(a, dtype=np.float64))


def rng_uniform(seed, count, lo=-1.0, hi=1.0):
    buf = np.empty(count)
    R.rng_uniform(seed, count, lo, hi, buf.ctypes.data)
    return buf


def fill(seed, m, n):
    """fill_uniform (matgen.hpp:30-33): column order from Rng(seed)."""
    return F(rng_uniform(seed, m * n).reshape(n, m).T)


def make_spd(n, seed):
    buf = np.empty(n * n)
    R.make_spd(n, seed, buf.ctypes.data)
    return F(buf.reshape(n, n).T)


def put(name, **arrs):
    for k, v in arrs.items():
        out[f"{name}/{k}"] = np.asarray(v)


# ---- dgemm: all four flag pairs, test_blas.cpp:44-95 shape (13, 9, 7), alpha 1.5, beta -0.5
for ta in "nt":
    for tb in "nt":
        m, n, k = 13, 9, 7
        a = fill(17, *((m, k) if ta == "n" else (k, m)))
        b = fill(18, *((k, n) if tb == "n" else (n, k)))
        c = fill(19, m, n)
        d = c.copy(order="F")
        assert R.dgemm(ta.encode(), tb.encode(), m, n, k, 1.5, a.ctypes.data, a.shape[0], b.ctypes.data,
                       b.shape[0], -0.5, d.ctypes.data, m) == 0
        put(f"dgemm_{ta}{tb}", a=a, b=b, c=c, out=d, mnk=[m, n, k], alpha=1.5, beta=-0.5)

# ---- dgemm config-1 shape: 3 problems of 64^3, alpha = beta = 1 (BASELINE.json configs[0])
for p in range(3):
    a, b, c = fill(100 + p, 64, 64), fill(200 + p, 64, 64), fill(300 + p, 64, 64)
    d = c.copy(order="F")
    R.dgemm(b"n", b"n", 64, 64, 64, 1.0, a.ctypes.data, 64, b.ctypes.data, 64, 1.0, d.ctypes.data, 64)
    put(f"dgemm_cfg1_{p}", a=a, b=b, c=c, out=d)

# ---- dsyrk both triangles / both transposes (test_blas.cpp:172-200: n 11, k 6, 1.25, -0.75)
for ul in "lu":
    for tr in "nt":
        n, k = 11, 6
        a = fill(29, *((n, k) if tr == "n" else (k, n)))
        c = fill(30, n, n)
        d = c.copy(order="F")
        R.dsyrk(ul.encode(), tr.encode(), n, k, 1.25, a.ctypes.data, a.shape[0], -0.75, d.ctypes.data, n)
        put(f"dsyrk_{ul}{tr}", a=a, c=c, out=d)

# ---- dpotrf: 2x2 worked example (test_factor.cpp:144-158), dyadic n=13 (195-249),
#      planted -2 pivot (251-277), random make_spd at config-3 sizes
a = F([[4.0, 2.0], [2.0, 5.0]])
for ul in "lu":
    d = a.copy(order="F")
    assert R.dpotrf(ul.encode(), 2, d.ctypes.data, 2) == 0
    put(f"dpotrf_2x2_{ul}", a=a, out=d, info=0)


def dyadic_chol_factor(n):
    l = np.zeros((n, n))
    for j in range(n):
        l[j, j] = float(1 << (j % 3)) * (0.5 if j % 2 else 1.0)
        for i in range(j + 1, n):
            pick = (i * 7 + j * 5) % 4
            v = 0.0 if pick == 0 else 0.25 * pick
            l[i, j] = -v if ((i + j) % 2 and pick != 0) else v
    return F(l)


l0 = dyadic_chol_factor(13)
a = F(l0 @ l0.T)
for ul in "lu":
    d = a.copy(order="F")
    assert R.dpotrf(ul.encode(), 13, d.ctypes.data, 13) == 0
    put(f"dpotrf_dyadic_{ul}", a=a, out=d, l0=l0, info=0)

a = make_spd(13, 71)
a[8, :] = 0.0
a[:, 8] = 0.0
a[8, 8] = -2.0
d = a.copy(order="F")
info = R.dpotrf(b"l", 13, d.ctypes.data, 13)
assert info == 9
put("dpotrf_planted", a=a, out=d, info=info)

for n in (16, 32, 64, 128):
    a = make_spd(n, 200 + n)
    d = a.copy(order="F")
    assert R.dpotrf(b"l", n, d.ctypes.data, n) == 0
    put(f"dpotrf_spd_{n}", a=a, out=d, info=0)

# ---- dgetrf: permutation / singular (test_factor.cpp:351-380), planted dyadic LU behind a
#      row rotation (395-440), zero pivot column (442-467), uniform config-4 sizes


def lu_plant(m, n, zero_col2=False):
    k = min(m, n)
    l = np.zeros((m, k))
    u = np.zeros((k, n))
    for j in range(k):
        l[j, j] = 1.0
        for i in range(j + 1, m):
            v = 0.25 if (i * 5 + j * 3) % 2 else 0.5
            l[i, j] = -v if (i + j) % 2 else v
    for i in range(k):
        u[i, i] = (-1.0 if i % 2 else 1.0) * float(1 << (1 + i % 3))
        for j in range(i + 1, n):
            u[i, j] = float((i * 3 + j * 5) % 9 - 4)
    if zero_col2:
        u[2, 2] = 0.0
        l[3:, 2] = 0.0
    return F(l @ u)


def getrf_case(name, a):
    m, n = a.shape
    d = a.copy(order="F")
    ip = np.zeros(min(m, n), np.int32)
    info = R.dgetrf(m, n, d.ctypes.data, m, ip.ctypes.data)
    put(name, a=a, out=d, ipiv=ip, info=info)


getrf_case("dgetrf_perm", F([[0.0, 1.0], [1.0, 0.0]]))
getrf_case("dgetrf_singular", F([[1.0, 2.0], [2.0, 4.0]]))
for (m, n) in [(13, 13), (9, 19), (19, 9)]:
    comp = lu_plant(m, n)
    a = F(np.zeros((m, n)))
    for i in range(m):
        a[(i + 3) % m, :] = comp[i, :]
    getrf_case(f"dgetrf_plant_{m}x{n}", a)
getrf_case("dgetrf_zero_col", lu_plant(6, 6, zero_col2=True))
for n in (24, 48, 96, 192):
    getrf_case(f"dgetrf_uniform_{n}", fill(400 + n, n, n))

# ---- dtrsm: all 16 flag combinations on diagonally dominant triangles (matgen make_tri style)
for sd in "lr":
    for ul in "lu":
        for tr in "nt":
            for dg in "nu":
                m, n = 9, 7
                t = m if sd == "l" else n
                a = fill(43, t, t)
                if dg == "u":
                    for j in range(t):
                        a[j, j] = 1.0
                else:
                    for j in range(t):
                        a[j, j] = (2.0 * t + 1.0) * (-1.0 if j % 2 else 1.0)
                b = fill(44, m, n)
                d = b.copy(order="F")
                assert R.dtrsm(sd.encode(), ul.encode(), tr.encode(), dg.encode(), m, n, 1.5, a.ctypes.data, t,
                               d.ctypes.data, m) == 0
                put(f"dtrsm_{sd}{ul}{tr}{dg}", a=a, b=b, out=d)

# ---- panel-major natives (ps = 4): gemm_nd NT/NN, syrk_nd, syrk_potrf_nd + trsm_rltn_nd
for tb in "nt":
    m, n, k = 9, 19, 13
    A = fill(51, m, k)
    B = fill(52, *((k, n) if tb == "n" else (n, k)))
    Cm = fill(53, m, n)
    ap, bp, cp = ob.pack(A, fill=np.nan), ob.pack(B, fill=np.nan), ob.pack(Cm, fill=np.nan)
    d = np.full(ob.panel_len(m, n), 9.0)
    br, bc = B.shape
    assert R.gemm_nd(b"n", tb.encode(), m, n, k, 0.75, ob.dmat(ap, m, k), ob.dmat(bp, br, bc), -1.25,
                     ob.dmat(cp, m, n), ob.dmat(d, m, n)) == 0
    put(f"gemm_nd_n{tb}", a=ap, b=bp, c=cp, out=d, mnk=[m, n, k], bshape=[br, bc])

n, k = 13, 7
A = fill(61, n, k)
Cs = fill(62, n, n)
ap, cp = ob.pack(A), ob.pack(Cs)
d = np.full(ob.panel_len(n, n), 3.5)
assert R.syrk_nd(n, k, 1.0, ob.dmat(ap, n, k), 1.0, ob.dmat(cp, n, n), ob.dmat(d, n, n)) == 0
put("syrk_nd", a=ap, c=cp, out=d, nk=[n, k])

for n in (6, 13, 21, 64):
    k = 7
    A = fill(70 + n, n, k)
    S = make_spd(n, 80 + n)
    ap, sp = ob.pack(A), ob.pack(S)
    d = np.full(ob.panel_len(n, n), 64.125)
    assert R.syrk_potrf_nd(n, k, ob.dmat(ap, n, k), ob.dmat(ap, n, k), ob.dmat(sp, n, n), ob.dmat(d, n, n)) == 0
    Bm = fill(90 + n, 11, n)
    bp = ob.pack(Bm)
    x = np.full(ob.panel_len(11, n), 2.5)
    assert R.trsm_rltn_nd(11, n, 1.5, ob.dmat(d, n, n), ob.dmat(bp, 11, n), ob.dmat(x, 11, n)) == 0
    put(f"chain_nd_{n}", a=ap, c=sp, l=d, b=bp, x=x, nk=[n, k])

# ---- dtrmm: all 16 flag combinations (bench.hpp:548-583 verify recipe shape), alpha 1.5
for sd in "lr":
    for ul in "lu":
        for tr in "nt":
            for dg in "nu":
                m, n = 9, 7
                t = m if sd == "l" else n
                a = fill(45, t, t)
                b = fill(46, m, n)
                d = b.copy(order="F")
                assert R.dtrmm(sd.encode(), ul.encode(), tr.encode(), dg.encode(), m, n, 1.5, a.ctypes.data, t,
                               d.ctypes.data, m) == 0
                put(f"dtrmm_{sd}{ul}{tr}{dg}", a=a, b=b, out=d)

# ---- trmm_rlnn_nd (level3.hpp:446-479), the Riccati stage's first call (riccati.hpp:319)
for (m, n) in ((11, 7), (13, 16)):
    A = fill(47, n, n)
    Bm = fill(48, m, n)
    ap, bp = ob.pack(A, fill=7.5), ob.pack(Bm, fill=-3.0)
    d = np.full(ob.panel_len(m, n), 1.25)
    assert R.trmm_rlnn_nd(m, n, 1.5, ob.dmat(ap, n, n), ob.dmat(bp, m, n), ob.dmat(d, m, n)) == 0
    put(f"trmm_nd_{m}x{n}", a=ap, b=bp, d0=np.full(ob.panel_len(m, n), 1.25), out=d, mn=[m, n])

# ---- pack / unpack (panel_mat.hpp:141-171), pad lanes untouched
for (m, n, tr) in ((9, 6, "n"), (9, 6, "t"), (4, 8, "n")):
    src = fill(49, *((m, n) if tr == "n" else (n, m)))
    d = np.full(ob.panel_len(m, n), -2.75)
    R.pack_from_colmajor(tr.encode(), src.ctypes.data, src.shape[0], src.shape[0], src.shape[1], ob.dmat(d, m, n))
    back = F(np.zeros((m, n)))
    R.unpack_to_colmajor(ob.dmat(d, m, n), back.ctypes.data, m)
    put(f"pack_{m}x{n}{tr}", src=src, out=d, back=back)

# ---- Riccati (riccati.hpp): make_ocp_data + RiccatiFusedWork stage factors, riccati_run residuals
for (nx, nu, N) in ((4, 2, 3), (6, 3, 5), (8, 4, 10)):
    seed = 1234 + nx
    a = np.zeros(nx * nx); b = np.zeros(nx * nu); q = np.zeros(nx * nx); r = np.zeros(nu * nu); s_ = np.zeros(nu * nx)
    R.make_ocp_data(nx, nu, seed, a.ctypes.data, b.ctypes.data, q.ctypes.data, r.ctypes.data, s_.ctypes.data)
    nt = nx + nu
    fst = np.zeros(N * nt * nt); lt = np.zeros(nx * nx)
    import ctypes
    fs = ctypes.c_int(0)
    assert R.riccati_fused(nx, nu, N, seed, fst.ctypes.data, lt.ctypes.data, ctypes.byref(fs)) == 0
    info = ctypes.c_int(0)
    res = [R.riccati_run(nx, nu, N, impl, seed, ctypes.byref(info)) for impl in (0, 1, 2)]
    put(f"riccati_{nx}_{nu}_{N}", a=a, b=b, q=q, r=r, s=s_, f=fst, lterm=lt, dims=[nx, nu, N, seed],
        residual=np.array(res))

# seeded generator check values (matgen.hpp:14-28): Rng(42).uniform() x 8
put("rng42", u=rng_uniform(42, 8))

np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
print(f"wrote {len(out)} arrays to {os.path.join(HERE, 'golden.npz')}")
