"""CPU: the oracle restatement is pinned to the reference (golden fixtures + compiled reference)."""
import os

import numpy as np
import pytest

from helpers import F, ch, ptr, same_bits
from oracle import binding as ob

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def cases(prefix):
    return sorted({k.split("/")[0] for k in GOLD.files if k.startswith(prefix)})


def g(case, key):
    return GOLD[f"{case}/{key}"]


@pytest.mark.parametrize("case", cases("dgemm_"))
def test_golden_dgemm(orc, case):
    a, b, c, out = (F(g(case, x)) for x in "a b c out".split())
    if case.startswith("dgemm_cfg1"):
        ta, tb, (m, n, k), al, be = "n", "n", (64, 64, 64), 1.0, 1.0
    else:
        ta, tb = case[-2], case[-1]
        m, n, k = g(case, "mnk"); al, be = float(g(case, "alpha")), float(g(case, "beta"))
    d = c.copy(order="F")
    assert orc.dgemm(ch(ta), ch(tb), int(m), int(n), int(k), al, ptr(a), a.shape[0], ptr(b), b.shape[0], be, ptr(d), int(m)) == 0
    assert same_bits(d, out)


@pytest.mark.parametrize("case", cases("dsyrk_"))
def test_golden_dsyrk(orc, case):
    a, c, out = (F(g(case, x)) for x in "a c out".split())
    ul, tr = case[-2], case[-1]
    n = c.shape[0]; k = a.shape[1] if tr == "n" else a.shape[0]
    d = c.copy(order="F")
    orc.dsyrk(ch(ul), ch(tr), n, k, 1.25, ptr(a), a.shape[0], -0.75, ptr(d), n)
    assert same_bits(d, out)


@pytest.mark.parametrize("case", cases("dpotrf_"))
def test_golden_dpotrf(orc, case):
    a, out = F(g(case, "a")), F(g(case, "out"))
    ul = "u" if case.endswith("_u") else "l"
    d = a.copy(order="F")
    assert orc.dpotrf(ch(ul), a.shape[0], ptr(d), a.shape[0]) == int(g(case, "info"))
    assert same_bits(d, out)
    if "dyadic" in case:  # the planted factor itself (test_factor.cpp:195-249)
        l0 = F(g(case, "l0"))
        tri = np.tril(np.ones(l0.shape, bool))
        assert same_bits(d[tri] if ul == "l" else d.T[tri], l0[tri])


@pytest.mark.parametrize("case", cases("dgetrf_"))
def test_golden_dgetrf(orc, case):
    a, out = F(g(case, "a")), F(g(case, "out"))
    m, n = a.shape
    d = a.copy(order="F"); ip = np.zeros(min(m, n), np.int32)
    assert orc.dgetrf(m, n, ptr(d), m, ptr(ip)) == int(g(case, "info"))
    assert np.array_equal(ip, g(case, "ipiv")) and same_bits(d, out)


@pytest.mark.parametrize("case", cases("dtrsm_"))
def test_golden_dtrsm(orc, case):
    a, b, out = F(g(case, "a")), F(g(case, "b")), F(g(case, "out"))
    sd, ul, tr, dg = case[-4:]
    m, n = b.shape
    d = b.copy(order="F")
    assert orc.dtrsm(ch(sd), ch(ul), ch(tr), ch(dg), m, n, 1.5, ptr(a), a.shape[0], ptr(d), m) == 0
    assert same_bits(d, out)


def test_golden_panel(orc):
    for tb in "nt":
        case = f"gemm_nd_n{tb}"
        m, n, k = (int(x) for x in g(case, "mnk")); br, bc = (int(x) for x in g(case, "bshape"))
        a, b, c = g(case, "a").copy(), g(case, "b").copy(), g(case, "c").copy()
        d = np.full(ob.panel_len(m, n), 9.0)
        assert orc.gemm_nd(b"n", ch(tb), m, n, k, 0.75, ob.dmat(a, m, k), ob.dmat(b, br, bc), -1.25, ob.dmat(c, m, n), ob.dmat(d, m, n)) == 0
        assert same_bits(d, g(case, "out"))
    n, k = (int(x) for x in g("syrk_nd", "nk"))
    a, c = g("syrk_nd", "a").copy(), g("syrk_nd", "c").copy()
    d = np.full(ob.panel_len(n, n), 3.5)
    orc.syrk_nd(n, k, 1.0, ob.dmat(a, n, k), 1.0, ob.dmat(c, n, n), ob.dmat(d, n, n))
    assert same_bits(d, g("syrk_nd", "out"))
    for case in cases("chain_nd_"):
        n, k = (int(x) for x in g(case, "nk"))
        a, c, b = g(case, "a").copy(), g(case, "c").copy(), g(case, "b").copy()
        d = np.full(ob.panel_len(n, n), 64.125)
        assert orc.syrk_potrf_nd(n, k, ob.dmat(a, n, k), ob.dmat(a, n, k), ob.dmat(c, n, n), ob.dmat(d, n, n)) == 0
        assert same_bits(d, g(case, "l"))
        x = np.full(ob.panel_len(11, n), 2.5)
        assert orc.trsm_rltn_nd(11, n, 1.5, ob.dmat(d, n, n), ob.dmat(b, 11, n), ob.dmat(x, 11, n)) == 0
        assert same_bits(x, g(case, "x"))


@pytest.mark.skipif(not ob.have_ref(), reason="oracle/_ref not built (needs /root/reference)")
def test_restatement_equals_reference_on_random_inputs(orc):
    """Bit-for-bit agreement with the reference compiled from its own headers."""
    R = ob.ref()
    rng = np.random.default_rng(1)
    for trial in range(12):
        m, n, k = (int(x) for x in rng.integers(1, 40, 3))
        for ta in "nt":
            for tb in "nt":
                a = F(rng.uniform(-1, 1, (m, k) if ta == "n" else (k, m)))
                b = F(rng.uniform(-1, 1, (k, n) if tb == "n" else (n, k)))
                c = F(rng.uniform(-1, 1, (m, n)))
                c1, c2 = c.copy(order="F"), c.copy(order="F")
                orc.dgemm(ch(ta), ch(tb), m, n, k, 1.5, ptr(a), a.shape[0], ptr(b), b.shape[0], -0.5, ptr(c1), m)
                R.dgemm(ch(ta), ch(tb), m, n, k, 1.5, ptr(a), a.shape[0], ptr(b), b.shape[0], -0.5, ptr(c2), m)
                assert same_bits(c1, c2)
        gg = rng.uniform(-1, 1, (n, n)); s = F(gg @ gg.T + n * np.eye(n))
        if trial % 3 == 0:
            s[n // 2, n // 2] = -1.0
        for ul in "lu":
            a1, a2 = s.copy(order="F"), s.copy(order="F")
            assert orc.dpotrf(ch(ul), n, ptr(a1), n) == R.dpotrf(ch(ul), n, ptr(a2), n)
            assert same_bits(a1, a2)
        a = F(rng.uniform(-1, 1, (m, n)))
        if trial % 4 == 0:
            a[:, min(m, n) // 2] = 0.0
        a1, a2 = a.copy(order="F"), a.copy(order="F")
        p1, p2 = np.zeros(min(m, n), np.int32), np.zeros(min(m, n), np.int32)
        assert orc.dgetrf(m, n, ptr(a1), m, ptr(p1)) == R.dgetrf(m, n, ptr(a2), m, ptr(p2))
        assert same_bits(a1, a2) and np.array_equal(p1, p2)
        for sd in "lr":
            for ul in "lu":
                for tr in "nt":
                    for dg in "nu":
                        t = m if sd == "l" else n
                        A = F(rng.uniform(-1, 1, (t, t))); A[np.arange(t), np.arange(t)] = 2 * t + 1.0
                        B = F(rng.uniform(-1, 1, (m, n))); b1, b2 = B.copy(order="F"), B.copy(order="F")
                        i1 = orc.dtrsm(ch(sd), ch(ul), ch(tr), ch(dg), m, n, 1.5, ptr(A), t, ptr(b1), m)
                        i2 = R.dtrsm(ch(sd), ch(ul), ch(tr), ch(dg), m, n, 1.5, ptr(A), t, ptr(b2), m)
                        assert i1 == i2 and same_bits(b1, b2)


@pytest.mark.skipif(not ob.have_ref(), reason="oracle/_ref not built (needs /root/reference)")
def test_naive_second_opinion(orc):
    """reference.hpp naive loops agree with the fast-path restatement (1e-13 normwise, pivots equal)."""
    R = ob.ref()
    rng = np.random.default_rng(5)
    for n in (7, 24, 48):
        a = F(rng.uniform(-1, 1, (n, n)))
        a1, a2 = a.copy(order="F"), a.copy(order="F")
        p1, p2 = np.zeros(n, np.int32), np.zeros(n, np.int32)
        orc.dgetrf(n, n, ptr(a1), n, ptr(p1)); R.naive_getrf(n, n, ptr(a2), n, ptr(p2))
        assert np.array_equal(p1, p2)
        assert np.abs(a1 - a2).max() <= 1e-12 * max(1.0, np.linalg.norm(a))


def test_argument_validation_matches_reference(orc):
    """Fortran-order argument indices (test_blas.cpp:97-119)."""
    buf = np.zeros(16)
    call = lambda ta, tb, m, n, k, lda, ldb, ldc: orc.dgemm(ch(ta), ch(tb), m, n, k, 1.0, ptr(buf), lda, ptr(buf), ldb, 0.0, ptr(buf), ldc)
    assert call("x", "t", 2, 2, 2, 2, 2, 2) == 1
    assert call("n", "q", 2, 2, 2, 2, 2, 2) == 2
    assert call("n", "n", -1, 2, 2, 2, 2, 2) == 3
    assert call("n", "n", 2, -1, 2, 2, 2, 2) == 4
    assert call("n", "n", 2, 2, -1, 2, 2, 2) == 5
    assert call("n", "n", 2, 2, 2, 1, 2, 2) == 8
    assert call("t", "n", 2, 2, 3, 2, 3, 2) == 8
    assert call("n", "n", 2, 2, 2, 2, 1, 2) == 10
    assert call("n", "t", 2, 3, 2, 2, 2, 2) == 10
    assert call("n", "n", 2, 2, 2, 2, 2, 1) == 13
    assert call("x", "q", -1, -1, -1, 0, 0, 0) == 1


# ---------------------------------------------------------------- round 2: trmm, pack, chain, Riccati
@pytest.mark.parametrize("case", cases("dtrmm_"))
def test_golden_dtrmm(orc, case):
    a, b, out = (F(g(case, x)) for x in "a b out".split())
    sd, ul, tr, dg = case[-4:]
    m, n = b.shape
    d = b.copy(order="F")
    assert orc.dtrmm(ch(sd), ch(ul), ch(tr), ch(dg), m, n, 1.5, ptr(a), a.shape[0], ptr(d), m) == 0
    assert same_bits(d, out)


@pytest.mark.parametrize("case", cases("trmm_nd_"))
def test_golden_trmm_rlnn_nd(orc, case):
    m, n = (int(x) for x in g(case, "mn"))
    ap, bp, d = g(case, "a").copy(), g(case, "b").copy(), g(case, "d0").copy()
    assert orc.trmm_rlnn_nd(m, n, 1.5, ob.dmat(ap, n, n), ob.dmat(bp, m, n), ob.dmat(d, m, n)) == 0
    assert same_bits(d, g(case, "out"))
    io = bp.copy()  # b aliases d (level3.hpp:443-445)
    assert orc.trmm_rlnn_nd(m, n, 1.5, ob.dmat(ap, n, n), ob.dmat(io, m, n), ob.dmat(io, m, n)) == 0
    assert same_bits(ob.unpack(io, m, n), ob.unpack(g(case, "out"), m, n))


@pytest.mark.parametrize("case", cases("pack_"))
def test_golden_pack(case):
    src, out = F(g(case, "src")), g(case, "out")
    tr = case[-1]
    m, n = (src.shape if tr == "n" else src.shape[::-1])
    d = np.full(ob.panel_len(m, n), -2.75)
    i = np.arange(m)[:, None]; j = np.arange(n)[None, :]
    cn = ob.round_up(n, 4)
    d[(i // 4) * 4 * cn + j * 4 + i % 4] = src if tr == "n" else src.T
    assert same_bits(d, out)
    assert same_bits(ob.unpack(out, m, n), F(g(case, "back")))


@pytest.mark.parametrize("case", cases("riccati_"))
def test_golden_riccati_fused(orc, case):
    """The oracle's composition of the packed stage loop reproduces RiccatiFusedWork bit for bit."""
    import riccati_ref as rr
    nx, nu, N, seed = (int(x) for x in g(case, "dims"))
    nt = nx + nu
    a = g(case, "a").reshape(nx, nx).T; b = g(case, "b").reshape(nu, nx).T
    q = g(case, "q").reshape(nx, nx).T; r = g(case, "r").reshape(nu, nu).T; s = g(case, "s").reshape(nx, nu).T
    m0p, qp, gp = rr.stage_data(a, b, q, r, s)
    fs, lterm, info, st = rr.fused_oracle(orc, m0p, qp, gp, nx, nu, N)
    assert info == 0
    assert same_bits(ob.unpack(lterm, nx, nx), F(g(case, "lterm").reshape(nx, nx).T))
    want = g(case, "f").reshape(N, nt, nt)
    for s_ in range(N):
        got = np.tril(ob.unpack(fs[s_], nt, nt))
        assert same_bits(F(got), F(want[s_].T))
    # whole-horizon residual (riccati_run) is tiny for every reference path
    assert (g(case, "residual") <= 1e-10).all()
    P = rr.textbook(a, b, q, r, s, N)
    for s_ in range(N):
        assert rr.chol_residual(ob.unpack(fs[s_], nt, nt)[nu:, nu:], P[s_]) <= 1e-10


@pytest.mark.skipif(not ob.have_ref(), reason="oracle/_ref not built (needs /root/reference)")
def test_round2_restatements_equal_reference(orc):
    """dtrmm (16 flag sets), trmm_rlnn_nd, the threaded gemm_nd and chain loops: bit for bit."""
    R = ob.ref()
    rng = np.random.default_rng(11)
    for trial in range(4):
        m, n = (int(x) for x in rng.integers(1, 30, 2))
        for sd in "lr":
            for ul in "lu":
                for tr in "nt":
                    for dg in "nu":
                        t = m if sd == "l" else n
                        A = F(rng.uniform(-1, 1, (t, t)))
                        B = F(rng.uniform(-1, 1, (m, n))); b1, b2 = B.copy(order="F"), B.copy(order="F")
                        i1 = orc.dtrmm(ch(sd), ch(ul), ch(tr), ch(dg), m, n, -0.75, ptr(A), t, ptr(b1), m)
                        i2 = R.dtrmm(ch(sd), ch(ul), ch(tr), ch(dg), m, n, -0.75, ptr(A), t, ptr(b2), m)
                        assert i1 == i2 == 0 and same_bits(b1, b2)
        A = rng.uniform(-1, 1, (n, n)); Bm = rng.uniform(-1, 1, (m, n))
        ap, bp = ob.pack(A), ob.pack(Bm)
        d1, d2 = np.full(ob.panel_len(m, n), 3.0), np.full(ob.panel_len(m, n), 3.0)
        assert orc.trmm_rlnn_nd(m, n, 0.5, ob.dmat(ap, n, n), ob.dmat(bp, m, n), ob.dmat(d1, m, n)) == 0
        assert R.trmm_rlnn_nd(m, n, 0.5, ob.dmat(ap, n, n), ob.dmat(bp, m, n), ob.dmat(d2, m, n)) == 0
        assert same_bits(d1, d2)
    # threaded loops over a small batch
    s = 12; batch = 9; L = s * s
    A, B, Cp = (rng.uniform(-1, 1, (batch, L)) for _ in range(3))
    D1, D2 = np.zeros((batch, L)), np.zeros((batch, L))
    dm = lambda x: ob.dmat(x, s, s)
    orc.gemm_nd_batch(b"n", b"t", s, s, s, 1.0, dm(A), L, dm(B), L, 1.0, dm(Cp), L, dm(D1), L, batch, 4)
    R.gemm_nd_batch(b"n", b"t", s, s, s, 1.0, dm(A), L, dm(B), L, 1.0, dm(Cp), L, dm(D2), L, batch, 4)
    assert same_bits(D1, D2)
    ns = (rng.integers(1, 17, 40) * 4).astype(np.int32)
    offs = np.concatenate([[0], np.cumsum(ns.astype(np.int64) ** 2)[:-1]]).astype(np.int64)
    tot = int((ns.astype(np.int64) ** 2).sum())
    for pm in (0, 1):
        Av = rng.uniform(-1, 1, tot); Bv = rng.uniform(-1, 1, tot)
        Cv = np.zeros(tot)
        for n_, o in zip(ns, offs):
            n_ = int(n_)
            idx = np.arange(n_)
            Cv[o + (idx * (n_ + 1) if pm == 0 else (idx // 4) * 4 * n_ + idx * 4 + idx % 4)] = n_
        outs = []
        for lib, fn in ((orc, "chain_batch"), (R, "chain_cm_batch" if pm == 0 else "chain_pm_batch")):
            a_, c_, b_ = Av.copy(), Cv.copy(), Bv.copy(); info = np.full(len(ns), -1, np.int32)
            args = (ptr(ns), ptr(offs), ptr(a_), ptr(c_), ptr(b_), ptr(info), len(ns), 4)
            getattr(lib, fn)(*((pm,) + args if fn == "chain_batch" else args))
            outs.append((c_, b_, info))
        assert same_bits(outs[0][0], outs[1][0]) and same_bits(outs[0][1], outs[1][1])
        assert np.array_equal(outs[0][2], outs[1][2]) and (outs[0][2] == 0).all()
