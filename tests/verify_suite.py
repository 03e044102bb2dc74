"""GPU differential verify suite — the analogue of the reference's verify_suite
(bench.hpp:485-646) with the GPU library in the engine's place.

`count` random cases per routine / flag family with dimensions in [1, 96]; each
runs through the public C ABI (host pointers, so every case goes host -> GPU ->
host) and is compared with the CPU oracle restatement at the reference's
tolerances: 1e-13 normwise (max |got - want| / max(1, ||want||_F)) for products,
solves and factor entries, plus reconstruction at 1e-12 * max(1, ||A||_F) for the
factorizations and bit-exact pivots for dgetrf.  Test infrastructure only (it
loads the oracle); run clean it must pass, and under PBGPU_MUTATE it must fail
(tests/test_gpu_round2.py::test_mutation_negative_control).
"""
from __future__ import annotations

import numpy as np


def _F(a):
    return np.asfortranarray(a, dtype=np.float64)


def normwise_dev(got, want):
    """bench.hpp:452-456."""
    scale = max(1.0, float(np.linalg.norm(want)))
    return float(np.abs(got - want).max()) / scale if got.size else 0.0


def make_tri(rng, uplo, diag, n):
    """matgen.hpp make_tri: well-conditioned triangle (dominant diagonal)."""
    a = rng.uniform(-1, 1, (n, n))
    a[np.arange(n), np.arange(n)] = (n + 1.0) * np.where(rng.uniform(0, 1, n) < 0.5, -1.0, 1.0)
    return _F(a)


def run(pb, orc, seed: int = 42, count: int = 8, filt: str = "") -> dict:
    rng = np.random.default_rng(seed)
    dim = lambda: int(rng.integers(1, 97))
    rep = {"cases_run": 0, "failures": 0, "failed": []}

    def record(routine, flags, m, n, k, dev, tolr, ok):
        rep["cases_run"] += 1
        if not (ok and dev <= tolr):
            rep["failures"] += 1
            rep["failed"].append({"routine": routine, "flags": flags, "m": m, "n": n, "k": k,
                                  "deviation": dev, "tolerance": tolr})

    hit = lambda r: not filt or filt == "all" or filt in r
    p = lambda x: x.ctypes.data
    if hit("dgemm"):
        for c in range(count):
            ta, tb = "nt"[c % 2], "nt"[(c // 2) % 2]
            m, n, k = dim(), dim(), dim()
            a = _F(rng.uniform(-1, 1, (m, k) if ta == "n" else (k, m)))
            b = _F(rng.uniform(-1, 1, (k, n) if tb == "n" else (n, k)))
            cm = _F(rng.uniform(-1, 1, (m, n)))
            al, be = rng.uniform(-2, 2), rng.uniform(-2, 2)
            got, want = cm.copy(order="F"), cm.copy(order="F")
            r = pb.dgemm(ta, tb, m, n, k, al, a, a.shape[0], b, b.shape[0], be, got, m)
            orc.dgemm(ta.encode(), tb.encode(), m, n, k, al, p(a), a.shape[0], p(b), b.shape[0], be, p(want), m)
            record("dgemm", ta + tb, m, n, k, normwise_dev(got, want), 1e-13, r.ok())
    if hit("dsyrk"):
        for c in range(count):
            ul, tr = "lu"[c % 2], "nt"[(c // 2) % 2]
            n, k = dim(), dim()
            a = _F(rng.uniform(-1, 1, (n, k) if tr == "n" else (k, n)))
            cm = _F(rng.uniform(-1, 1, (n, n)))
            al, be = rng.uniform(-2, 2), rng.uniform(-2, 2)
            got, want = cm.copy(order="F"), cm.copy(order="F")
            r = pb.dsyrk(ul, tr, n, k, al, a, a.shape[0], be, got, n)
            orc.dsyrk(ul.encode(), tr.encode(), n, k, al, p(a), a.shape[0], be, p(want), n)
            record("dsyrk", ul + tr, n, n, k, normwise_dev(got, want), 1e-13, r.ok())
    for solve in (False, True):
        name = "dtrsm" if solve else "dtrmm"
        if not hit(name):
            continue
        for c in range(count):
            sd, ul, tr, dg = "lr"[c % 2], "lu"[(c // 2) % 2], "nt"[(c // 4) % 2], "nu"[(c // 8) % 2]
            m, n = dim(), dim()
            t = m if sd == "l" else n
            a = make_tri(rng, ul, dg, t)
            b = _F(rng.uniform(-1, 1, (m, n)))
            al = rng.uniform(-2, 2)
            got, want = b.copy(order="F"), b.copy(order="F")
            fn = pb.dtrsm if solve else pb.dtrmm
            ofn = orc.dtrsm if solve else orc.dtrmm
            r = fn(sd, ul, tr, dg, m, n, al, a, t, got, m)
            oi = ofn(sd.encode(), ul.encode(), tr.encode(), dg.encode(), m, n, al, p(a), t, p(want), m)
            record(name, sd + ul + tr + dg, m, n, 0, normwise_dev(got, want), 1e-13, r.ok() and oi == 0)
    if hit("dpotrf"):
        for c in range(count):
            ul = "lu"[c % 2]
            n = dim()
            g = rng.uniform(-1, 1, (n, n))
            a = _F(g @ g.T + n * np.eye(n))
            got, want = a.copy(order="F"), a.copy(order="F")
            r = pb.dpotrf(ul, n, got, n)
            oi = orc.dpotrf(ul.encode(), n, p(want), n)
            tri = np.tril(np.ones((n, n), bool)) if ul == "l" else np.triu(np.ones((n, n), bool))
            dev = normwise_dev(np.where(tri, got, 0), np.where(tri, want, 0))
            L = np.where(tri, got, 0)
            rec = L @ L.T if ul == "l" else L.T @ L
            recon = float(np.abs(rec - a).max()) / max(1.0, float(np.linalg.norm(a)))
            record("dpotrf", ul, n, n, 0, max(dev, recon), 1e-12, r.ok() and oi == 0 and dev <= 1e-13)
    if hit("dgetrf"):
        for c in range(count):
            m, n = dim(), dim()
            a = _F(rng.uniform(-1, 1, (m, n)))
            got, want = a.copy(order="F"), a.copy(order="F")
            gp, wp = np.zeros(min(m, n), np.int32), np.zeros(min(m, n), np.int32)
            r = pb.dgetrf(m, n, got, m, gp)
            oi = orc.dgetrf(m, n, p(want), m, p(wp))
            record("dgetrf", "", m, n, 0, normwise_dev(got, want), 1e-13,
                   r.info == oi and np.array_equal(gp, wp))
    return rep


if __name__ == "__main__":
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1902_08115_b200 as pb
    from oracle import binding as ob
    out = run(pb, ob.oracle(), count=int(sys.argv[1]) if len(sys.argv) > 1 else 8)
    print(out["cases_run"], "cases,", out["failures"], "failures")
    for f in out["failed"]:
        print(f)
