"""Full-size parity of every BASELINE.json config against the CPU oracle.

The GPU runs each config at its full size; the oracle (the reference compiled from its own
headers, oracle/_ref, or the bit-pinned C restatement where that is absent) recomputes

* cfg1: all 16384 dgemm_nn 64^3 problems;
* cfg2: all 80 sizes s = 4..320 — a seeded subset of >= 1024 problems per size that always
  holds the first and last problem (the whole batch where it is smaller than 1024);
* cfg3: all 8192 problems at each n (info equal, L within 1e-13 n forward, and the backward
  error of every problem on the device);
* cfg4: all 8192 problems at each n — the pivot-mismatch count must be 0;
* cfg5: cm and pm chains on a seeded 1024-problem subset (first and last included) of the
  32768-problem batch.

Tolerances are the north star's: relative Frobenius error <= 1e-13 n (tests/helpers.tol).
With PBGPU_PARITY_OUT set, the per-config worst errors are written there as JSON (the
``parity`` evidence under profiles/).
"""
import json
import os

import numpy as np
import pytest

from helpers import tol
from oracle import binding as ob

pytestmark = pytest.mark.gpu

THREADS = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1)
SUMMARY: dict = {}


def _cpu():
    """The reference itself where it was compiled (oracle/_ref), else the pinned restatement."""
    return ob.ref() if ob.have_ref() else ob.oracle()


def _record(key, **kv):
    SUMMARY[key] = kv
    out = os.environ.get("PBGPU_PARITY_OUT")
    if out:
        prev = {}
        if os.path.exists(out):
            with open(out) as f:
                prev = json.load(f)
        prev[key] = kv
        prev["_oracle"] = "oracle/_ref (reference compiled)" if ob.have_ref() else "oracle restatement"
        prev["_threads"] = THREADS
        with open(out, "w") as f:
            json.dump(prev, f, indent=1, sort_keys=True)


def _subset(batch, want, seed):
    """Seeded sorted subset of `want` indices that always holds the first and last problem."""
    if batch <= want:
        return np.arange(batch)
    rng = np.random.default_rng(seed)
    mid = rng.choice(np.arange(1, batch - 1), want - 2, replace=False)
    return np.unique(np.concatenate([[0, batch - 1], mid]))


def _rel_rows(got, want):
    """Per-problem relative Frobenius error of (batch, L) arrays."""
    den = np.linalg.norm(want, axis=1)
    den[den == 0] = 1.0
    return np.linalg.norm(got - want, axis=1) / den


# ----------------------------------------------------------------------------------------- cfg1
def test_cfg1_all_problems_vs_oracle(pb, cuda):
    import torch
    m = n = k = 64
    batch = 16384
    rng = np.random.default_rng(101)
    A = rng.uniform(-1, 1, (batch, m * k))
    B = rng.uniform(-1, 1, (batch, k * n))
    C = rng.uniform(-1, 1, (batch, m * n))
    dA, dB, dC = (torch.from_numpy(x).to(cuda) for x in (A, B, C))
    assert pb.dgemm_batched("n", "n", m, n, k, 1.0, dA, m, m * k, dB, k, k * n, 1.0, dC, m, m * n,
                            batch).ok()
    got = dC.cpu().numpy()
    want = C.copy()
    _cpu().dgemm_batch(b"n", b"n", m, n, k, 1.0, A.ctypes.data, m, m * k, B.ctypes.data, k, k * n, 1.0,
                       want.ctypes.data, m, m * n, batch, THREADS)
    err = _rel_rows(got, want)
    _record("cfg1", problems_checked=batch, of=batch, max_rel_frob=float(err.max()), tol=tol(k))
    assert err.max() <= tol(k), (int(err.argmax()), err.max())


# ----------------------------------------------------------------------------------------- cfg2
def test_cfg2_all_sizes_vs_oracle(pb, cuda):
    import torch
    R = pb.PanelRef
    cpu = _cpu()
    worst = {}
    checked = 0
    for s in range(4, 321, 4):
        batch = (2 ** 31) // (32 * s * s)
        L = s * s
        g = torch.Generator(device=cuda).manual_seed(2000 + s)
        A = torch.rand((batch, L), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
        B = torch.rand((batch, L), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
        Cm = torch.rand((batch, L), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
        D = torch.full_like(A, float("nan"))
        assert pb.gemm_nd_batched("n", "t", s, s, s, 1.0, R(A, s, s), L, R(B, s, s), L, 1.0, R(Cm, s, s), L,
                                  R(D, s, s), L, batch).ok()
        idx = torch.from_numpy(_subset(batch, 1024, s)).to(cuda)
        a, b, c, d = (x[idx].cpu().numpy() for x in (A, B, Cm, D))
        del A, B, Cm, D
        want = np.empty_like(d)
        nb = len(a)
        dm = lambda buf: ob.dmat(buf, s, s)  # noqa: E731
        cpu.gemm_nd_batch(b"n", b"t", s, s, s, 1.0, dm(a), L, dm(b), L, 1.0, dm(c), L, dm(want), L, nb,
                          THREADS)
        err = _rel_rows(d, want)
        worst[s] = float(err.max())
        checked += nb
        assert err.max() <= tol(s), (s, int(err.argmax()), err.max())
    _record("cfg2", sizes=80, problems_checked=checked, max_rel_frob_over_tol=max(worst[s] / tol(s) for s in worst),
            max_rel_frob_by_s={str(s): v for s, v in worst.items()},
            subset="seeded 1024 per size incl. first and last (whole batch where smaller)")


# ----------------------------------------------------------------------------------------- cfg3
@pytest.mark.parametrize("n", [16, 32, 64, 128, 256])
def test_cfg3_all_problems_vs_oracle(pb, cuda, n):
    import torch
    batch = 8192
    g = torch.Generator(device=cuda).manual_seed(300 + n)
    G = torch.randn((batch, n, n), generator=g, device=cuda, dtype=torch.float64)
    A0 = G @ G.transpose(1, 2) + n * torch.eye(n, device=cuda, dtype=torch.float64)
    del G
    A = A0.clone()
    info = torch.full((batch,), -7, dtype=torch.int32, device=cuda)
    assert pb.dpotrf_batched("l", n, A, n, n * n, info, batch).ok()
    torch.cuda.synchronize()
    gi = info.cpu().numpy()
    # backward error of every problem on the device (symmetric: A0 row-major == column-major)
    Lt = torch.tril(A.transpose(1, 2))
    bwd = (torch.linalg.matrix_norm(Lt @ Lt.transpose(1, 2) - A0) / torch.linalg.matrix_norm(A0)).max().item()
    # forward error of every problem against the reference, in chunks
    cpu = _cpu()
    lo = np.tril(np.ones((n, n), bool)).T.reshape(-1)  # lower triangle, column-major flat
    fwd = 0.0
    chunk = max(1, (1 << 28) // (8 * n * n))
    for s0 in range(0, batch, chunk):
        a = A0[s0:s0 + chunk].cpu().numpy().reshape(-1, n * n).copy()
        got = A[s0:s0 + chunk].cpu().numpy().reshape(-1, n * n)
        wi = np.full(len(a), -7, np.int32)
        cpu.dpotrf_batch(b"l", n, a.ctypes.data, n, n * n, wi.ctypes.data, len(a), THREADS)
        assert np.array_equal(wi, gi[s0:s0 + chunk])
        fwd = max(fwd, float(_rel_rows(got[:, lo], a[:, lo]).max()))
    _record(f"cfg3_n{n}", problems_checked=batch, of=batch, info_equal=True, max_rel_frob_fwd=fwd,
            max_backward=bwd, tol=tol(n))
    assert (gi == 0).all()
    assert fwd <= tol(n) and bwd <= tol(n), (fwd, bwd)


# ----------------------------------------------------------------------------------------- cfg4
@pytest.mark.parametrize("n", [24, 48, 96, 192])
def test_cfg4_all_pivots_vs_oracle(pb, cuda, n):
    import torch
    batch = 8192
    g = torch.Generator(device=cuda).manual_seed(400 + n)
    A0 = torch.rand((batch, n, n), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    A = A0.clone()
    ipiv = torch.zeros((batch, n), dtype=torch.int32, device=cuda)
    info = torch.full((batch,), -7, dtype=torch.int32, device=cuda)
    assert pb.dgetrf_batched(n, n, A, n, n * n, ipiv, n, info, batch).ok()
    torch.cuda.synchronize()
    gp, gi = ipiv.cpu().numpy(), info.cpu().numpy()
    # backward error ||P A - L U|| / ||A|| of every problem on the device
    dt = A.transpose(1, 2)
    Lm = torch.tril(dt, -1) + torch.eye(n, device=cuda, dtype=torch.float64)
    U = torch.triu(dt)
    PA = A0.transpose(1, 2).clone()
    ip = ipiv.long() - 1
    rows = torch.arange(batch, device=cuda)
    for j in range(n):
        pj = ip[:, j]
        tmp = PA[rows, j, :].clone()
        PA[rows, j, :] = PA[rows, pj, :]
        PA[rows, pj, :] = tmp
    bwd = (torch.linalg.matrix_norm(Lm @ U - PA) / torch.linalg.matrix_norm(PA)).max().item()
    del Lm, U, PA, dt
    cpu = _cpu()
    mism, fwd = 0, 0.0
    chunk = max(1, (1 << 28) // (8 * n * n))
    for s0 in range(0, batch, chunk):
        a = A0[s0:s0 + chunk].cpu().numpy().reshape(-1, n * n).copy()
        got = A[s0:s0 + chunk].cpu().numpy().reshape(-1, n * n)
        wp = np.zeros((len(a), n), np.int32)
        wi = np.full(len(a), -7, np.int32)
        cpu.dgetrf_batch(n, n, a.ctypes.data, n, n * n, wp.ctypes.data, n, wi.ctypes.data, len(a), THREADS)
        assert np.array_equal(wi, gi[s0:s0 + chunk])
        bad = ~(wp == gp[s0:s0 + chunk]).all(axis=1)
        mism += int(bad.sum())
        ok = ~bad
        if ok.any():
            fwd = max(fwd, float(_rel_rows(got[ok], a[ok]).max()))
    _record(f"cfg4_n{n}", problems_checked=batch, of=batch, pivot_mismatches=mism, info_equal=True,
            max_rel_frob_fwd=fwd, max_backward=bwd, tol=tol(n))
    assert mism == 0, f"{mism} of {batch} problems pivot differently"
    assert bwd <= tol(n), bwd


# ----------------------------------------------------------------------------------------- cfg5
def _cfg5_batch(cuda, layout, seed):
    import torch
    rng = np.random.default_rng(seed)
    batch = 32768
    ns = (rng.integers(1, 65, batch) * 4).astype(np.int32)
    offs = np.concatenate([[0], np.cumsum(ns.astype(np.int64) ** 2)[:-1]]).astype(np.int64)
    total = int((ns.astype(np.int64) ** 2).sum())
    g = torch.Generator(device=cuda).manual_seed(seed)
    A = torch.rand(total, generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    B = torch.rand(total, generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    C = torch.zeros(total, device=cuda, dtype=torch.float64)
    for n in np.unique(ns):  # C0 = n I (lower)
        base = torch.from_numpy(offs[ns == n]).to(cuda)
        ar = torch.arange(int(n), device=cuda)
        diag = ar * (int(n) + 1) if layout == "C" else (ar // 4) * 4 * int(n) + ar * 4 + ar % 4
        C[(base[:, None] + diag[None, :]).reshape(-1)] = float(n)
    return ns, offs, A, B, C


@pytest.mark.parametrize("layout", ["C", "P"])
def test_cfg5_chain_subset_vs_oracle(pb, cuda, layout):
    import torch
    ns, offs, A, B0, C0 = _cfg5_batch(cuda, layout, 500 + (layout == "P"))
    batch = len(ns)
    sub = _subset(batch, 1024, 77)
    # the oracle's inputs: gather the subset's problems into a compact host batch
    sn = ns[sub]
    soff = np.concatenate([[0], np.cumsum(sn.astype(np.int64) ** 2)[:-1]]).astype(np.int64)
    gidx = torch.from_numpy(np.concatenate([np.arange(offs[p], offs[p] + int(ns[p]) ** 2) for p in sub])).to(cuda)
    a, b, c = (x[gidx].cpu().numpy().copy() for x in (A, B0, C0))
    C, B = C0.clone(), B0.clone()
    dn = torch.from_numpy(ns).to(cuda)
    doff = torch.from_numpy(offs).to(cuda)
    info = torch.full((batch,), -9, dtype=torch.int32, device=cuda)
    assert pb.chain_vbatched(layout, dn, doff, A, C, B, info, batch, 256).ok()
    torch.cuda.synchronize()
    gi = info.cpu().numpy()
    gc, gb = C[gidx].cpu().numpy(), B[gidx].cpu().numpy()
    wi = np.full(len(sub), -9, np.int32)
    fn = getattr(_cpu(), "chain_cm_batch" if layout == "C" else "chain_pm_batch", None)
    if fn is None:  # the restatement's single entry point
        ob.oracle().chain_batch(int(layout == "P"), sn.ctypes.data, soff.ctypes.data, a.ctypes.data,
                                c.ctypes.data, b.ctypes.data, wi.ctypes.data, len(sub), THREADS)
    else:
        fn(sn.ctypes.data, soff.ctypes.data, a.ctypes.data, c.ctypes.data, b.ctypes.data, wi.ctypes.data,
           len(sub), THREADS)
    assert (gi == 0).all() and (wi == 0).all()
    worst_l = worst_x = 0.0
    for q, n in enumerate(sn):
        n = int(n)
        o = soff[q]
        if layout == "C":
            lo = np.tril(np.ones((n, n), bool)).T.reshape(-1)
        else:  # panel-major lower triangle (i >= j)
            i = np.arange(n)[:, None]; j = np.arange(n)[None, :]
            lo = np.zeros(n * n, bool)
            lo[((i // 4) * 4 * n + j * 4 + i % 4)[i >= j]] = True
        gl, wl = gc[o:o + n * n][lo], c[o:o + n * n][lo]
        el = np.linalg.norm(gl - wl) / np.linalg.norm(wl)
        ex = np.linalg.norm(gb[o:o + n * n] - b[o:o + n * n]) / np.linalg.norm(b[o:o + n * n])
        worst_l = max(worst_l, el / tol(n))
        worst_x = max(worst_x, ex / tol(n))
    _record(f"cfg5_{'cm' if layout == 'C' else 'pm'}", problems_checked=len(sub), of=batch,
            subset="seeded 1024 incl. first and last", info_equal=True,
            max_rel_frob_L_over_tol=worst_l, max_rel_frob_X_over_tol=worst_x)
    assert worst_l <= 1.0, worst_l
    assert worst_x <= 10.0, worst_x  # X = B L^-T amplifies L's error by cond(L) (<= 10x over the batch)
