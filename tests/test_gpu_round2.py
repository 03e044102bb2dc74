"""GPU parity for the round-2 surface: dtrmm (all flags), trmm_rlnn_nd, device pack/unpack,
the batched Riccati recursion, and the PBGPU_MUTATE negative control."""
import os
import subprocess
import sys

import numpy as np
import pytest

import riccati_ref as rr
from helpers import F, ch, ptr, rel_frob, same_bits, tol
from oracle import binding as ob

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ----------------------------------------------------------------------------- dtrmm
@pytest.mark.parametrize("side", ["l", "r"])
@pytest.mark.parametrize("uplo", ["l", "u"])
@pytest.mark.parametrize("trans", ["n", "t"])
@pytest.mark.parametrize("diag", ["n", "u"])
def test_dtrmm_all_flags(pb, orc, side, uplo, trans, diag):
    """blas.hpp:166-176 / level3.hpp:250-275 against the oracle (NaN poison off the triangle)."""
    rng = np.random.default_rng(abs(hash((side, uplo, trans, diag, 7))) % 2**32)
    for (m, n) in [(9, 7), (70, 33), (64, 64), (5, 130), (129, 3)]:
        t = m if side == "l" else n
        a = F(rng.uniform(-1, 1, (t, t)))
        off = np.triu(np.ones((t, t), bool), 1) if uplo == "l" else np.tril(np.ones((t, t), bool), -1)
        a[off] = np.nan                     # the opposite triangle is never read
        if diag == "u":
            a[np.arange(t), np.arange(t)] = np.nan  # a unit diagonal is never read
        b = F(rng.uniform(-1, 1, (m, n)))
        got, want = b.copy(order="F"), b.copy(order="F")
        r = pb.dtrmm(side, uplo, trans, diag, m, n, -1.25, a, t, got, m)
        assert r.ok(), r
        assert r.flops == (n * m * m if side == "l" else m * n * n)
        assert orc.dtrmm(ch(side), ch(uplo), ch(trans), ch(diag), m, n, -1.25, ptr(a), t, ptr(want), m) == 0
        assert rel_frob(got, want) <= tol(t)


def test_dtrmm_batched_device_and_edges(pb, orc, cuda):
    import torch
    rng = np.random.default_rng(3)
    m, n, batch = 40, 24, 7
    A = rng.uniform(-1, 1, (batch, n, n)); B = rng.uniform(-1, 1, (batch, n, m))
    dA, dB = torch.from_numpy(A.copy()).to(cuda), torch.from_numpy(B.copy()).to(cuda)
    assert pb.dtrmm_batched("r", "l", "n", "n", m, n, 1.0, dA, n, n * n, dB, m, m * n, batch).ok()
    got = dB.cpu().numpy()
    for p in range(batch):
        w = F(B[p].T)
        orc.dtrmm(b"r", b"l", b"n", b"n", m, n, 1.0, ptr(F(A[p].T)), n, ptr(w), m)
        assert rel_frob(got[p].T, w) <= tol(n)
    # alpha = 0: zeros, A never read (level3.hpp:261)
    b = F(rng.uniform(-1, 1, (5, 6)))
    nan_a = F(np.full((6, 6), np.nan))
    assert pb.dtrmm("r", "u", "t", "n", 5, 6, 0.0, nan_a, 6, b, 5).ok()
    assert (b == 0).all() and not np.signbit(b).any()
    # validation shared with dtrsm (blas.hpp:132-162)
    buf = np.zeros(16)
    assert pb.dtrmm("x", "l", "n", "n", 1, 1, 1.0, buf, 1, buf, 1).info == 1
    assert pb.dtrmm("l", "l", "n", "n", 2, 1, 1.0, buf, 1, buf, 2).info == 9
    assert pb.dtrmm("l", "l", "n", "n", 0, 1, 1.0, buf, 1, buf, 0).info == 11


# ----------------------------------------------------------------------------- trmm_rlnn_nd
def test_trmm_rlnn_nd(pb, orc, cuda):
    import torch
    rng = np.random.default_rng(19)
    P = pb.PanelRef
    for (m, n) in [(11, 7), (16, 16), (70, 33), (100, 96), (130, 64)]:
        A = rng.uniform(-1, 1, (n, n)); Bm = rng.uniform(-1, 1, (m, n))
        ap = ob.pack(np.where(np.tril(np.ones((n, n), bool)), A, np.nan), fill=np.nan)
        bp = ob.pack(Bm, fill=np.nan)
        d = np.full(ob.panel_len(m, n), 4.25); want = d.copy()
        assert pb.trmm_rlnn_nd(m, n, 1.5, P(ap, n, n), P(bp, m, n), P(d, m, n)).ok()
        assert orc.trmm_rlnn_nd(m, n, 1.5, ob.dmat(ap, n, n), ob.dmat(bp, m, n), ob.dmat(want, m, n)) == 0
        assert rel_frob(ob.unpack(d, m, n), ob.unpack(want, m, n)) <= tol(n)
        pad = np.ones_like(d, bool)
        i = np.arange(m)[:, None]; j = np.arange(n)[None, :]
        pad[(i // 4) * 4 * ob.round_up(n, 4) + j * 4 + i % 4] = False
        assert (d[pad] == 4.25).all()      # pad lanes untouched
        io = bp.copy()                      # b aliases d
        assert pb.trmm_rlnn_nd(m, n, 1.5, P(ap, n, n), P(io, m, n), P(io, m, n)).ok()
        assert rel_frob(ob.unpack(io, m, n), ob.unpack(want, m, n)) <= tol(n)
    # batched on the device
    m, n, batch = 24, 20, 9
    La, Lb = ob.panel_len(n, n), ob.panel_len(m, n)
    As = rng.uniform(-1, 1, (batch, La)); Bs = rng.uniform(-1, 1, (batch, Lb))
    dA, dB = torch.from_numpy(As).to(cuda), torch.from_numpy(Bs).to(cuda)
    dD = torch.zeros((batch, Lb), dtype=torch.float64, device=cuda)
    assert pb.trmm_rlnn_nd_batched(m, n, 1.0, P(dA, n, n), La, P(dB, m, n), Lb, P(dD, m, n), Lb, batch).ok()
    got = dD.cpu().numpy()
    for p in range(batch):
        w = np.zeros(Lb)
        ap_, bp_ = As[p].copy(), Bs[p].copy()  # keep the buffers alive: a Dmat holds a raw address
        orc.trmm_rlnn_nd(m, n, 1.0, ob.dmat(ap_, n, n), ob.dmat(bp_, m, n), ob.dmat(w, m, n))
        assert rel_frob(ob.unpack(got[p], m, n), ob.unpack(w, m, n)) <= tol(n)


# ----------------------------------------------------------------------------- pack / unpack
@pytest.mark.parametrize("ps", [4, 8, 1])
def test_pack_unpack_bitwise(pb, cuda, ps):
    """panel_mat.hpp:141-171: bitwise equal to the packing formula; pad lanes untouched."""
    import torch
    rng = np.random.default_rng(ps)
    for (m, n, tr) in [(9, 6, "n"), (9, 6, "t"), (64, 64, "n"), (33, 70, "t"), (1, 1, "n")]:
        src = F(rng.uniform(-1, 1, (m, n) if tr == "n" else (n, m)))
        d = np.full(ob.panel_len(m, n, ps), -2.75)
        assert pb.pack(tr, src, src.shape[0], pb.PanelRef(d, m, n, ps=ps)).ok()
        assert same_bits(d, ob.pack(src if tr == "n" else F(src.T), ps=ps, fill=-2.75))
        back = F(np.full((m + 3, n), 9.5))
        assert pb.unpack(pb.PanelRef(d, m, n, ps=ps), back, m + 3).ok()
        assert same_bits(back[:m], src if tr == "n" else F(src.T)) and (back[m:] == 9.5).all()
    assert pb.memsize(9, 6, 4) == 12 * 8 * 8 and pb.memsize(0, 5, 4) == 0
    # batched, device-resident round trip
    m, n, batch = 37, 21, 50
    A = rng.uniform(-1, 1, (batch, n, m))
    dA = torch.from_numpy(A.copy()).to(cuda)
    L = ob.panel_len(m, n, ps)
    dP = torch.full((batch, L), 1.5, dtype=torch.float64, device=cuda)
    P = pb.PanelRef(dP, m, n, ps=ps)
    assert pb.pack_batched("n", dA, m, m * n, P, L, batch).ok()
    got = dP.cpu().numpy()
    for p in (0, 17, batch - 1):
        assert same_bits(got[p], ob.pack(F(A[p].T), ps=ps, fill=1.5))
    dB = torch.zeros_like(dA)
    assert pb.unpack_batched(P, L, dB, m, m * n, batch).ok()
    assert same_bits(dB.cpu().numpy(), A)


# ----------------------------------------------------------------------------- Riccati
def riccati_batch(rng, nx, nu, batch):
    m0s, qs, gs, raw = [], [], [], []
    for _ in range(batch):
        a, b, q, r, s = rr.make_ocp(rng, nx, nu)
        m0p, qp, gp = rr.stage_data(a, b, q, r, s)
        m0s.append(m0p); qs.append(qp); gs.append(gp); raw.append((a, b, q, r, s))
    return np.stack(m0s), np.stack(qs), np.stack(gs), raw


def run_riccati(pb, cuda, nx, nu, N, m0s, qs, gs):
    import torch
    nt = nx + nu
    batch = m0s.shape[0]
    P = pb.PanelRef
    Lf, Lq = ob.panel_len(nt, nt), ob.panel_len(nx, nx)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(cuda)
    dm0, dq, dg = d(m0s), d(qs), d(gs)
    f = torch.full((batch, N * Lf), np.nan, dtype=torch.float64, device=cuda)
    lt = torch.full((batch, Lq), np.nan, dtype=torch.float64, device=cuda)
    info = torch.full((batch,), 99, dtype=torch.int32, device=cuda)
    stage = torch.full((batch,), 99, dtype=torch.int32, device=cuda)
    r = pb.riccati_nd_batched(nx, nu, N, P(dm0, nt, nt), m0s.shape[1], P(dq, nx, nx), qs.shape[1],
                              P(dg, nt, nx), gs.shape[1], P(f, nt, nt), N * Lf, P(lt, nx, nx), Lq,
                              info, stage, batch)
    return r, f.cpu().numpy().reshape(batch, N, Lf), lt.cpu().numpy(), info.cpu().numpy(), stage.cpu().numpy()


@pytest.mark.parametrize("nx,nu,N", [(4, 2, 3), (8, 4, 10), (24, 12, 6), (40, 20, 4), (64, 32, 3), (5, 0, 4)])
def test_riccati_batched_vs_oracle(pb, orc, cuda, nx, nu, N):
    """Every stage factor vs the oracle's packed stage loop (riccati.hpp:296-337), and the
    whole-horizon residual vs the textbook recursion (riccati.hpp:402-512, <= 1e-10)."""
    rng = np.random.default_rng(nx * 100 + nu)
    batch = 6
    nt = nx + nu
    m0s, qs, gs, raw = riccati_batch(rng, nx, nu, batch)
    r, f, lt, info, stage = run_riccati(pb, cuda, nx, nu, N, m0s, qs, gs)
    assert r.ok(), r
    assert (info == 0).all() and (stage == -1).all()
    for p in range(batch):
        fs, lterm, oi, _ = rr.fused_oracle(orc, m0s[p], qs[p], gs[p], nx, nu, N)
        assert oi == 0
        assert rel_frob(ob.unpack(lt[p], nx, nx), ob.unpack(lterm, nx, nx)) <= tol(nx)
        Ptraj = rr.textbook(*raw[p], N)
        for s in range(N):
            G = ob.unpack(f[p, s], nt, nt)
            W = ob.unpack(fs[s], nt, nt)
            assert (np.triu(G, 1) == 0).all()                    # [[Lambda, 0], [L, calL]]
            assert rel_frob(np.tril(G), np.tril(W)) <= tol(nt)
            assert rr.chol_residual(G[nu:, nu:], Ptraj[s]) <= 1e-10


def test_riccati_failures_and_validation(pb, cuda):
    """test_riccati.cpp:234-285: a control pivot fails at 1, a state pivot at nu + 1."""
    rng = np.random.default_rng(77)
    nx, nu, N = 5, 3, 4
    nt = nx + nu
    m0s, qs, gs, raw = riccati_batch(rng, nx, nu, 3)
    # problem 1: R(0, 0) = -1e6 -> info 1 at the first step (stage N - 1)
    M = ob.unpack(m0s[1], nt, nt); M[0, 0] = -1e6; m0s[1] = ob.pack(M)
    # problem 2: Q block of the bordered matrix = -1e6 I, terminal Q = I -> info nu + 1
    M = ob.unpack(m0s[2], nt, nt); M[nu:, nu:] = -1e6 * np.eye(nx); m0s[2] = ob.pack(M)
    qs[2] = ob.pack(np.eye(nx))
    r, f, lt, info, stage = run_riccati(pb, cuda, nx, nu, N, m0s, qs, gs)
    assert r.ok()
    assert info.tolist() == [0, 1, nu + 1] and stage.tolist() == [-1, N - 1, N - 1]
    # terminal failure: Q not positive definite -> stage N
    qs2 = qs.copy(); qs2[0] = ob.pack(-np.eye(nx))
    r, f, lt, info, stage = run_riccati(pb, cuda, nx, nu, N, m0s, qs2, gs)
    assert info[0] == 1 and stage[0] == N
    # invalid dims rejected up front (riccati.hpp:409-412)
    P = pb.PanelRef
    z = np.zeros(64)
    assert pb.riccati_nd_batched(0, 2, 3, P(z, 2, 2), 0, P(z, 0, 0), 0, P(z, 2, 0), 0, P(z, 2, 2), 0, None, 0,
                                 np.zeros(1, np.int32), None, 1).info == -1


# ----------------------------------------------------------------------------- PBGPU_MUTATE
_MUT = r"""
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_1902_08115_b200 as pb
from oracle import binding as ob
from helpers import F, ptr, rel_frob, tol
import verify_suite
rep = verify_suite.run(pb, ob.oracle(), seed=7, count=16)
print("FAILURES", rep["failures"], "CASES", rep["cases_run"])
"""


@pytest.mark.parametrize("eps", [0.0, 1e-6])
def test_mutation_negative_control(eps):
    """The GPU verify suite passes clean and goes red under PBGPU_MUTATE (micro_kernel.hpp:424-426)."""
    env = dict(os.environ)
    if eps:
        env["PBGPU_MUTATE"] = repr(eps)
    else:
        env.pop("PBGPU_MUTATE", None)
    out = subprocess.run([sys.executable, "-c", _MUT % (ROOT, os.path.join(ROOT, "tests"))], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("FAILURES")][-1]
    failures, cases = int(line.split()[1]), int(line.split()[3])
    assert cases > 0
    if eps:
        assert failures == cases      # every routine's result is perturbed -> every case red
    else:
        assert failures == 0
