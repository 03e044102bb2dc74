"""Test helpers for the batched Riccati recursion (riccati.hpp), CPU side.

* ``stage_data`` packs one OCP's stage-constant blocks as RiccatiFusedWork's
  constructor does (riccati.hpp:271-294): the bordered matrix fully symmetric,
  Q, and G = [B^T; A^T].
* ``fused_oracle`` runs the same stage loop on the C oracle restatement
  (orc_syrk_potrf_nd with k = 0, then per stage orc_trmm_rlnn_nd +
  orc_syrk_potrf_nd + the trailing-block copy, riccati.hpp:296-337).
* ``textbook`` / ``chol_residual`` restate riccati_oracle_step and
  chol_residual (riccati.hpp:124-180) in numpy for the whole-horizon residual.
"""
import numpy as np

from oracle import binding as ob


def make_ocp(rng, nx, nu):
    """make_ocp_data's recipe (riccati.hpp:65-103) on a numpy generator."""
    gain = 1.0 / np.sqrt(nx + nu)
    a = rng.uniform(-gain, gain, (nx, nx))
    b = rng.uniform(-gain, gain, (nx, nu))
    s = rng.uniform(-0.1, 0.1, (nu, nx))
    mq = rng.uniform(-1, 1, (nx, nx))
    q = mq.T @ mq + nx * np.eye(nx)
    kr = rng.uniform(-1, 1, (nu, nu))
    r = kr.T @ kr + nu * np.eye(nu)
    return a, b, q, r, s


def stage_data(a, b, q, r, s):
    nx, nu = a.shape[0], b.shape[1]
    nt = nx + nu
    m0 = np.zeros((nt, nt))
    m0[:nu, :nu] = r
    m0[:nu, nu:] = s
    m0[nu:, :nu] = s.T
    m0[nu:, nu:] = q
    g = np.zeros((nt, nx))
    g[:nu, :] = b.T
    g[nu:, :] = a.T
    return ob.pack(m0), ob.pack(q), ob.pack(g)


def fused_oracle(orc, m0p, qp, gp, nx, nu, N):
    """Returns (stage factors F_s packed nt x nt for s = 0..N-1, terminal calL packed, info, stage)."""
    nt = nx + nu
    call = np.zeros(ob.panel_len(nx, nx))
    none = np.zeros(4)
    info = orc.syrk_potrf_nd(nx, 0, ob.dmat(none, nx, 0), ob.dmat(none, nx, 0), ob.dmat(qp, nx, nx),
                             ob.dmat(call, nx, nx))
    lterm = call.copy()
    fs = [None] * N
    if info:
        return fs, lterm, info, N
    for st in range(N - 1, -1, -1):
        c = np.zeros(ob.panel_len(nt, nx))
        assert orc.trmm_rlnn_nd(nt, nx, 1.0, ob.dmat(call, nx, nx), ob.dmat(gp, nt, nx), ob.dmat(c, nt, nx)) == 0
        f = np.zeros(ob.panel_len(nt, nt))
        info = orc.syrk_potrf_nd(nt, nx, ob.dmat(c, nt, nx), ob.dmat(c, nt, nx), ob.dmat(m0p, nt, nt),
                                 ob.dmat(f, nt, nt))
        fs[st] = f
        if info:
            return fs, lterm, info, st
        F = ob.unpack(f, nt, nt)
        call = ob.pack(np.tril(F[nu:, nu:]))
    return fs, lterm, 0, -1


def textbook(a, b, q, r, s, N):
    """riccati_oracle_step (riccati.hpp:145-180) from P_N = Q: returns [P_0 .. P_N]."""
    P = [None] * (N + 1)
    P[N] = q.copy()
    for n in range(N - 1, -1, -1):
        pn = P[n + 1]
        w = r + b.T @ pn @ b
        k = s + b.T @ pn @ a
        p = q + a.T @ pn @ a - k.T @ np.linalg.solve(w, k)
        P[n] = 0.5 * (p + p.T)
    return P


def chol_residual(l, p):
    """riccati.hpp:124-140: ||tril(l) tril(l)^T - p||_F / ||p||_F."""
    L = np.tril(l)
    den = np.linalg.norm(p)
    num = np.linalg.norm(L @ L.T - p)
    return num / den if den > 0 else num
