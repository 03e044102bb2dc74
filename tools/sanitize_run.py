"""One small launch of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck).

usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py [family ...]
Families: gemm_cm gemm_engine gemm_nd potrf getrf trsm trmm chain pack riccati.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1902_08115_b200 as pb  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
P = pb.PanelRef


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def rand(*shape):
    return t(rng.uniform(-1, 1, shape))


def spd(batch, n):
    G = rng.standard_normal((batch, n, n))
    return t(G @ G.transpose(0, 2, 1) + n * np.eye(n))


def gemm_cm():
    A, B, C = rand(4, 64, 64), rand(4, 64, 64), rand(4, 64, 64)
    assert pb.dgemm_batched("n", "n", 64, 64, 64, 1.0, A, 64, 4096, B, 64, 4096, 1.0, C, 64, 4096, 4).ok()


def gemm_engine():
    for (ta, tb, m, n, k) in [("n", "t", 70, 33, 45), ("t", "n", 130, 96, 64), ("t", "t", 9, 200, 17)]:
        A, B, C = rand(3, 256 * 256), rand(3, 256 * 256), rand(3, 256 * 256)
        lda = m if ta == "n" else k
        ldb = k if tb == "n" else n
        assert pb.dgemm_batched(ta, tb, m, n, k, 0.5, A, lda, 65536, B, ldb, 65536, 1.0, C, m, 65536, 3).ok()
    C = rand(3, 96 * 96); A = rand(3, 96 * 80)
    assert pb.dsyrk_batched("l", "n", 96, 80, 1.0, A, 96, 96 * 80, 1.0, C, 96, 96 * 96, 3).ok()


def gemm_nd():
    for s in (4, 8, 20, 24, 48, 96, 116, 160):
        L = s * s
        A, B, C = rand(5, L), rand(5, L), rand(5, L)
        D = torch.empty_like(A)
        assert pb.gemm_nd_batched("n", "t", s, s, s, 1.0, P(A, s, s), L, P(B, s, s), L, 1.0, P(C, s, s), L,
                                  P(D, s, s), L, 5).ok()


def potrf():
    for n in (8, 16, 32, 48, 64, 128, 160, 200):
        A = spd(3, n)
        info = torch.empty(3, dtype=torch.int32, device=dev)
        assert pb.dpotrf_batched("l", n, A, n, n * n, info, 3).ok()


def getrf():
    for n in (8, 24, 32, 40, 48, 64, 79, 96, 104, 130, 160):  # 40..96 and the 104/160 tails: getrf_sq
        A = rand(3, n, n)
        ip = torch.empty((3, n), dtype=torch.int32, device=dev)
        info = torch.empty(3, dtype=torch.int32, device=dev)
        assert pb.dgetrf_batched(n, n, A, n, n * n, ip, n, info, 3).ok()


def trsm():
    for n in (8, 40, 96, 200):
        L = spd(2, n)
        info = torch.empty(2, dtype=torch.int32, device=dev)
        pb.dpotrf_batched("l", n, L, n, n * n, info, 2)
        B = rand(2, n, 37)
        assert pb.dtrsm_batched("r", "l", "t", "n", 37, n, 1.0, L, n, n * n, B, 37, 37 * n, info, 2).ok()
        B = rand(2, n, 37)
        assert pb.dtrsm_batched("l", "u", "n", "n", n, 37, 1.0, L, n, n * n, B, n, 37 * n, info, 2).ok()


def trmm():
    A, B = rand(2, 50 * 50), rand(2, 50 * 70)
    assert pb.dtrmm_batched("r", "l", "n", "n", 70, 50, 1.0, A, 50, 2500, B, 70, 3500, 2).ok()
    assert pb.dtrmm_batched("l", "u", "t", "u", 50, 70, 1.0, A, 50, 2500, B, 50, 3500, 2).ok()


def chain():
    ns = np.array([4, 36, 160, 164, 256], np.int32)
    offs = np.concatenate([[0], np.cumsum(ns.astype(np.int64) ** 2)[:-1]]).astype(np.int64)
    tot = int((ns.astype(np.int64) ** 2).sum())
    for lay in "CP":
        A, B = rand(tot), rand(tot)
        C = torch.zeros(tot, dtype=torch.float64, device=dev)
        for p, n in enumerate(ns):
            ar = torch.arange(int(n), device=dev)
            diag = ar * (int(n) + 1) if lay == "C" else (ar // 4) * 4 * int(n) + ar * 4 + ar % 4
            C[int(offs[p]) + diag] = float(n)
        info = torch.empty(len(ns), dtype=torch.int32, device=dev)
        assert pb.chain_vbatched(lay, t(ns), t(offs), A, C, B, info, len(ns), 256).ok()


def pack():
    A = rand(3, 21, 37)
    D = torch.zeros((3, 40 * 24), dtype=torch.float64, device=dev)
    assert pb.pack_batched("n", A, 37, 37 * 21, P(D, 37, 21), 40 * 24, 3).ok()
    assert pb.unpack_batched(P(D, 37, 21), 40 * 24, A, 37, 37 * 21, 3).ok()


def riccati():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import riccati_ref as rr
    from oracle import binding as ob
    nx, nu, N, batch = 8, 4, 3, 2
    nt = nx + nu
    m0s, qs, gs = [], [], []
    for _ in range(batch):
        m0p, qp, gp = rr.stage_data(*rr.make_ocp(rng, nx, nu))
        m0s.append(m0p); qs.append(qp); gs.append(gp)
    m0s, qs, gs = np.stack(m0s), np.stack(qs), np.stack(gs)
    Lf, Lq = ob.panel_len(nt, nt), ob.panel_len(nx, nx)
    f = torch.zeros((batch, N * Lf), dtype=torch.float64, device=dev)
    lt = torch.zeros((batch, Lq), dtype=torch.float64, device=dev)
    info = torch.empty(batch, dtype=torch.int32, device=dev)
    st = torch.empty(batch, dtype=torch.int32, device=dev)
    assert pb.riccati_nd_batched(nx, nu, N, P(t(m0s), nt, nt), m0s.shape[1], P(t(qs), nx, nx), qs.shape[1],
                                 P(t(gs), nt, nx), gs.shape[1], P(f, nt, nt), N * Lf, P(lt, nx, nx), Lq,
                                 info, st, batch).ok()


FAMILIES = dict(gemm_cm=gemm_cm, gemm_engine=gemm_engine, gemm_nd=gemm_nd, potrf=potrf, getrf=getrf,
                trsm=trsm, trmm=trmm, chain=chain, pack=pack, riccati=riccati)

if __name__ == "__main__":
    names = sys.argv[1:] or list(FAMILIES)
    for nm in names:
        FAMILIES[nm]()
        torch.cuda.synchronize()
        print("ok", nm, flush=True)
