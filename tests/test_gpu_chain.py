"""GPU parity: fused syrk_potrf_nd and the variable-size chain (config 5) vs the oracle."""
import os

import numpy as np
import pytest

from helpers import F, ch, ptr, rel_frob, same_bits, tol
from oracle.binding import dmat, pack, panel_len, unpack

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def spd(rng, n):
    g = rng.uniform(-1, 1, (n, n))
    return g @ g.T + n * np.eye(n)


@pytest.mark.parametrize("n,k", [(6, 7), (13, 7), (21, 7), (13, 0), (64, 64), (100, 30), (160, 16), (200, 24)])
def test_syrk_potrf_nd_vs_oracle(pb, orc, n, k):
    rng = np.random.default_rng(n * 31 + k)
    A = rng.uniform(-1, 1, (n, k)) if k else np.zeros((n, 0))
    S = spd(rng, n)
    ap = pack(A, fill=np.nan) if k else np.zeros(4)
    cp = pack(S, fill=np.nan)
    sentinel = 64.125
    d = np.full(panel_len(n, n), sentinel); want = d.copy()
    r = pb.syrk_potrf_nd(n, k, pb.PanelRef(ap, n, k), pb.PanelRef(ap, n, k), pb.PanelRef(cp, n, n), pb.PanelRef(d, n, n))
    assert r.ok(), r
    assert orc.syrk_potrf_nd(n, k, dmat(ap, n, k), dmat(ap, n, k), dmat(cp, n, n), dmat(want, n, n)) == 0
    L, W = unpack(d, n, n), unpack(want, n, n)
    lo = np.tril(np.ones((n, n), bool))
    assert rel_frob(L[lo], W[lo]) <= tol(n)
    # strictly-upper: zero inside 8-row diagonal bands, untouched beyond (test_level3.cpp:655-668)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    band = (i < j) & (j < np.minimum(n, (i // 8) * 8 + 8))
    assert (L[band] == 0.0).all()
    assert (L[(i < j) & ~band] == sentinel).all()
    rec = np.tril(L) @ np.tril(L).T
    M = S + A @ A.T
    assert rel_frob(rec, M) <= tol(n)


def test_syrk_potrf_nd_golden_alias_and_failure(pb):
    for n in (6, 13, 21, 64):
        case = f"chain_nd_{n}"
        nn, k = (int(x) for x in GOLD[f"{case}/nk"])
        a, c = GOLD[f"{case}/a"].copy(), GOLD[f"{case}/c"].copy()
        d = np.full(panel_len(n, n), 64.125)
        assert pb.syrk_potrf_nd(n, k, pb.PanelRef(a, n, k), pb.PanelRef(a, n, k), pb.PanelRef(c, n, n), pb.PanelRef(d, n, n)).ok()
        want = GOLD[f"{case}/l"]
        assert rel_frob(d, want) <= tol(n)
        # c aliasing d gives the same factor
        io = c.copy()
        assert pb.syrk_potrf_nd(n, k, pb.PanelRef(a, n, k), pb.PanelRef(a, n, k), pb.PanelRef(io, n, n), pb.PanelRef(io, n, n)).ok()
        lo = np.tril(np.ones((n, n), bool))
        assert same_bits(unpack(io, n, n)[lo], unpack(d, n, n)[lo])
        # trsm_rltn_nd on the factor reproduces the reference's X
        b = GOLD[f"{case}/b"].copy()
        x = np.full(panel_len(11, n), 2.5)
        assert pb.trsm_rltn_nd(11, n, 1.5, pb.PanelRef(d, n, n), pb.PanelRef(b, 11, n), pb.PanelRef(x, 11, n)).ok()
        assert rel_frob(x, GOLD[f"{case}/x"]) <= tol(n)
    # test_level3.cpp:688-705: M = diag(4, 1, -1) fails at 3; -4 at 1
    ap = np.zeros(panel_len(3, 2)); cp = np.zeros(panel_len(3, 3)); dp = np.zeros(panel_len(3, 3))
    C = np.diag([4.0, 1.0, -1.0]); cp[:] = pack(C)
    assert pb.syrk_potrf_nd(3, 2, pb.PanelRef(ap, 3, 2), pb.PanelRef(ap, 3, 2), pb.PanelRef(cp, 3, 3), pb.PanelRef(dp, 3, 3)).info == 3
    C[0, 0] = -4.0; cp[:] = pack(C)
    assert pb.syrk_potrf_nd(3, 2, pb.PanelRef(ap, 3, 2), pb.PanelRef(ap, 3, 2), pb.PanelRef(cp, 3, 3), pb.PanelRef(dp, 3, 3)).info == 1


@pytest.mark.parametrize("layout", ["C", "P"])
def test_chain_vbatched(pb, orc, cuda, layout):
    """Config 5 shape: n = 4*U{1..64}; per problem C0 = n I, A, B uniform; checked per problem."""
    import torch
    rng = np.random.default_rng(5 if layout == "C" else 6)
    batch = 48
    ns = rng.integers(1, 65, batch) * 4
    ns[:4] = [4, 160, 164, 256]
    offs = np.concatenate([[0], np.cumsum(ns.astype(np.int64) ** 2)[:-1]])
    total = int((ns.astype(np.int64) ** 2).sum())
    A = rng.uniform(-1, 1, total); B = rng.uniform(-1, 1, total)
    C = np.zeros(total)
    for p, n in enumerate(ns):  # C0 = n I (diagonal only; same in both layouts)
        blk = np.zeros((n, n)); blk[np.arange(n), np.arange(n)] = n
        C[offs[p]:offs[p] + n * n] = blk.reshape(-1, order="F") if layout == "C" else pack(blk)
    dA, dB, dC = (torch.from_numpy(x.copy()).to(cuda) for x in (A, B, C))
    dn = torch.from_numpy(ns.astype(np.int32)).to(cuda)
    doff = torch.from_numpy(offs.astype(np.int64)).to(cuda)
    info = torch.full((batch,), -9, dtype=torch.int32, device=cuda)
    r = pb.chain_vbatched(layout, dn, doff, dA, dC, dB, info, batch, int(ns.max()))
    assert r.ok(), r
    gC, gB, gi = dC.cpu().numpy(), dB.cpu().numpy(), info.cpu().numpy()
    assert (gi == 0).all()
    for p, n in enumerate(ns):
        o = offs[p]
        a = A[o:o + n * n].copy(); c = C[o:o + n * n].copy(); b = B[o:o + n * n].copy()
        if layout == "C":
            a, c, b = (np.asfortranarray(x.reshape(n, n, order="F")) for x in (a, c, b))
            orc.dsyrk(b"l", b"n", n, n, 1.0, ptr(a), n, 1.0, ptr(c), n)
            assert orc.dpotrf(b"l", n, ptr(c), n) == 0
            assert orc.dtrsm(b"r", b"l", b"t", b"n", n, n, 1.0, ptr(c), n, ptr(b), n) == 0
            gc = gC[o:o + n * n].reshape(n, n, order="F"); gb = gB[o:o + n * n].reshape(n, n, order="F")
            lo = np.tril(np.ones((n, n), bool))
            assert rel_frob(gc[lo], c[lo]) <= tol(n)
            assert rel_frob(gb, b) <= tol(n) * 10
        else:
            assert orc.syrk_potrf_nd(n, n, dmat(a, n, n), dmat(a, n, n), dmat(c, n, n), dmat(c, n, n)) == 0
            assert orc.trsm_rltn_nd(n, n, 1.0, dmat(c, n, n), dmat(b, n, n), dmat(b, n, n)) == 0
            assert rel_frob(gC[o:o + n * n], c) <= tol(n)
            assert rel_frob(gB[o:o + n * n], b) <= tol(n) * 10


def test_chain_cfg5_full_batch_properties(pb, cuda):
    """Config 5 at full size (32768 problems, n = 4 U{1..64}, column-major): every problem
    checked on the device by size-independent properties — the factor reproduces
    C0 + A A^T (||L L^T - S|| / ||S||) and the solve satisfies ||X L^T - B|| / ||B|| —
    within the north star's 1e-13 n."""
    import torch
    rng = np.random.default_rng(55)
    batch = 32768
    ns = rng.integers(1, 65, batch) * 4
    offs = np.concatenate([[0], np.cumsum(ns.astype(np.int64) ** 2)[:-1]])
    total = int((ns.astype(np.int64) ** 2).sum())
    g = torch.Generator(device=cuda).manual_seed(55)
    A = torch.rand(total, generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    B0 = torch.rand(total, generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    C = torch.zeros(total, device=cuda, dtype=torch.float64)
    for n in np.unique(ns):
        idx = np.nonzero(ns == n)[0]
        base = torch.from_numpy(offs[idx]).to(cuda)
        ar = torch.arange(int(n), device=cuda)
        C[(base[:, None] + (ar * (int(n) + 1))[None, :]).reshape(-1)] = float(n)
    B = B0.clone()
    dn = torch.from_numpy(ns.astype(np.int32)).to(cuda)
    doff = torch.from_numpy(offs).to(cuda)
    info = torch.full((batch,), -9, dtype=torch.int32, device=cuda)
    assert pb.chain_vbatched("C", dn, doff, A, C, B, info, batch, 256).ok()
    torch.cuda.synchronize()
    assert int(info.abs().sum()) == 0
    worst = 0.0
    for n in np.unique(ns):
        n = int(n)
        idx = torch.from_numpy(offs[ns == n]).to(cuda)
        gidx = (idx[:, None] + torch.arange(n * n, device=cuda)[None, :])
        # column-major n x n blocks: element (i, j) at i + j n -> view as (batch, j, i), transpose
        a = A[gidx].view(-1, n, n).transpose(1, 2)
        l = torch.tril(C[gidx].view(-1, n, n).transpose(1, 2))
        x = B[gidx].view(-1, n, n).transpose(1, 2)
        b = B0[gidx].view(-1, n, n).transpose(1, 2)
        s = a @ a.transpose(1, 2) + n * torch.eye(n, device=cuda, dtype=torch.float64)
        e1 = (torch.linalg.matrix_norm(l @ l.transpose(1, 2) - s) / torch.linalg.matrix_norm(s)).max().item()
        e2 = (torch.linalg.matrix_norm(x @ l.transpose(1, 2) - b) / torch.linalg.matrix_norm(b)).max().item()
        worst = max(worst, e1 / tol(n), e2 / tol(n))
    assert worst <= 1.0, worst


@pytest.mark.parametrize("layout", ["C", "P"])
def test_chain_host_plan_and_host_pointers(pb, cuda, layout):
    """pb_chain_vbatched with host n / offset (device matrices: no synchronisation) and with
    everything on the host (staged): bit-identical to the all-device call."""
    import torch
    rng = np.random.default_rng(21)
    batch = 40
    ns = (rng.integers(1, 65, batch) * 4).astype(np.int32)
    ns[:3] = [4, 168, 256]
    offs = np.concatenate([[0], np.cumsum(ns.astype(np.int64) ** 2)[:-1]]).astype(np.int64)
    total = int((ns.astype(np.int64) ** 2).sum())
    A = rng.uniform(-1, 1, total); B = rng.uniform(-1, 1, total); C = np.zeros(total)
    for p, n in enumerate(ns):
        blk = np.zeros((n, n)); blk[np.arange(n), np.arange(n)] = n
        C[offs[p]:offs[p] + n * n] = blk.reshape(-1, order="F") if layout == "C" else pack(blk)
    runs = []
    for mode in ("device", "host_plan", "host"):
        if mode == "host":
            a, c, b = A.copy(), C.copy(), B.copy()
            info = np.full(batch, -9, np.int32)
            assert pb.chain_vbatched(layout, ns, offs, a, c, b, info, batch, 256).ok()
            runs.append((c, b, info))
            continue
        a, c, b = (torch.from_numpy(x.copy()).to(cuda) for x in (A, C, B))
        info = torch.full((batch,), -9, dtype=torch.int32, device=cuda)
        n_arg = torch.from_numpy(ns).to(cuda) if mode == "device" else ns
        o_arg = torch.from_numpy(offs).to(cuda) if mode == "device" else offs
        assert pb.chain_vbatched(layout, n_arg, o_arg, a, c, b, info, batch, 256).ok()
        torch.cuda.synchronize()
        runs.append((c.cpu().numpy(), b.cpu().numpy(), info.cpu().numpy()))
    for other in runs[1:]:
        assert (other[2] == 0).all()
        assert same_bits(other[0], runs[0][0]) and same_bits(other[1], runs[0][1])


def test_chain_cm_odd_orders_take_the_workspace_path(pb, orc, cuda):
    """Column-major chain with odd orders: the offsets are odd, so the large orders cannot ride
    the engine's offset tensor maps in place (16-byte alignment) and go through the gathered
    strided workspace instead; same results, strict upper triangle of C untouched."""
    import torch
    rng = np.random.default_rng(77)
    ns = np.array([5, 33, 161, 163, 201, 255, 170, 64, 7, 199], dtype=np.int64)
    batch = len(ns)
    offs = np.concatenate([[0], np.cumsum(ns ** 2)[:-1]])
    total = int((ns ** 2).sum())
    A = rng.uniform(-1, 1, total); B = rng.uniform(-1, 1, total)
    C = rng.uniform(-1, 1, total)  # the strict upper part is noise that must survive
    for p, n in enumerate(ns):
        blk = C[offs[p]:offs[p] + n * n].reshape(n, n, order="F")
        blk[np.tril_indices(n)] = 0.0
        blk[np.arange(n), np.arange(n)] = n
    C0 = C.copy()
    dA, dB, dC = (torch.from_numpy(x.copy()).to(cuda) for x in (A, B, C))
    dn = torch.from_numpy(ns.astype(np.int32)).to(cuda)
    doff = torch.from_numpy(offs.astype(np.int64)).to(cuda)
    info = torch.full((batch,), -9, dtype=torch.int32, device=cuda)
    r = pb.chain_vbatched("C", dn, doff, dA, dC, dB, info, batch, int(ns.max()))
    assert r.ok(), r
    gC, gB, gi = dC.cpu().numpy(), dB.cpu().numpy(), info.cpu().numpy()
    assert (gi == 0).all()
    for p, n in enumerate(ns):
        n = int(n); o = offs[p]
        a, c, b = (np.asfortranarray(x[o:o + n * n].reshape(n, n, order="F").copy()) for x in (A, C0, B))
        orc.dsyrk(b"l", b"n", n, n, 1.0, ptr(a), n, 1.0, ptr(c), n)
        assert orc.dpotrf(b"l", n, ptr(c), n) == 0
        assert orc.dtrsm(b"r", b"l", b"t", b"n", n, n, 1.0, ptr(c), n, ptr(b), n) == 0
        gc = gC[o:o + n * n].reshape(n, n, order="F"); gb = gB[o:o + n * n].reshape(n, n, order="F")
        lo = np.tril(np.ones((n, n), bool))
        assert rel_frob(gc[lo], c[lo]) <= tol(n)
        assert rel_frob(gb, b) <= tol(n) * 10
        up = np.triu(np.ones((n, n), bool), 1)
        assert np.array_equal(gc[up], C0[o:o + n * n].reshape(n, n, order="F")[up])
