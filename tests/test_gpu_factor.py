"""GPU parity: dpotrf / dtrsm / trsm_rltn_nd through the C ABI vs the oracle and exact fixtures."""
import numpy as np
import pytest

from helpers import F, ch, ptr, rel_frob, same_bits, tol
from oracle.binding import dmat, pack, panel_len, unpack

pytestmark = pytest.mark.gpu


def spd(rng, n):
    """make_spd (matgen.hpp:44-57): G G^T + n I with G uniform[-1, 1]."""
    g = rng.uniform(-1, 1, (n, n))
    return F(g @ g.T + n * np.eye(n))


def dyadic_chol_factor(n):
    """test_factor.cpp:39-51 recipe: power-of-two diagonal, multiples of 1/4 below."""
    l = np.zeros((n, n))
    for j in range(n):
        l[j, j] = float(1 << (j % 3)) * (0.5 if j % 2 else 1.0)
        for i in range(j + 1, n):
            pick = (i * 7 + j * 5) % 4
            v = 0.0 if pick == 0 else 0.25 * pick
            l[i, j] = -v if ((i + j) % 2 and pick != 0) else v
    return F(l)


# ----------------------------------------------------------------------------- potrf
@pytest.mark.parametrize("uplo", ["l", "u"])
@pytest.mark.parametrize("n", [1, 4, 7, 13, 16, 29, 32, 64, 100, 128, 160, 200, 256])
def test_dpotrf_batched_vs_oracle(pb, orc, cuda, uplo, n):
    import torch
    rng = np.random.default_rng(1000 + n)
    batch = 6
    A = np.ascontiguousarray(np.stack([spd(rng, n) for _ in range(batch)]))  # (batch, n, n) logical
    store = A.transpose(0, 2, 1).copy()                         # column-major per problem
    # poison the opposite triangle: it must never be read
    iu = np.triu_indices(n, 1) if uplo == "l" else np.tril_indices(n, -1)
    for p in range(batch):
        s = store[p].T.copy(); s[iu] = np.nan; store[p] = s.T
    d = torch.from_numpy(store.copy()).to(cuda)
    info = torch.full((batch,), -7, dtype=torch.int32, device=cuda)
    r = pb.dpotrf_batched(uplo, n, d, n, n * n, info, batch)
    assert r.ok()
    got = d.cpu().numpy()
    assert (info.cpu().numpy() == 0).all()
    for p in range(batch):
        g = got[p].T  # logical
        want = F(store[p].T.copy())
        assert orc.dpotrf(ch(uplo), n, ptr(want), n) == 0
        tri = np.tril(np.ones((n, n), bool)) if uplo == "l" else np.triu(np.ones((n, n), bool))
        L = np.where(tri, g, 0.0)
        rec = L @ L.T if uplo == "l" else L.T @ L
        assert rel_frob(rec, A[p]) <= tol(n)                    # backward error
        assert rel_frob(np.where(tri, g, 0), np.where(tri, want, 0)) <= tol(n)
        assert np.isnan(g[~tri]).all()                          # opposite triangle untouched


def test_dpotrf_cfg3_full_batch(pb, cuda):
    """Config 3 at full size (8192 problems, N(0,1) SPD), backward error on every problem."""
    import torch
    g = torch.Generator(device=cuda).manual_seed(3)
    for n in (64, 128):
        batch = 8192
        B = torch.randn((batch, n, n), generator=g, device=cuda, dtype=torch.float64)
        A = B @ B.transpose(1, 2) + n * torch.eye(n, device=cuda, dtype=torch.float64)
        d = A.clone()
        info = torch.empty(batch, dtype=torch.int32, device=cuda)
        assert pb.dpotrf_batched("l", n, d, n, n * n, info, batch).ok()
        torch.cuda.synchronize()
        assert int(info.abs().sum()) == 0
        L = torch.tril(d.transpose(1, 2))  # storage is column-major: logical = transpose of view
        rec = L @ L.transpose(1, 2)
        At = A.transpose(1, 2)
        err = (torch.linalg.matrix_norm(rec - At) / torch.linalg.matrix_norm(At)).max().item()
        assert err <= tol(n)


def test_dpotrf_exact_fixtures(pb):
    # test_factor.cpp:144-158: [[4,2],[2,5]] -> [[2,.],[1,2]], other triangle kept
    a = F([[4.0, -9.0], [2.0, 5.0]])
    assert pb.dpotrf("l", 2, a, 2).ok()
    assert a[0, 0] == 2.0 and a[1, 0] == 1.0 and a[1, 1] == 2.0 and a[0, 1] == -9.0
    a = F([[4.0, 2.0], [-9.0, 5.0]])
    assert pb.dpotrf("u", 2, a, 2).ok()
    assert a[0, 0] == 2.0 and a[0, 1] == 1.0 and a[1, 1] == 2.0 and a[1, 0] == -9.0
    # test_factor.cpp:195-249: dyadic factor recovered bitwise in both triangles
    n = 13
    l0 = dyadic_chol_factor(n)
    A = F(l0 @ l0.T)
    for uplo in "lu":
        d = A.copy(order="F")
        assert pb.dpotrf(uplo, n, d, n).ok()
        want = l0 if uplo == "l" else l0.T
        tri = np.tril(np.ones((n, n), bool)) if uplo == "l" else np.triu(np.ones((n, n), bool))
        assert same_bits(d[tri], want[tri])
        assert same_bits(d[~tri], A[~tri])
    # diag(4,-1,9) -> info 2 (test_blas.cpp:344-351); [[1,2],[2,1]] -> 2; 0 -> 1
    assert pb.dpotrf("l", 3, F(np.diag([4.0, -1.0, 9.0])), 3).info == 2
    assert pb.dpotrf("l", 2, F([[1.0, 2.0], [2.0, 1.0]]), 2).info == 2
    assert pb.dpotrf("l", 1, F([[0.0]]), 1).info == 1


@pytest.mark.parametrize("n,bad", [(13, 8), (13, 0), (40, 21), (64, 63), (100, 37)])
def test_dpotrf_failure_writes_match_reference(pb, orc, n, bad):
    """test_factor.cpp:251-277: info = first bad pivot, and exactly the tiles the
    reference stored before failing are written (the rest keeps its sentinel)."""
    rng = np.random.default_rng(71 + n + bad)
    a = spd(rng, n)
    a[bad, :] = 0.0; a[:, bad] = 0.0; a[bad, bad] = -2.0
    got = a.copy(order="F"); want = a.copy(order="F")
    r = pb.dpotrf("l", n, got, n)
    iw = orc.dpotrf(b"l", n, ptr(want), n)
    assert r.info == iw == bad + 1
    changed_g = ~same_bits_mask(got, a)
    changed_w = ~same_bits_mask(want, a)
    assert (changed_g == changed_w).all()
    assert rel_frob(got, want) <= tol(n)


def same_bits_mask(x, y):
    return np.ascontiguousarray(x).view(np.uint64) == np.ascontiguousarray(y).view(np.uint64)


def test_dpotrf_argument_errors(pb):
    buf = np.zeros(4)
    r = pb.dpotrf("x", 1, buf, 1)
    assert r.info == -1 and r.error.index == 1 and r.error.routine == "dpotrf"
    assert pb.dpotrf("l", -1, buf, 1).info == -2
    assert pb.dpotrf("l", 2, buf, 1).info == -4
    with pytest.raises(pb.ArgError) as e:
        pb.dpotrf("l", 2, buf, 1, cfg=pb.BlasConfig(abort_on_error=True))
    assert e.value.index == 4 and "dpotrf" in str(e.value)


# ----------------------------------------------------------------------------- trsm
def make_tri(rng, uplo, diag, n):
    """matgen.hpp:63-91 recipe."""
    a = rng.uniform(-1, 1, (n, n))
    if diag == "u":
        for j in range(n):
            a[j, j] = 1.0
            for i in range(n):
                if (i > j if uplo == "l" else i < j):
                    a[i, j] *= 0.5 / n
        return F(a)
    for j in range(n):
        rs = sum(abs(a[i, j]) for i in range(n) if (i > j if uplo == "l" else i < j))
        cs = sum(abs(a[j, i]) for i in range(n) if (j > i if uplo == "l" else j < i))
        d = 2.0 * max(rs, cs) + 1.0
        a[j, j] = -d if rng.uniform(0, 1) < 0.5 else d
    return F(a)


@pytest.mark.parametrize("side", ["l", "r"])
@pytest.mark.parametrize("uplo", ["l", "u"])
@pytest.mark.parametrize("trans", ["n", "t"])
@pytest.mark.parametrize("diag", ["n", "u"])
def test_dtrsm_all_flags(pb, orc, side, uplo, trans, diag):
    rng = np.random.default_rng(hash((side, uplo, trans, diag)) % 2**32)
    for (m, n) in [(9, 7), (70, 33), (64, 64), (5, 130)]:
        t = m if side == "l" else n
        a = make_tri(rng, uplo, diag, t)
        b = F(rng.uniform(-1, 1, (m, n)))
        got, want = b.copy(order="F"), b.copy(order="F")
        r = pb.dtrsm(side, uplo, trans, diag, m, n, 1.5, a, t, got, m)
        assert r.ok(), r
        assert orc.dtrsm(ch(side), ch(uplo), ch(trans), ch(diag), m, n, 1.5, ptr(a), t, ptr(want), m) == 0
        assert rel_frob(got, want) <= tol(t)


def test_dtrsm_dyadic_exact_and_zero_diag(pb, orc):
    # test_level3.cpp:345-383 style: dyadic triangle, integer solution, alpha = 2 -> exactly 2*x0
    n, m = 7, 11
    a = F(np.full((n, n), 777.0))
    for j in range(n):
        for i in range(n):
            if i > j:
                a[i, j] = float((i * 7 + j * 3) % 7 - 3)
        a[j, j] = (-1.0 if j % 2 else 1.0) * float(1 << (j % 3))
    x0 = F([[((i * 3 + j * 7 + 2) % 8 + 1) * (-1 if (i + j) % 2 else 1) for j in range(n)] for i in range(m)])
    L = np.tril(a)
    b = F(x0 @ L)  # X * A = B  ('r','l','n','n')
    d = b.copy(order="F")
    assert pb.dtrsm("r", "l", "n", "n", m, n, 2.0, a, n, d, m).ok()
    assert same_bits(d, F(2.0 * x0))
    # zero diagonal -> info before any write (test_level3.cpp:385-409)
    a[2, 2] = 0.0
    d = F(np.full((m, n), -31.5))
    r = pb.dtrsm("r", "l", "n", "n", m, n, 1.0, a, n, d, m)
    assert r.info == 3 and r.error is None
    assert (d == -31.5).all()
    # unit diagonal ignores it; alpha = 0 never reads the triangle
    assert pb.dtrsm("r", "l", "n", "u", m, n, 1.0, a, n, d, m).ok()
    nan_a = F(np.full((n, n), np.nan))
    assert pb.dtrsm("r", "l", "n", "n", m, n, 0.0, nan_a, n, d, m).ok()
    assert (d == 0.0).all()


def test_trsm_rltn_nd(pb, orc):
    rng = np.random.default_rng(91)
    for (m, n) in [(5, 7), (16, 16), (33, 64), (100, 96)]:
        A = make_tri(rng, "l", "n", n)
        Bm = rng.uniform(-1, 1, (m, n))
        ap, bp = pack(A, fill=np.nan), pack(Bm, fill=np.nan)
        d = np.full(panel_len(m, n), 4.25); want = d.copy()
        r = pb.trsm_rltn_nd(m, n, 1.5, pb.PanelRef(ap, n, n), pb.PanelRef(bp, m, n), pb.PanelRef(d, m, n))
        assert r.ok()
        assert orc.trsm_rltn_nd(m, n, 1.5, dmat(ap, n, n), dmat(bp, m, n), dmat(want, m, n)) == 0
        assert rel_frob(unpack(d, m, n), unpack(want, m, n)) <= tol(n)
        # in place: b aliases d
        io = bp.copy()
        assert pb.trsm_rltn_nd(m, n, 1.5, pb.PanelRef(ap, n, n), pb.PanelRef(io, m, n), pb.PanelRef(io, m, n)).ok()
        assert rel_frob(unpack(io, m, n), unpack(want, m, n)) <= tol(n)


def test_trsm_rltn_nd_alpha_zero(pb, orc):
    """level3.hpp:493-504: alpha == 0 -> zero-diagonal check first, then +0 without reading B."""
    rng = np.random.default_rng(5)
    m, n = 9, 12
    A = make_tri(rng, "l", "n", n)
    ap = pack(A, fill=np.nan)
    bp = pack(np.full((m, n), np.inf), fill=np.nan)
    bp[::3] = np.nan
    d = np.full(panel_len(m, n), 4.25)
    want = d.copy()
    assert pb.trsm_rltn_nd(m, n, 0.0, pb.PanelRef(ap, n, n), pb.PanelRef(bp, m, n), pb.PanelRef(d, m, n)).ok()
    assert orc.trsm_rltn_nd(m, n, 0.0, dmat(ap, n, n), dmat(bp, m, n), dmat(want, m, n)) == 0
    assert same_bits(d, want)                       # +0 in the m x n entries, pad lanes untouched
    # a zero diagonal is still reported before any write
    A2 = A.copy(order="F"); A2[4, 4] = 0.0
    ap2 = pack(A2, fill=np.nan)
    d2 = np.full(panel_len(m, n), -3.5)
    r = pb.trsm_rltn_nd(m, n, 0.0, pb.PanelRef(ap2, n, n), pb.PanelRef(bp, m, n), pb.PanelRef(d2, m, n))
    assert r.info == 5 and (d2 == -3.5).all()
    # batched on the device, per-problem info
    import torch
    batch = 3
    L = panel_len(m, n)
    As = torch.from_numpy(np.stack([ap, ap2, ap])).cuda()
    Bs = torch.from_numpy(np.stack([bp] * batch)).cuda()
    Ds = torch.full((batch, L), 7.0, dtype=torch.float64, device="cuda")
    info = torch.full((batch,), -9, dtype=torch.int32, device="cuda")
    P = pb.PanelRef
    assert pb.trsm_rltn_nd_batched(m, n, 0.0, P(As, n, n), n * n, P(Bs, m, n), L, P(Ds, m, n), L, info, batch).ok()
    assert info.cpu().tolist() == [0, 5, 0]
    out = Ds.cpu().numpy()
    want7 = np.full(L, 7.0)
    assert orc.trsm_rltn_nd(m, n, 0.0, dmat(ap, n, n), dmat(bp, m, n), dmat(want7, m, n)) == 0
    assert same_bits(out[0], want7) and same_bits(out[2], want7) and (out[1] == 7.0).all()


def test_dgetrf_host_ipiv_stride_gaps(pb, orc):
    """Strided host ipiv (stride > min(m, n)): the entries between problems survive."""
    rng = np.random.default_rng(17)
    n, batch, sp = 12, 5, 20
    A = rng.uniform(-1, 1, (batch, n, n))
    a = np.ascontiguousarray(A).reshape(-1).copy()
    ipiv = np.full(batch * sp, -77, np.int32)
    info = np.full(batch, 9, np.int32)
    assert pb.dgetrf_batched(n, n, a, n, n * n, ipiv, sp, info, batch).ok()
    assert (info == 0).all()
    for p in range(batch):
        w = F(A[p].T); wp = np.zeros(n, np.int32)
        orc.dgetrf(n, n, ptr(w), n, ptr(wp))
        assert np.array_equal(ipiv[p * sp:p * sp + n], wp)
        assert (ipiv[p * sp + n:(p + 1) * sp] == -77).all()
