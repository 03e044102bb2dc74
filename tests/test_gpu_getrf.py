"""GPU parity: batched dgetrf — pivots bit-exact vs the oracle, PA = LU backward error, exact fixtures."""
import numpy as np
import pytest

from helpers import F, ch, ptr, rel_frob, same_bits, tol

pytestmark = pytest.mark.gpu


def lu_parts(d, m, n):
    k = min(m, n)
    L = np.tril(d[:, :k], -1) + np.eye(m, k)
    U = np.triu(d[:k, :])
    return L, U


def apply_swaps(a, ipiv):
    pa = a.copy()
    for j, p in enumerate(ipiv):
        p -= 1
        if p != j:
            pa[[j, p], :] = pa[[p, j], :]
    return pa


@pytest.mark.parametrize("shape", [(24, 24), (48, 48), (96, 96), (192, 192), (13, 13), (9, 19), (19, 9),
                                   (1, 1), (160, 160), (200, 150), (70, 250),
                                   # getrf_sq: every order 40..96, and blocked paths whose trailing
                                   # square block (72, 96, 40) runs on it with its left-column interchanges
                                   (40, 40), (56, 56), (64, 64), (72, 72), (80, 80), (88, 88),
                                   (104, 104), (128, 128), (136, 136)])
def test_dgetrf_batched_vs_oracle(pb, orc, cuda, shape):
    import torch
    m, n = shape
    rng = np.random.default_rng(m * 1000 + n)
    batch = 8
    A = rng.uniform(-1, 1, (batch, n, m))  # problem-major, column-major inside
    d = torch.from_numpy(A.copy()).to(cuda)
    k = min(m, n)
    ipiv = torch.zeros((batch, k), dtype=torch.int32, device=cuda)
    info = torch.full((batch,), -5, dtype=torch.int32, device=cuda)
    assert pb.dgetrf_batched(m, n, d, m, m * n, ipiv, k, info, batch).ok()
    got, gp, gi = d.cpu().numpy(), ipiv.cpu().numpy(), info.cpu().numpy()
    for p in range(batch):
        a = F(A[p].T)
        want = a.copy(order="F"); wp = np.zeros(k, np.int32)
        wi = orc.dgetrf(m, n, ptr(want), m, ptr(wp))
        assert gi[p] == wi
        assert np.array_equal(gp[p], wp)                       # pivots bit-exact
        g = got[p].T
        L, U = lu_parts(g, m, n)
        assert rel_frob(L @ U, apply_swaps(a, gp[p])) <= tol(max(m, n))  # backward error
        assert rel_frob(g, want) <= tol(max(m, n)) * 10


def test_dgetrf_cfg4_full_batch(pb, orc, cuda):
    """Config 4 at full size: 8192 problems per n; pivots vs the oracle on a seeded subset
    (first and last problems included), backward error on every problem (GPU-side)."""
    import torch
    for n in (24, 48, 96, 192):
        batch = 8192
        g = torch.Generator(device=cuda).manual_seed(n)
        A = torch.rand((batch, n, n), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
        d = A.clone()
        ipiv = torch.zeros((batch, n), dtype=torch.int32, device=cuda)
        info = torch.empty(batch, dtype=torch.int32, device=cuda)
        assert pb.dgetrf_batched(n, n, d, n, n * n, ipiv, n, info, batch).ok()
        torch.cuda.synchronize()
        assert int(info.abs().sum()) == 0
        # backward error ||P A - L U|| / ||A|| on all problems
        dt = d.transpose(1, 2)
        L = torch.tril(dt, -1) + torch.eye(n, device=cuda, dtype=torch.float64)
        U = torch.triu(dt)
        PA = A.transpose(1, 2).clone()
        ip = ipiv.long() - 1
        rows = torch.arange(batch, device=cuda)
        for j in range(n):
            pj = ip[:, j]
            tmp = PA[rows, j, :].clone()
            PA[rows, j, :] = PA[rows, pj, :]
            PA[rows, pj, :] = tmp
        err = (torch.linalg.matrix_norm(L @ U - PA) / torch.linalg.matrix_norm(PA)).max().item()
        assert err <= tol(n)
        sub = [0, 1, 2, 3, batch // 2, batch - 2, batch - 1]
        Ah = A[sub].cpu().numpy(); gp = ipiv[sub].cpu().numpy()
        for q in range(len(sub)):
            a = F(Ah[q].T); wp = np.zeros(n, np.int32)
            orc.dgetrf(n, n, ptr(a), n, ptr(wp))
            assert np.array_equal(gp[q], wp)


def lu_plant(m, n, zero_col2=False):
    """test_factor.cpp:70-100 recipe (exact dyadic L and U)."""
    k = min(m, n)
    l = np.zeros((m, k)); u = np.zeros((k, n))
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
    return l, u, F(l @ u)


def test_dgetrf_exact_fixtures(pb, orc):
    # permutation: ipiv {2,2}, L = U = I (test_factor.cpp:351-365)
    a = F([[0.0, 1.0], [1.0, 0.0]]); ip = np.zeros(2, np.int32)
    assert pb.dgetrf(2, 2, a, 2, ip).ok()
    assert list(ip) == [2, 2] and np.array_equal(a, np.eye(2))
    # singular: info 2, bitwise equal to the oracle
    s = F([[1.0, 2.0], [2.0, 4.0]]); w = s.copy(order="F"); ip = np.zeros(2, np.int32); wp = ip.copy()
    assert pb.dgetrf(2, 2, s, 2, ip).info == 2
    assert orc.dgetrf(2, 2, ptr(w), 2, ptr(wp)) == 2
    assert same_bits(s, w) and np.array_equal(ip, wp)
    # planted dyadic LU behind a row rotation: bitwise L, U and pivots (test_factor.cpp:395-440)
    for (m, n) in [(13, 13), (9, 19), (19, 9)]:
        l, u, comp = lu_plant(m, n)
        a = F(np.zeros((m, n)))
        for i in range(m):
            a[(i + 3) % m, :] = comp[i, :]
        d = a.copy(order="F"); w = a.copy(order="F")
        k = min(m, n); ip = np.zeros(k, np.int32); wp = ip.copy()
        assert pb.dgetrf(m, n, d, m, ip).ok()
        assert orc.dgetrf(m, n, ptr(w), m, ptr(wp)) == 0
        assert np.array_equal(ip, wp) and same_bits(d, w)
        if m <= n:
            want = np.where(np.tril(np.ones((m, n), bool), -1), np.pad(l, ((0, 0), (0, n - k))), np.pad(u, ((0, m - k), (0, 0))))
            assert same_bits(d, F(want))
    # zero pivot column: info 3, ipiv[2] = 3, rest is the plant (test_factor.cpp:442-467)
    l, u, comp = lu_plant(6, 6, zero_col2=True)
    d = comp.copy(order="F"); ip = np.zeros(6, np.int32)
    r = pb.dgetrf(6, 6, d, 6, ip)
    assert r.info == 3 and ip[2] == 3
    want = np.where(np.tril(np.ones((6, 6), bool), -1), l, u)
    assert same_bits(d, F(want))


def test_dgetrf_padded_ld_and_errors(pb):
    rng = np.random.default_rng(63)
    m = n = 6; ld = 9
    a = rng.uniform(-2, 2, (m, n))
    padded = F(np.full((ld, n), -4.5)); padded[:m, :] = a
    ip = np.zeros(6, np.int32)
    assert pb.dgetrf(m, n, padded, ld, ip).ok()
    assert (padded[m:, :] == -4.5).all()
    buf = np.zeros(4); ip = np.zeros(2, np.int32)
    r = pb.dgetrf(-1, 1, buf, 1, ip)
    assert r.info == -1 and r.error.index == 1
    assert pb.dgetrf(1, -1, buf, 1, ip).info == -2
    assert pb.dgetrf(2, 1, buf, 1, ip).info == -4
