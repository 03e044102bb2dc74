"""GPU parity: batched dgemm / dsyrk / gemm_nd / syrk_nd through the C ABI vs the oracle."""
import numpy as np
import pytest

from helpers import F, ch, ptr, rel_frob, same_bits, tol
from oracle.binding import dmat, pack, panel_len, unpack

pytestmark = pytest.mark.gpu


def _cm_batch(rng, rows, cols, batch, ld=None):
    ld = ld or rows
    x = rng.uniform(-1, 1, (batch, cols, ld))  # problem-major, column-major inside
    return x


@pytest.mark.parametrize("ta,tb", [("n", "n"), ("n", "t"), ("t", "n"), ("t", "t")])
@pytest.mark.parametrize("shape", [(64, 64, 64), (13, 9, 7), (1, 1, 1), (70, 33, 45), (128, 96, 160), (3, 130, 2)])
def test_dgemm_batched_device(pb, orc, cuda, ta, tb, shape):
    import torch
    m, n, k = shape
    rng = np.random.default_rng(hash((ta, tb, shape)) % 2**32)
    batch = 5
    ar, ac = (m, k) if ta == "n" else (k, m)
    br, bc = (k, n) if tb == "n" else (n, k)
    A = rng.uniform(-1, 1, (batch, ac, ar))
    B = rng.uniform(-1, 1, (batch, bc, br))
    Cm = rng.uniform(-1, 1, (batch, n, m))
    alpha, beta = 1.5, -0.5
    dA, dB, dC = (torch.from_numpy(x.copy()).to(cuda) for x in (A, B, Cm))
    r = pb.dgemm_batched(ta, tb, m, n, k, alpha, dA, ar, ar * ac, dB, br, br * bc, beta, dC, m, m * n, batch)
    assert r.info == 0 and r.flops == 2 * m * n * k * batch
    got = dC.cpu().numpy()
    for p in range(batch):
        want = F(Cm[p].T)
        a = F(A[p].T)
        b = F(B[p].T)
        orc.dgemm(ch(ta), ch(tb), m, n, k, alpha, ptr(a), ar, ptr(b), br, beta, ptr(want), m)
        assert rel_frob(got[p].T, want) <= tol(k)


@pytest.mark.parametrize("ta,tb", [("n", "n"), ("n", "t"), ("t", "n"), ("t", "t")])
@pytest.mark.parametrize("shape", [(4, 4, 4), (8, 8, 8), (16, 16, 16), (24, 24, 24), (32, 32, 32), (5, 31, 3),
                                   (32, 7, 70), (17, 25, 33), (8, 16, 200), (1, 32, 1)])
def test_dgemm_small_cm(pb, orc, cuda, ta, tb, shape):
    """The small-n branch (gemm_cmsmall.cu: m, n <= 32, warp per problem): every trans pair, ragged
    shapes, k over several 32-chunks, padded and odd leading dimensions, beta = 0 with NaN in C."""
    import torch
    m, n, k = shape
    rng = np.random.default_rng(hash((ta, tb, shape, "small")) % 2**32)
    batch = 37
    ar, ac = (m, k) if ta == "n" else (k, m)
    br, bc = (k, n) if tb == "n" else (n, k)
    for (pa, pb_, pc, alpha, beta) in [(0, 0, 0, 1.0, 1.0), (3, 1, 5, -0.75, 0.0), (2, 4, 2, 1.5, -0.5)]:
        lda, ldb, ldc = ar + pa, br + pb_, m + pc
        A = rng.uniform(-1, 1, (batch, ac, lda))
        B = rng.uniform(-1, 1, (batch, bc, ldb))
        Cm = rng.uniform(-1, 1, (batch, n, ldc))
        if beta == 0.0:
            Cm[:, :, :m] = np.nan  # never read
        dA, dB, dC = (torch.from_numpy(x.copy()).to(cuda) for x in (A, B, Cm))
        r = pb.dgemm_batched(ta, tb, m, n, k, alpha, dA, lda, lda * ac, dB, ldb, ldb * bc, beta, dC, ldc, ldc * n, batch)
        assert r.info == 0 and r.flops == 2 * m * n * k * batch
        got = dC.cpu().numpy()
        for p in range(batch):
            want = F(Cm[p].T)
            a = F(A[p].T)
            b = F(B[p].T)
            orc.dgemm(ch(ta), ch(tb), m, n, k, alpha, ptr(a), lda, ptr(b), ldb, beta, ptr(want), ldc)
            assert not np.isnan(got[p].T[:m]).any()
            assert rel_frob(got[p].T[:m], want[:m]) <= tol(k)
            assert same_bits(got[p].T[m:], F(Cm[p].T)[m:])  # pad rows of C untouched


def test_dgemm_cfg1_full_batch(pb, orc, cuda):
    """Config 1 at full size: 16384 problems of 64^3, alpha = beta = 1; every problem checked."""
    import torch
    m = n = k = 64
    batch = 16384
    g = torch.Generator(device=cuda).manual_seed(7)
    A = torch.rand((batch, k, m), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    B = torch.rand((batch, n, k), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    Cm = torch.rand((batch, n, m), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    # storage is column-major: C^T = C^T + B^T A^T in the (batch, cols, rows) view
    want = torch.baddbmm(Cm, B, A)  # fp64 torch reference
    r = pb.dgemm_batched("n", "n", m, n, k, 1.0, A, m, m * k, B, k, k * n, 1.0, Cm, m, m * n, batch)
    torch.cuda.synchronize()
    assert r.ok()
    err = (torch.linalg.matrix_norm(Cm - want) / torch.linalg.matrix_norm(want)).max().item()
    assert err <= tol(k)


@pytest.mark.parametrize("s", [32, 40, 48, 56, 64])
def test_dgemm_square_nn_beta_zero_nan_c(pb, orc, cuda, s):
    """Square packed NN branch of the size switch: beta = 0 never reads C (NaN C), alpha scaling."""
    import torch
    rng = np.random.default_rng(600 + s)
    batch = 41
    A = rng.uniform(-1, 1, (batch, s, s)); B = rng.uniform(-1, 1, (batch, s, s))
    dA, dB = (torch.from_numpy(x.copy()).to(cuda) for x in (A, B))
    dC = torch.full((batch, s, s), float("nan"), device=cuda, dtype=torch.float64)
    assert pb.dgemm_batched("n", "n", s, s, s, -2.0, dA, s, s * s, dB, s, s * s, 0.0, dC, s, s * s, batch).ok()
    got = dC.cpu().numpy()
    assert np.isfinite(got).all()
    for p in range(0, batch, 8):
        want = np.zeros((s, s), order="F")
        a_p, b_p = F(A[p].T), F(B[p].T)  # keep the operands alive across the call
        orc.dgemm(b"n", b"n", s, s, s, -2.0, ptr(a_p), s, ptr(b_p), s, 0.0, ptr(want), s)
        assert rel_frob(got[p].T, want) <= tol(s)


def test_dgemm_host_pointers_single(pb, orc):
    """The netlib-shaped single call with host buffers (staged through the GPU)."""
    rng = np.random.default_rng(3)
    for (m, n, k) in [(13, 9, 7), (64, 64, 64), (5, 1, 33)]:
        a = F(rng.uniform(-1, 1, (m, k))); b = F(rng.uniform(-1, 1, (k, n))); c = F(rng.uniform(-1, 1, (m, n)))
        got = c.copy(order="F"); want = c.copy(order="F")
        r = pb.dgemm("n", "n", m, n, k, 1.0, a, m, b, k, 1.0, got, m)
        assert r.ok()
        orc.dgemm(b"n", b"n", m, n, k, 1.0, ptr(a), m, ptr(b), k, 1.0, ptr(want), m)
        assert rel_frob(got, want) <= tol(k)


def test_dgemm_integer_data_bitwise(pb, orc):
    """Exact-arithmetic inputs (test_gemm.cpp style): results equal the reference bit for bit."""
    rng = np.random.default_rng(11)
    for (m, n, k) in [(13, 9, 7), (64, 64, 64), (67, 65, 66)]:
        for ta in "nt":
            for tb in "nt":
                a = F(rng.integers(-4, 5, (m, k) if ta == "n" else (k, m)).astype(float))
                b = F(rng.integers(-4, 5, (k, n) if tb == "n" else (n, k)).astype(float))
                c = F(rng.integers(-4, 5, (m, n)).astype(float))
                got, want = c.copy(order="F"), c.copy(order="F")
                assert pb.dgemm(ta, tb, m, n, k, 2.0, a, a.shape[0], b, b.shape[0], -1.0, got, m).ok()
                orc.dgemm(ch(ta), ch(tb), m, n, k, 2.0, ptr(a), a.shape[0], ptr(b), b.shape[0], -1.0, ptr(want), m)
                assert same_bits(got, want)


def test_dgemm_beta_zero_never_reads_c(pb):
    """test_gemm.cpp:264-286: beta = 0 with NaN in C yields clean results."""
    rng = np.random.default_rng(5)
    m, n, k = 21, 17, 9
    a = F(rng.uniform(-1, 1, (m, k))); b = F(rng.uniform(-1, 1, (k, n)))
    c = F(np.full((m, n), np.nan))
    assert pb.dgemm("n", "n", m, n, k, 1.0, a, m, b, k, 0.0, c, m).ok()
    assert np.isfinite(c).all()
    assert rel_frob(c, a @ b) <= tol(k)


def test_dgemm_quick_returns_and_scale(pb):
    """test_blas.cpp:121-170: alpha=0/k=0 paths never touch NaN operands."""
    m, n, k = 5, 4, 3
    a = F(np.full((m, k), np.nan)); b = F(np.full((k, n), np.nan))
    c = F(np.array([[1.0 + i + 10.0 * j for j in range(n)] for i in range(m)]))
    c1 = c.copy(order="F")
    assert pb.dgemm("n", "n", m, n, k, 0.0, a, m, b, k, 1.0, c1, m).ok() and same_bits(c1, c)
    c3 = c.copy(order="F")
    assert pb.dgemm("n", "n", m, n, k, 0.0, a, m, b, k, -2.0, c3, m).ok()
    assert np.array_equal(c3, -2.0 * c)
    c4 = c.copy(order="F")
    assert pb.dgemm("n", "n", m, n, 0, 1.0, a, m, b, k, 0.0, c4, m).ok()
    assert (c4 == 0.0).all()


@pytest.mark.parametrize("s", [4, 8, 12, 28, 36, 48, 60, 64, 72, 84, 100, 108, 132, 320])
def test_gemm_nd_nt_batched(pb, orc, cuda, s):
    """Config 2: panel-major D = A B^T + C (non-destructive), checked per problem."""
    import torch
    rng = np.random.default_rng(s)
    batch = 3
    L = panel_len(s, s)
    A = rng.uniform(-1, 1, (batch, L)); B = rng.uniform(-1, 1, (batch, L)); Cp = rng.uniform(-1, 1, (batch, L))
    dA, dB, dC = (torch.from_numpy(x.copy()).to(cuda) for x in (A, B, Cp))
    dD = torch.full((batch, L), 5.0, device=cuda, dtype=torch.float64)
    r = pb.gemm_nd_batched("n", "t", s, s, s, 1.0, pb.PanelRef(dA, s, s), L, pb.PanelRef(dB, s, s), L,
                           1.0, pb.PanelRef(dC, s, s), L, pb.PanelRef(dD, s, s), L, batch)
    assert r.ok()
    got = dD.cpu().numpy()
    for p in range(batch):
        want = np.full(L, 5.0)
        orc.gemm_nd(b"n", b"t", s, s, s, 1.0, dmat(A[p], s, s), dmat(B[p], s, s), 1.0, dmat(Cp[p], s, s), dmat(want, s, s))
        assert rel_frob(unpack(got[p], s, s), unpack(want, s, s)) <= tol(s)


@pytest.mark.parametrize("s", [4, 8, 16, 32, 44, 56, 76, 96])
def test_gemm_nd_small_alpha_beta_alias(pb, orc, cuda, s):
    """Small-size branch: beta == 0 never reads C (NaN C), alpha scaling, D aliasing C."""
    import torch
    rng = np.random.default_rng(300 + s)
    batch = 37
    L = panel_len(s, s)
    A = rng.uniform(-1, 1, (batch, L)); B = rng.uniform(-1, 1, (batch, L)); Cp = rng.uniform(-1, 1, (batch, L))
    dA, dB = (torch.from_numpy(x.copy()).to(cuda) for x in (A, B))
    dC = torch.full((batch, L), float("nan"), device=cuda, dtype=torch.float64)
    dD = torch.empty((batch, L), device=cuda, dtype=torch.float64)
    R = pb.PanelRef
    assert pb.gemm_nd_batched("n", "t", s, s, s, -1.5, R(dA, s, s), L, R(dB, s, s), L, 0.0, R(dC, s, s), L,
                              R(dD, s, s), L, batch).ok()
    got = dD.cpu().numpy()
    assert not np.isnan(got).any()
    dIO = torch.from_numpy(Cp.copy()).to(cuda)  # in place: D aliases C, beta = 0.5
    assert pb.gemm_nd_batched("n", "t", s, s, s, 1.0, R(dA, s, s), L, R(dB, s, s), L, 0.5, R(dIO, s, s), L,
                              R(dIO, s, s), L, batch).ok()
    io = dIO.cpu().numpy()
    for p in range(0, batch, 6):
        c_nan, want = np.full(L, np.nan), np.zeros(L)
        orc.gemm_nd(b"n", b"t", s, s, s, -1.5, dmat(A[p], s, s), dmat(B[p], s, s), 0.0, dmat(c_nan, s, s),
                    dmat(want, s, s))
        assert rel_frob(unpack(got[p], s, s), unpack(want, s, s)) <= tol(s)
        c_in, want2 = Cp[p].copy(), Cp[p].copy()
        orc.gemm_nd(b"n", b"t", s, s, s, 1.0, dmat(A[p], s, s), dmat(B[p], s, s), 0.5, dmat(c_in, s, s),
                    dmat(want2, s, s))
        assert rel_frob(unpack(io[p], s, s), unpack(want2, s, s)) <= tol(s)


def test_gemm_nd_odd_shapes_and_nn(pb, orc):
    rng = np.random.default_rng(21)
    for (m, n, k) in [(5, 7, 3), (9, 19, 13), (66, 70, 37)]:
        for tb in "nt":
            A = rng.uniform(-1, 1, (m, k)); B = rng.uniform(-1, 1, (k, n) if tb == "n" else (n, k))
            Cm = rng.uniform(-1, 1, (m, n))
            ap, bp, cp = pack(A, fill=np.nan), pack(B, fill=np.nan), pack(Cm, fill=np.nan)
            d = np.full(panel_len(m, n), 9.0); want = d.copy()
            br, bc = B.shape
            r = pb.gemm_nd("n", tb, m, n, k, 0.75, pb.PanelRef(ap, m, k), pb.PanelRef(bp, br, bc), -1.25,
                           pb.PanelRef(cp, m, n), pb.PanelRef(d, m, n))
            assert r.ok()
            orc.gemm_nd(b"n", ch(tb), m, n, k, 0.75, dmat(ap, m, k), dmat(bp, br, bc), -1.25, dmat(cp, m, n), dmat(want, m, n))
            assert rel_frob(unpack(d, m, n), unpack(want, m, n)) <= tol(k)
            # pad lanes of d are untouched (panel_mat.hpp:8-12)
            mask = np.ones(panel_len(m, n), bool)
            i = np.arange(m)[:, None]; j = np.arange(n)[None, :]
            cn = (n + 3) // 4 * 4
            mask[(i // 4) * 4 * cn + j * 4 + i % 4] = False
            assert (d[mask] == 9.0).all()


@pytest.mark.parametrize("uplo", ["l", "u"])
@pytest.mark.parametrize("trans", ["n", "t"])
def test_dsyrk(pb, orc, uplo, trans):
    rng = np.random.default_rng(31)
    for (n, k) in [(11, 6), (64, 64), (100, 37)]:
        a = F(rng.uniform(-1, 1, (n, k) if trans == "n" else (k, n)))
        c = F(rng.uniform(-1, 1, (n, n)))
        got, want = c.copy(order="F"), c.copy(order="F")
        assert pb.dsyrk(uplo, trans, n, k, 1.25, a, a.shape[0], -0.75, got, n).ok()
        orc.dsyrk(ch(uplo), ch(trans), n, k, 1.25, ptr(a), a.shape[0], -0.75, ptr(want), n)
        assert rel_frob(got, want) <= tol(k)
        tri = np.tril(np.ones((n, n), bool), -1) if uplo == "u" else np.triu(np.ones((n, n), bool), 1)
        assert same_bits(got[tri], c[tri])  # opposite triangle untouched


@pytest.mark.parametrize("uplo", ["l", "u"])
@pytest.mark.parametrize("trans", ["n", "t"])
@pytest.mark.parametrize("nk", [(4, 4), (8, 3), (16, 40), (23, 17), (32, 32)])
def test_dsyrk_small_batched(pb, orc, cuda, uplo, trans, nk):
    """dsyrk at n <= 32 (the warp-per-problem small-n branch): both triangles and trans, padded
    leading dimensions, beta = 0 with NaN in the stored triangle; the opposite triangle untouched."""
    import torch
    n, k = nk
    rng = np.random.default_rng(n * 100 + k)
    batch = 19
    ar, ac = (n, k) if trans == "n" else (k, n)
    tri = np.tril(np.ones((n, n), bool)) if uplo == "l" else np.triu(np.ones((n, n), bool))
    for (pa, pc, alpha, beta) in [(0, 0, 1.0, 1.0), (3, 1, -0.5, 0.0), (2, 2, 1.25, -2.0)]:
        lda, ldc = ar + pa, n + pc
        A = rng.uniform(-1, 1, (batch, ac, lda))
        C = rng.uniform(-1, 1, (batch, n, ldc))
        if beta == 0.0:  # NaN in the triangle dsyrk overwrites (never read)
            Cv = C[:, :, :n]              # [p, j, i]
            Cv[:, tri.T] = np.nan
        dA, dC = torch.from_numpy(A.copy()).to(cuda), torch.from_numpy(C.copy()).to(cuda)
        r = pb.dsyrk_batched(uplo, trans, n, k, alpha, dA, lda, lda * ac, beta, dC, ldc, ldc * n, batch)
        assert r.info == 0
        got = dC.cpu().numpy()
        for p in range(batch):
            a = F(A[p].T)
            c0 = F(C[p].T)
            want = c0.copy(order="F")
            orc.dsyrk(ch(uplo), ch(trans), n, k, alpha, ptr(a), lda, beta, ptr(want), ldc)
            g, w = got[p].T[:n], want[:n]
            assert not np.isnan(g[tri]).any()
            assert np.linalg.norm(g[tri] - w[tri]) <= tol(k) * max(np.linalg.norm(w[tri]), 1e-300)
            assert same_bits(g[~tri], c0[:n][~tri])        # opposite triangle untouched
            assert same_bits(got[p].T[n:], c0[n:])          # pad rows untouched


def test_syrk_nd(pb, orc):
    rng = np.random.default_rng(41)
    for (n, k) in [(13, 7), (64, 64), (96, 20)]:
        A = rng.uniform(-1, 1, (n, k)); Cs = rng.uniform(-1, 1, (n, n))
        ap, cp = pack(A), pack(Cs)
        d = np.full(panel_len(n, n), 3.5); want = d.copy()
        assert pb.syrk_nd(n, k, 1.0, pb.PanelRef(ap, n, k), 1.0, pb.PanelRef(cp, n, n), pb.PanelRef(d, n, n)).ok()
        orc.syrk_nd(n, k, 1.0, dmat(ap, n, k), 1.0, dmat(cp, n, n), dmat(want, n, n))
        assert rel_frob(unpack(d, n, n), unpack(want, n, n)) <= tol(k)
        assert rel_frob(d, want) <= tol(k)  # includes the untouched upper part


@pytest.mark.parametrize("s", [4, 48, 96])
def test_gemm_nd_cfg2_full_batch(pb, cuda, s):
    """Config 2 at full size (batch = 2^31 / (32 s^2)) on the size-switched kernels: every problem
    checked against torch fp64 through the panel-major layout (element (i, j) at (i/4)*4s + 4j + i%4)."""
    import torch
    batch = (2 ** 31) // (32 * s * s)
    L = s * s
    g = torch.Generator(device=cuda).manual_seed(s)
    A = torch.rand((batch, L), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    B = torch.rand((batch, L), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    C = torch.rand((batch, L), generator=g, device=cuda, dtype=torch.float64) * 2 - 1
    D = torch.empty_like(A)
    R = pb.PanelRef
    assert pb.gemm_nd_batched("n", "t", s, s, s, 1.0, R(A, s, s), L, R(B, s, s), L, 1.0, R(C, s, s), L,
                              R(D, s, s), L, batch).ok()

    def dense(x):  # (batch, s/4 panels, s cols, 4 rows) -> (batch, s rows, s cols)
        return x.view(batch, s // 4, s, 4).permute(0, 1, 3, 2).reshape(batch, s, s)
    want = dense(A) @ dense(B).transpose(1, 2) + dense(C)
    err = (torch.linalg.matrix_norm(dense(D) - want) / torch.linalg.matrix_norm(want)).max().item()
    assert err <= tol(s)


def test_host_pointer_calls_from_concurrent_threads(pb, orc):
    """§8(b) threading: host-pointer calls from several threads at once (each thread has its
    own staging streams and buffers) all match the oracle."""
    import threading
    rng = np.random.default_rng(42)
    m = n = k = 40
    batch = 600
    jobs = []
    for _ in range(4):
        A = rng.uniform(-1, 1, (batch, k, m)); B = rng.uniform(-1, 1, (batch, n, k)); C = rng.uniform(-1, 1, (batch, n, m))
        jobs.append([A, B, C, C.copy()])
    errors = []

    def work(job):
        try:
            A, B, C, out = job
            for _ in range(3):
                out[:] = C
                r = pb.dgemm_batched("n", "n", m, n, k, 1.0, A, m, m * k, B, k, k * n, 1.0, out, m, m * n, batch)
                assert r.ok(), r
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=work, args=(j,)) for j in jobs]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for A, B, C, out in jobs:
        want = C.copy()
        orc.dgemm_batch(b"n", b"n", m, n, k, 1.0, A.ctypes.data, m, m * k, B.ctypes.data, k, k * n, 1.0,
                        want.ctypes.data, m, m * n, batch, 4)
        assert rel_frob(out, want) <= tol(k)
