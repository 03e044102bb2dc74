"""Special-value pivots on every size class of the factorization kernels, against the oracle.

dpotrf (micro_kernel.hpp:309-325 edge_potrf): only ``piv <= 0`` fails — a denormal positive
pivot is an ordinary pivot, a +Inf pivot gives L_jj = Inf and a zero column below it
(1/Inf = 0), a NaN pivot does NOT fail (NaN <= 0 is false) and propagates.
dgetrf (factor.hpp:141-158): the strict ``>`` scan never picks a NaN candidate, a NaN
diagonal keeps its row, an Inf candidate wins, and an exactly zero pivot records info
without swapping.  Sizes cover potrf_reg (n <= 32), potrf_cta (33..160) and the blocked
path (> 160); getrf_reg (<= 32), getrf_sq (square 40..96, also the trailing block of the
blocked path: 104, 160, 192), getrf_cta (other shapes < 80) and the blocked getrf_rows path.
"""
import numpy as np
import pytest

from helpers import F, ptr, tol

pytestmark = pytest.mark.gpu


def same_special(got, want, n, what=""):
    """NaN and Inf positions identical (Inf sign included); finite entries within 1e-13 n."""
    gn, wn = np.isnan(got), np.isnan(want)
    assert np.array_equal(gn, wn), f"{what}: NaN pattern differs at {np.argwhere(gn != wn)[:4].tolist()} (gpu NaN: {gn[gn != wn][:4].tolist()})"
    gi, wi = np.isinf(got), np.isinf(want)
    assert np.array_equal(gi, wi) and np.array_equal(got[gi], want[wi])
    fin = np.isfinite(want)
    g, w = got[fin], want[fin]
    den = np.linalg.norm(w)
    assert np.linalg.norm(g - w) <= tol(n) * (den if den > 0 else 1.0)


def dyadic_lower(rng, n):
    """Lower factor with dyadic entries: A = L L^T is exact in fp64."""
    L = np.tril(rng.integers(-8, 9, (n, n)) / 8.0, -1)
    L[np.arange(n), np.arange(n)] = 2.0 + rng.integers(0, 3, n)
    return L


def potrf_cases(rng, n):
    cases = []
    for j in sorted({0, min(1, n - 1), n // 2, min(7, n - 1), min(8, n - 1), n - 1}):
        L = dyadic_lower(rng, n)
        # denormal pivot at column j: row j of L empty left of the diagonal, L_jj = 2^-520
        L[j, :j] = 0.0
        L[j, j] = 2.0 ** -520
        A = L @ L.T
        assert A[j, j] == 2.0 ** -1040 and 0 < A[j, j] < np.finfo(float).tiny
        cases.append(("denormal", j, A))
        A = dyadic_lower(rng, n); A = A @ A.T
        A[j, j] = np.inf
        cases.append(("inf", j, A))
        A = dyadic_lower(rng, n); A = A @ A.T
        A[j, j] = np.nan
        cases.append(("nan_diag", j, A))
        if j + 1 < n:
            A = dyadic_lower(rng, n); A = A @ A.T
            A[n - 1, j] = A[j, n - 1] = np.nan     # NaN below the diagonal of column j
            cases.append(("nan_below", j, A))
    return cases


@pytest.mark.parametrize("n", [4, 8, 16, 24, 32, 40, 64, 100, 128, 160, 200])
def test_dpotrf_special_pivots(pb, orc, cuda, n):
    import torch
    rng = np.random.default_rng(n)
    cases = potrf_cases(rng, n)
    batch = len(cases)
    H = np.stack([c[2].T for c in cases])  # (batch, j, i): column-major problems
    d = torch.from_numpy(H.copy()).to(cuda)
    info = torch.full((batch,), -9, dtype=torch.int32, device=cuda)
    assert pb.dpotrf_batched("l", n, d, n, n * n, info, batch).ok()
    got, gi = d.cpu().numpy(), info.cpu().numpy()
    lo = np.tril(np.ones((n, n), bool))
    for p, (kind, j, A) in enumerate(cases):
        w = F(A.copy())
        wi = orc.dpotrf(b"l", n, ptr(w), n)
        assert gi[p] == wi, (kind, j, gi[p], wi)
        g = got[p].T
        if wi == 0:
            same_special(g[lo], w[lo], n, (kind, j))
        if kind == "denormal":
            assert wi == 0 and g[j, j] == 2.0 ** -520     # accepted as an ordinary pivot, exact sqrt
        if kind == "nan_diag":
            assert wi == 0 and np.isnan(g[j, j])          # NaN <= 0 is false: no failure
    # single-call host path, denormal case through pb_dpotrf
    kind, j, A = cases[0]
    a = F(A.copy()); w = F(A.copy())
    r = pb.dpotrf("l", n, a, n)
    assert r.info == orc.dpotrf(b"l", n, ptr(w), n)
    same_special(a[lo], w[lo], n)


def getrf_cases(rng, n):
    cases = []
    for j in sorted({0, n // 3, n // 2, n - 1}):
        A = rng.uniform(-1, 1, (n, n))
        A[min(j + 1, n - 1), j] = np.nan if j + 1 < n else A[j, j]   # NaN candidate below the diagonal
        cases.append(("nan_candidate", j, A))
        A = rng.uniform(-1, 1, (n, n))
        A[j, j] = np.nan                                             # NaN diagonal keeps its row
        cases.append(("nan_diag", j, A))
        A = rng.uniform(-1, 1, (n, n))
        A[n - 1, j] = np.inf                                         # Inf candidate wins
        cases.append(("inf_candidate", j, A))
        A = rng.uniform(-1, 1, (n, n))
        A[:, j] = 0.0                                                # zero column: info j + 1, no swap
        cases.append(("zero_col", j, A))
    # denormal first column (finite reciprocal 2^1026 / k): exact dyadic multipliers
    A = rng.uniform(-1, 1, (n, n))
    A[:, 0] = 2.0 ** -1026 * rng.integers(1, 9, n) * rng.choice([-1.0, 1.0], n)
    cases.append(("denormal_col", 0, A))
    return cases


@pytest.mark.parametrize("n", [3, 8, 24, 32, 40, 48, 64, 79, 88, 96, 104, 130, 160, 192])
def test_dgetrf_special_pivots(pb, orc, cuda, n):
    import torch
    rng = np.random.default_rng(1000 + n)
    cases = getrf_cases(rng, n)
    batch = len(cases)
    H = np.stack([c[2].T for c in cases])
    d = torch.from_numpy(H.copy()).to(cuda)
    ipiv = torch.zeros((batch, n), dtype=torch.int32, device=cuda)
    info = torch.full((batch,), -9, dtype=torch.int32, device=cuda)
    assert pb.dgetrf_batched(n, n, d, n, n * n, ipiv, n, info, batch).ok()
    got, gp, gi = d.cpu().numpy(), ipiv.cpu().numpy(), info.cpu().numpy()
    for p, (kind, j, A) in enumerate(cases):
        w = F(A.copy()); wp = np.zeros(n, np.int32)
        wi = orc.dgetrf(n, n, ptr(w), n, ptr(wp))
        assert gi[p] == wi, (kind, j, gi[p], wi)
        assert np.array_equal(gp[p], wp), (kind, j, np.nonzero(gp[p] != wp)[0][:5])
        same_special(got[p].T, w, n, (kind, j))
        if kind == "zero_col":
            assert 0 < wi <= j + 1
