"""Shared test helpers: seeded inputs, tolerances, bit comparisons."""
import numpy as np

from oracle.binding import ch, ptr  # noqa: F401  (re-exported for tests)


def F(a):
    return np.asfortranarray(a, dtype=np.float64)


def same_bits(x: np.ndarray, y: np.ndarray) -> bool:
    return np.array_equal(np.ascontiguousarray(x).view(np.uint64), np.ascontiguousarray(y).view(np.uint64))


def rel_frob(got: np.ndarray, want: np.ndarray) -> float:
    """||got - want||_F / max(||want||_F, tiny) — the north-star metric."""
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (den if den > 0 else 1.0))


def tol(n: int) -> float:
    """BASELINE.json north star: relative Frobenius error <= 1e-13 * n."""
    return 1e-13 * max(n, 1)
