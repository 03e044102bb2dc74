"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU oracle.

Two libraries, both built by ``oracle/Makefile`` (and ``__graft_entry__.build()``):

* ``_build/liboracle.so`` — the plain-C restatement (``pb_oracle.c``), prefix ``orc_``;
* ``_ref/libpanelblas_ref.so`` — the reference's own headers compiled in place
  behind ``ref_shim.cpp``, prefix ``ref_`` (present only where
  ``/root/reference`` was available when it was built).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg import this module.  Matrices are numpy float64
arrays in Fortran (column-major) order; panel-major operands are flat arrays
plus a shape, mirroring ``panelblas::PanelRef`` (panel_mat.hpp:51-81).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpanelblas_ref.so")


class Dmat(C.Structure):
    """Byte-compatible with pb_dmat / panelblas::PanelRef {data, ps, m, n, pm, cn}."""

    _fields_ = [("data", C.c_void_p), ("ps", C.c_int), ("m", C.c_int), ("n", C.c_int),
                ("pm", C.c_int), ("cn", C.c_int)]


def round_up(v: int, q: int) -> int:
    return (v + q - 1) // q * q


def panel_len(m: int, n: int, ps: int = 4) -> int:
    return round_up(m, ps) * round_up(n, ps)


def dmat(buf: np.ndarray, m: int, n: int, ps: int = 4) -> Dmat:
    return Dmat(buf.ctypes.data, ps, m, n, round_up(m, ps), round_up(n, ps))


def pack(a: np.ndarray, ps: int = 4, fill: float = 0.0) -> np.ndarray:
    """Column-major (m, n) -> flat panel-major buffer (panel_mat.hpp:141-160)."""
    m, n = a.shape
    pm, cn = round_up(m, ps), round_up(n, ps)
    out = np.full(pm * cn, fill)
    i = np.arange(m)[:, None]
    j = np.arange(n)[None, :]
    out[(i // ps) * ps * cn + j * ps + i % ps] = a
    return out


def unpack(buf: np.ndarray, m: int, n: int, ps: int = 4) -> np.ndarray:
    """Flat panel-major buffer -> Fortran (m, n) array (panel_mat.hpp:164-171)."""
    cn = round_up(n, ps)
    i = np.arange(m)[:, None]
    j = np.arange(n)[None, :]
    return np.asfortranarray(buf[(i // ps) * ps * cn + j * ps + i % ps])


_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_CH = C.c_char
_LL = C.c_longlong

_SIGS = {
    "dgemm": (_I, [_CH, _CH, _I, _I, _I, _D, _P, _I, _P, _I, _D, _P, _I]),
    "dsyrk": (_I, [_CH, _CH, _I, _I, _D, _P, _I, _D, _P, _I]),
    "dtrsm": (_I, [_CH, _CH, _CH, _CH, _I, _I, _D, _P, _I, _P, _I]),
    "dpotrf": (_I, [_CH, _I, _P, _I]),
    "dgetrf": (_I, [_I, _I, _P, _I, _P]),
    "gemm_nd": (_I, [_CH, _CH, _I, _I, _I, _D, Dmat, Dmat, _D, Dmat, Dmat]),
    "syrk_nd": (_I, [_I, _I, _D, Dmat, _D, Dmat, Dmat]),
    "trsm_rltn_nd": (_I, [_I, _I, _D, Dmat, Dmat, Dmat]),
    "syrk_potrf_nd": (_I, [_I, _I, Dmat, Dmat, Dmat, Dmat]),
    "dgemm_batch": (None, [_CH, _CH, _I, _I, _I, _D, _P, _I, _LL, _P, _I, _LL, _D, _P, _I, _LL,
                           _LL, _I]),
    "dpotrf_batch": (None, [_CH, _I, _P, _I, _LL, _P, _LL, _I]),
    "dgetrf_batch": (None, [_I, _I, _P, _I, _LL, _P, _LL, _P, _LL, _I]),
    "dtrmm": (_I, [_CH, _CH, _CH, _CH, _I, _I, _D, _P, _I, _P, _I]),
    "trmm_rlnn_nd": (_I, [_I, _I, _D, Dmat, Dmat, Dmat]),
    "gemm_nd_batch": (None, [_CH, _CH, _I, _I, _I, _D, Dmat, _LL, Dmat, _LL, _D, Dmat, _LL, Dmat,
                             _LL, _LL, _I]),
    "chain_batch": (None, [_I, _P, _P, _P, _P, _P, _P, _LL, _I]),
}
_REF_ONLY = {
    "naive_gemm": (None, [_CH, _CH, _I, _I, _I, _D, _P, _I, _P, _I, _D, _P, _I]),
    "naive_potrf": (_I, [_CH, _I, _P, _I]),
    "naive_getrf": (_I, [_I, _I, _P, _I, _P]),
    "naive_trsm": (_I, [_CH, _CH, _CH, _CH, _I, _I, _D, _P, _I, _P, _I]),
    "naive_trmm": (None, [_CH, _CH, _CH, _CH, _I, _I, _D, _P, _I, _P, _I]),
    "rng_uniform": (None, [C.c_uint64, _LL, _D, _D, _P]),
    "make_spd": (None, [_I, C.c_uint64, _P]),
    "hw_threads": (_I, []),
    "last_error_index": (_I, []),
    "chain_cm_batch": (None, [_P, _P, _P, _P, _P, _P, _LL, _I]),
    "chain_pm_batch": (None, [_P, _P, _P, _P, _P, _P, _LL, _I]),
    "pack_from_colmajor": (None, [_CH, _P, _I, _I, _I, Dmat]),
    "unpack_to_colmajor": (None, [Dmat, _P, _I]),
    "memsize": (_LL, [_I, _I, _I]),
    "make_ocp_data": (None, [_I, _I, C.c_uint64, _P, _P, _P, _P, _P]),
    "riccati_fused": (_I, [_I, _I, _I, C.c_uint64, _P, _P, C.POINTER(_I)]),
    "riccati_run": (_D, [_I, _I, _I, _I, C.c_uint64, C.POINTER(_I)]),
    "chol_residual": (_D, [_I, _P, _I, _P, _I]),
    "riccati_oracle_step": (_I, [_I, _I, C.c_uint64, _P, _P]),
    "riccati_seed": (C.c_uint64, []),
}


class _Lib:
    def __init__(self, path: str, prefix: str, sigs: dict):
        self.path = path
        self.lib = C.CDLL(path)
        for name, (res, args) in sigs.items():
            sym = prefix + name
            if not hasattr(self.lib, sym):
                continue
            f = getattr(self.lib, sym)
            f.restype = res
            f.argtypes = args
            setattr(self, name, f)


_cache: dict = {}


def oracle() -> _Lib:
    """The plain-C restatement (always built)."""
    if "orc" not in _cache:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle oracle`")
        _cache["orc"] = _Lib(ORACLE_SO, "orc_", _SIGS)
    return _cache["orc"]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref() -> _Lib:
    """The reference library compiled from /root/reference (oracle/_ref)."""
    if "ref" not in _cache:
        if not have_ref():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        _cache["ref"] = _Lib(REF_SO, "ref_", {**_SIGS, **_REF_ONLY})
    return _cache["ref"]


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def ch(c: str) -> bytes:
    return c.encode()
