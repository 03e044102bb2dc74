"""paper_1902_08115_b200 — B200-native batched FP64 small-matrix BLAS/LAPACK.

Python mirror of the reference's hot-path interface (panelblas,
/root/reference/proj/include/panelblas/): the netlib-shaped adapters
``dgemm / dsyrk / dtrsm / dpotrf / dgetrf`` (blas.hpp:73-215), the native
panel-major routines ``gemm_nd / syrk_nd / trsm_rltn_nd / syrk_potrf_nd``
(level3.hpp:360-575), plus batched and variable-size forms.  Everything goes
through the C ABI of ``libpbgpu.so`` (include/pbgpu.h) into sm_100a kernels;
there is no CPU compute path, and importing this package without the built
library raises.

Array arguments may be numpy arrays (host memory: the call stages through the
GPU and returns when done), torch CUDA tensors (device memory: the call is
asynchronous on ``stream``) or raw integer addresses.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

__all__ = [
    "ArgError", "BlasCallError", "BlasConfig", "BlasResult", "PanelRef", "lib", "library_path",
    "dgemm", "dsyrk", "dtrsm", "dpotrf", "dgetrf",
    "gemm_nd", "syrk_nd", "trsm_rltn_nd", "syrk_potrf_nd",
    "dgemm_batched", "dsyrk_batched", "dtrsm_batched", "dpotrf_batched", "dgetrf_batched",
    "gemm_nd_batched", "syrk_nd_batched", "trsm_rltn_nd_batched", "syrk_potrf_nd_batched",
    "chain_vbatched", "dtrmm", "dtrmm_batched", "trmm_rlnn_nd", "trmm_rlnn_nd_batched",
    "memsize", "pack", "pack_batched", "unpack", "unpack_batched", "riccati_nd_batched",
    "INFO_UNSUPPORTED", "INFO_CUDA_ERROR", "INFO_NO_DEVICE",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_PKG, "libpbgpu.so")

INFO_UNSUPPORTED = -1000
INFO_CUDA_ERROR = -2000
INFO_NO_DEVICE = -2001


class _Dmat(C.Structure):
    _fields_ = [("data", C.c_void_p), ("ps", C.c_int), ("m", C.c_int), ("n", C.c_int),
                ("pm", C.c_int), ("cn", C.c_int)]


class _Result(C.Structure):
    _fields_ = [("info", C.c_int), ("error_index", C.c_int), ("routine", C.c_char_p),
                ("message", C.c_char_p), ("flops", C.c_longlong)]


_P, _I, _D, _CH, _LL = C.c_void_p, C.c_int, C.c_double, C.c_char, C.c_longlong
_R = C.POINTER(_Result)
_SIGS = {
    "pb_version": (_I, []),
    "pb_device_count": (_I, []),
    "pb_probe_dmma_tflops": (_D, []),
    "pb_dgemm": (_I, [_CH, _CH, _I, _I, _I, _D, _P, _I, _P, _I, _D, _P, _I, _R]),
    "pb_dsyrk": (_I, [_CH, _CH, _I, _I, _D, _P, _I, _D, _P, _I, _R]),
    "pb_dtrsm": (_I, [_CH, _CH, _CH, _CH, _I, _I, _D, _P, _I, _P, _I, _R]),
    "pb_dpotrf": (_I, [_CH, _I, _P, _I, _R]),
    "pb_dgetrf": (_I, [_I, _I, _P, _I, _P, _R]),
    "pb_gemm_nd": (_I, [_CH, _CH, _I, _I, _I, _D, _Dmat, _Dmat, _D, _Dmat, _Dmat, _R]),
    "pb_syrk_nd": (_I, [_I, _I, _D, _Dmat, _D, _Dmat, _Dmat, _R]),
    "pb_trsm_rltn_nd": (_I, [_I, _I, _D, _Dmat, _Dmat, _Dmat, _R]),
    "pb_syrk_potrf_nd": (_I, [_I, _I, _Dmat, _Dmat, _Dmat, _Dmat, _R]),
    "pb_dgemm_batched": (_I, [_CH, _CH, _I, _I, _I, _D, _P, _I, _LL, _P, _I, _LL, _D, _P, _I, _LL,
                              _I, _P, _R]),
    "pb_dsyrk_batched": (_I, [_CH, _CH, _I, _I, _D, _P, _I, _LL, _D, _P, _I, _LL, _I, _P, _R]),
    "pb_dtrsm_batched": (_I, [_CH, _CH, _CH, _CH, _I, _I, _D, _P, _I, _LL, _P, _I, _LL, _P, _I, _P,
                              _R]),
    "pb_dpotrf_batched": (_I, [_CH, _I, _P, _I, _LL, _P, _I, _P, _R]),
    "pb_dgetrf_batched": (_I, [_I, _I, _P, _I, _LL, _P, _LL, _P, _I, _P, _R]),
    "pb_gemm_nd_batched": (_I, [_CH, _CH, _I, _I, _I, _D, _Dmat, _LL, _Dmat, _LL, _D, _Dmat, _LL,
                                _Dmat, _LL, _I, _P, _R]),
    "pb_syrk_nd_batched": (_I, [_I, _I, _D, _Dmat, _LL, _D, _Dmat, _LL, _Dmat, _LL, _I, _P, _R]),
    "pb_trsm_rltn_nd_batched": (_I, [_I, _I, _D, _Dmat, _LL, _Dmat, _LL, _Dmat, _LL, _P, _I, _P,
                                     _R]),
    "pb_syrk_potrf_nd_batched": (_I, [_I, _I, _Dmat, _LL, _Dmat, _LL, _Dmat, _LL, _Dmat, _LL, _P,
                                      _I, _P, _R]),
    "pb_chain_vbatched": (_I, [_CH, _P, _P, _P, _P, _P, _P, _I, _I, _P, _R]),
    "pb_dtrmm": (_I, [_CH, _CH, _CH, _CH, _I, _I, _D, _P, _I, _P, _I, _R]),
    "pb_dtrmm_batched": (_I, [_CH, _CH, _CH, _CH, _I, _I, _D, _P, _I, _LL, _P, _I, _LL, _I, _P, _R]),
    "pb_trmm_rlnn_nd": (_I, [_I, _I, _D, _Dmat, _Dmat, _Dmat, _R]),
    "pb_trmm_rlnn_nd_batched": (_I, [_I, _I, _D, _Dmat, _LL, _Dmat, _LL, _Dmat, _LL, _I, _P, _R]),
    "pb_memsize": (_LL, [_I, _I, _I]),
    "pb_pack": (_I, [_CH, _P, _I, _Dmat, _R]),
    "pb_pack_batched": (_I, [_CH, _P, _I, _LL, _Dmat, _LL, _I, _P, _R]),
    "pb_unpack": (_I, [_Dmat, _P, _I, _R]),
    "pb_unpack_batched": (_I, [_Dmat, _LL, _P, _I, _LL, _I, _P, _R]),
    "pb_riccati_nd_batched": (_I, [_I, _I, _I, _Dmat, _LL, _Dmat, _LL, _Dmat, _LL, _Dmat, _LL, _Dmat,
                                   _LL, _P, _P, _I, _P, _R]),
}

#: every symbol include/pbgpu.h declares (checked by tests/test_abi.py)
EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Loads libpbgpu.so (raises when it has not been built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise ImportError(f"{library_path} is missing: run `python -m paper_1902_08115_b200.build` "
                              "(pbgpu has no CPU fallback)")
        L = C.CDLL(library_path)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


# ----------------------------------------------------------------- result types
class ArgError(ValueError):
    """Raised in abort_on_error mode (mat_view.hpp:60-68): index is 1-based."""

    def __init__(self, index: int, message: str):
        super().__init__(message)
        self.index = index


@dataclass
class BlasCallError:
    routine: str
    index: int
    message: str


@dataclass
class BlasResult:
    """blas.hpp:32-40 (variant/stats have no GPU meaning and are omitted)."""

    info: int = 0
    error: Optional[BlasCallError] = None
    flops: int = 0
    message: Optional[str] = None

    def ok(self) -> bool:
        return self.info == 0


@dataclass
class BlasConfig:
    """blas.hpp:21-25: abort_on_error mimics xerbla by raising ArgError."""

    abort_on_error: bool = False


_DEFAULT = BlasConfig()


def _result(cfg: BlasConfig, r: _Result) -> BlasResult:
    out = BlasResult(info=r.info, flops=r.flops,
                     message=r.message.decode() if r.message else None)
    if r.error_index:
        out.error = BlasCallError(r.routine.decode() if r.routine else "", r.error_index,
                                  r.message.decode() if r.message else "")
        if cfg.abort_on_error:
            raise ArgError(r.error_index, f"{out.error.routine}: {out.error.message}")
    if r.info in (INFO_CUDA_ERROR, INFO_NO_DEVICE):
        raise RuntimeError(f"pbgpu: {out.message}")
    return out


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):  # torch tensor
        return x.data_ptr()
    if hasattr(x, "ctypes"):  # numpy array
        return x.ctypes.data
    raise TypeError(f"unsupported array type {type(x)!r}")


def _ch(c: str) -> bytes:
    return c.encode() if isinstance(c, str) else bytes(c)


def _stream(stream) -> Optional[int]:
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


# ------------------------------------------------------------------ panel refs
def _round_up(v: int, q: int) -> int:
    return (v + q - 1) // q * q


@dataclass
class PanelRef:
    """panel_mat.hpp:51-81: {data, ps, m, n, pm, cn}; element (i, j) at
    (i/ps)*ps*cn + j*ps + i%ps.  ``data`` is an array or address."""

    data: object
    m: int
    n: int
    ps: int = 4
    pm: Optional[int] = None
    cn: Optional[int] = None

    def c(self) -> _Dmat:
        pm = self.pm if self.pm is not None else _round_up(self.m, self.ps)
        cn = self.cn if self.cn is not None else _round_up(self.n, self.ps)
        return _Dmat(_ptr(self.data), self.ps, self.m, self.n, pm, cn)


# ------------------------------------------------------------- netlib adapters
def dgemm(transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_dgemm(_ch(transa), _ch(transb), m, n, k, alpha, _ptr(a), lda, _ptr(b), ldb, beta,
                   _ptr(c), ldc, C.byref(r))
    return _result(cfg, r)


def dsyrk(uplo, trans, n, k, alpha, a, lda, beta, c, ldc, cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_dsyrk(_ch(uplo), _ch(trans), n, k, alpha, _ptr(a), lda, beta, _ptr(c), ldc, C.byref(r))
    return _result(cfg, r)


def dtrsm(side, uplo, transa, diag, m, n, alpha, a, lda, b, ldb, cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_dtrsm(_ch(side), _ch(uplo), _ch(transa), _ch(diag), m, n, alpha, _ptr(a), lda, _ptr(b),
                   ldb, C.byref(r))
    return _result(cfg, r)


def dpotrf(uplo, n, a, lda, cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_dpotrf(_ch(uplo), n, _ptr(a), lda, C.byref(r))
    return _result(cfg, r)


def dgetrf(m, n, a, lda, ipiv, cfg: BlasConfig = _DEFAULT):
    """ipiv: int32 array of min(m, n) entries (1-based pivots on return)."""
    r = _Result()
    lib().pb_dgetrf(m, n, _ptr(a), lda, _ptr(ipiv), C.byref(r))
    return _result(cfg, r)


# ------------------------------------------------------------- panel natives
def gemm_nd(transa, transb, m, n, k, alpha, a: PanelRef, b: PanelRef, beta, c: PanelRef, d: PanelRef):
    r = _Result()
    lib().pb_gemm_nd(_ch(transa), _ch(transb), m, n, k, alpha, a.c(), b.c(), beta, c.c(), d.c(),
                     C.byref(r))
    return _result(_DEFAULT, r)


def syrk_nd(n, k, alpha, a: PanelRef, beta, c: PanelRef, d: PanelRef):
    r = _Result()
    lib().pb_syrk_nd(n, k, alpha, a.c(), beta, c.c(), d.c(), C.byref(r))
    return _result(_DEFAULT, r)


def trsm_rltn_nd(m, n, alpha, a: PanelRef, b: PanelRef, d: PanelRef):
    r = _Result()
    lib().pb_trsm_rltn_nd(m, n, alpha, a.c(), b.c(), d.c(), C.byref(r))
    return _result(_DEFAULT, r)


def syrk_potrf_nd(n, k, a: PanelRef, b: PanelRef, c: PanelRef, d: PanelRef):
    r = _Result()
    lib().pb_syrk_potrf_nd(n, k, a.c(), b.c(), c.c(), d.c(), C.byref(r))
    return _result(_DEFAULT, r)


# ------------------------------------------------------------------- batched
def dgemm_batched(transa, transb, m, n, k, alpha, a, lda, stride_a, b, ldb, stride_b, beta, c, ldc,
                  stride_c, batch, stream=None, cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_dgemm_batched(_ch(transa), _ch(transb), m, n, k, alpha, _ptr(a), lda, stride_a, _ptr(b),
                           ldb, stride_b, beta, _ptr(c), ldc, stride_c, batch, _stream(stream),
                           C.byref(r))
    return _result(cfg, r)


def dsyrk_batched(uplo, trans, n, k, alpha, a, lda, stride_a, beta, c, ldc, stride_c, batch,
                  stream=None, cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_dsyrk_batched(_ch(uplo), _ch(trans), n, k, alpha, _ptr(a), lda, stride_a, beta, _ptr(c),
                           ldc, stride_c, batch, _stream(stream), C.byref(r))
    return _result(cfg, r)


def dtrsm_batched(side, uplo, transa, diag, m, n, alpha, a, lda, stride_a, b, ldb, stride_b, info,
                  batch, stream=None, cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_dtrsm_batched(_ch(side), _ch(uplo), _ch(transa), _ch(diag), m, n, alpha, _ptr(a), lda,
                           stride_a, _ptr(b), ldb, stride_b, _ptr(info), batch, _stream(stream),
                           C.byref(r))
    return _result(cfg, r)


def dpotrf_batched(uplo, n, a, lda, stride_a, info, batch, stream=None, cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_dpotrf_batched(_ch(uplo), n, _ptr(a), lda, stride_a, _ptr(info), batch, _stream(stream),
                            C.byref(r))
    return _result(cfg, r)


def dgetrf_batched(m, n, a, lda, stride_a, ipiv, stride_ipiv, info, batch, stream=None,
                   cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_dgetrf_batched(m, n, _ptr(a), lda, stride_a, _ptr(ipiv), stride_ipiv, _ptr(info), batch,
                            _stream(stream), C.byref(r))
    return _result(cfg, r)


def gemm_nd_batched(transa, transb, m, n, k, alpha, a: PanelRef, stride_a, b: PanelRef, stride_b,
                    beta, c: PanelRef, stride_c, d: PanelRef, stride_d, batch, stream=None):
    r = _Result()
    lib().pb_gemm_nd_batched(_ch(transa), _ch(transb), m, n, k, alpha, a.c(), stride_a, b.c(),
                             stride_b, beta, c.c(), stride_c, d.c(), stride_d, batch,
                             _stream(stream), C.byref(r))
    return _result(_DEFAULT, r)


def syrk_nd_batched(n, k, alpha, a: PanelRef, stride_a, beta, c: PanelRef, stride_c, d: PanelRef,
                    stride_d, batch, stream=None):
    r = _Result()
    lib().pb_syrk_nd_batched(n, k, alpha, a.c(), stride_a, beta, c.c(), stride_c, d.c(), stride_d,
                             batch, _stream(stream), C.byref(r))
    return _result(_DEFAULT, r)


def trsm_rltn_nd_batched(m, n, alpha, a: PanelRef, stride_a, b: PanelRef, stride_b, d: PanelRef,
                         stride_d, info, batch, stream=None):
    r = _Result()
    lib().pb_trsm_rltn_nd_batched(m, n, alpha, a.c(), stride_a, b.c(), stride_b, d.c(), stride_d,
                                  _ptr(info), batch, _stream(stream), C.byref(r))
    return _result(_DEFAULT, r)


def syrk_potrf_nd_batched(n, k, a: PanelRef, stride_a, b: PanelRef, stride_b, c: PanelRef, stride_c,
                          d: PanelRef, stride_d, info, batch, stream=None):
    r = _Result()
    lib().pb_syrk_potrf_nd_batched(n, k, a.c(), stride_a, b.c(), stride_b, c.c(), stride_c, d.c(),
                                   stride_d, _ptr(info), batch, _stream(stream), C.byref(r))
    return _result(_DEFAULT, r)


def chain_vbatched(layout, n, offset, A, C_, B, info, batch, max_n, stream=None):
    r = _Result()
    lib().pb_chain_vbatched(_ch(layout), _ptr(n), _ptr(offset), _ptr(A), _ptr(C_), _ptr(B), _ptr(info),
                            batch, max_n, _stream(stream), C.byref(r))
    return _result(_DEFAULT, r)


# ------------------------------------------------------- dtrmm / trmm_rlnn_nd
def dtrmm(side, uplo, transa, diag, m, n, alpha, a, lda, b, ldb, cfg: BlasConfig = _DEFAULT):
    """blas.hpp:166-176: B <- alpha op(A) B (side 'l') or alpha B op(A) (side 'r')."""
    r = _Result()
    lib().pb_dtrmm(_ch(side), _ch(uplo), _ch(transa), _ch(diag), m, n, alpha, _ptr(a), lda, _ptr(b),
                   ldb, C.byref(r))
    return _result(cfg, r)


def dtrmm_batched(side, uplo, transa, diag, m, n, alpha, a, lda, stride_a, b, ldb, stride_b, batch,
                  stream=None, cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_dtrmm_batched(_ch(side), _ch(uplo), _ch(transa), _ch(diag), m, n, alpha, _ptr(a), lda,
                           stride_a, _ptr(b), ldb, stride_b, batch, _stream(stream), C.byref(r))
    return _result(cfg, r)


def trmm_rlnn_nd(m, n, alpha, a: PanelRef, b: PanelRef, d: PanelRef):
    """level3.hpp:446-479: d <- alpha b a, a lower non-unit."""
    r = _Result()
    lib().pb_trmm_rlnn_nd(m, n, alpha, a.c(), b.c(), d.c(), C.byref(r))
    return _result(_DEFAULT, r)


def trmm_rlnn_nd_batched(m, n, alpha, a: PanelRef, stride_a, b: PanelRef, stride_b, d: PanelRef,
                         stride_d, batch, stream=None):
    r = _Result()
    lib().pb_trmm_rlnn_nd_batched(m, n, alpha, a.c(), stride_a, b.c(), stride_b, d.c(), stride_d,
                                  batch, _stream(stream), C.byref(r))
    return _result(_DEFAULT, r)


# ------------------------------------------------------------- pack / unpack
def memsize(m, n, ps=4) -> int:
    """panel_mat.hpp:45-48."""
    return int(lib().pb_memsize(m, n, ps))


def pack(trans, a, lda, d: PanelRef, cfg: BlasConfig = _DEFAULT):
    """panel_mat.hpp:141-160: d <- packed op(a); pad lanes untouched."""
    r = _Result()
    lib().pb_pack(_ch(trans), _ptr(a), lda, d.c(), C.byref(r))
    return _result(cfg, r)


def pack_batched(trans, a, lda, stride_a, d: PanelRef, stride_d, batch, stream=None,
                 cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_pack_batched(_ch(trans), _ptr(a), lda, stride_a, d.c(), stride_d, batch, _stream(stream),
                          C.byref(r))
    return _result(cfg, r)


def unpack(s: PanelRef, a, lda, cfg: BlasConfig = _DEFAULT):
    """panel_mat.hpp:164-171: a <- unpacked s."""
    r = _Result()
    lib().pb_unpack(s.c(), _ptr(a), lda, C.byref(r))
    return _result(cfg, r)


def unpack_batched(s: PanelRef, stride_s, a, lda, stride_a, batch, stream=None,
                   cfg: BlasConfig = _DEFAULT):
    r = _Result()
    lib().pb_unpack_batched(s.c(), stride_s, _ptr(a), lda, stride_a, batch, _stream(stream), C.byref(r))
    return _result(cfg, r)


# ------------------------------------------------------------------ Riccati
def riccati_nd_batched(nx, nu, N, m0: PanelRef, stride_m0, q: PanelRef, stride_q, g: PanelRef,
                       stride_g, f: PanelRef, stride_f, lterm: Optional[PanelRef], stride_lterm,
                       info, stage, batch, stream=None):
    """Batched RiccatiFusedWork stage loop (riccati.hpp:257-373, 402-512); see include/pbgpu.h."""
    r = _Result()
    lt = lterm.c() if lterm is not None else _Dmat(None, 4, nx, nx, _round_up(nx, 4), _round_up(nx, 4))
    lib().pb_riccati_nd_batched(nx, nu, N, m0.c(), stride_m0, q.c(), stride_q, g.c(), stride_g, f.c(),
                                stride_f, lt, stride_lterm, _ptr(info), _ptr(stage), batch,
                                _stream(stream), C.byref(r))
    return _result(_DEFAULT, r)
