"""Thin ctypes binding of libftblas.so (include/ftblas.h).  Argument marshalling only.

Every step of the hot path runs in the CUDA kernels of the shared library; this
module converts Python values / torch tensors to the C ABI and back.  There is
no CPU fallback: if the library cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as ct
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libftblas.so")

TILE_M = 128
TILE_N = 128
ERR_CUDA = 1000


class ftblas_correction(ct.Structure):
    _fields_ = [("tile_m", ct.c_int64), ("tile_n", ct.c_int64), ("i", ct.c_int64),
                ("j", ct.c_int64), ("residual", ct.c_double), ("kind", ct.c_int32),
                ("pad", ct.c_int32)]


class ftblas_err_report(ct.Structure):
    _fields_ = [("entries", ct.POINTER(ftblas_correction)), ("capacity", ct.c_int64),
                ("count", ct.c_int64), ("tiles_flagged", ct.c_int64),
                ("rows_flagged", ct.c_int64), ("cols_flagged", ct.c_int64)]


class FtblasError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libftblas.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = ct.CDLL(LIB_PATH)
    P = ct.c_void_p
    I = ct.c_int64
    D = ct.c_double
    common = [ct.c_char, ct.c_char, I, I, I, D, P, I, P, I, D, P, I]
    L.ftblas_dgemm.argtypes = common + [ct.POINTER(ftblas_err_report)]
    L.ftblas_dgemm.restype = ct.c_int
    L.ftblas_dgemm_noft.argtypes = common
    L.ftblas_dgemm_noft.restype = ct.c_int
    L.ftblas_dgemm_host.argtypes = common + [ct.POINTER(ftblas_err_report)]
    L.ftblas_dgemm_host.restype = ct.c_int
    L.ftblas_report_fetch.argtypes = [ct.POINTER(ftblas_err_report)]
    L.ftblas_report_fetch.restype = ct.c_int
    L.ftblas_set_fault_plan.argtypes = [I, P, P, P]
    L.ftblas_set_fault_plan.restype = ct.c_int
    L.ftblas_set_stream.argtypes = [P]
    L.ftblas_set_stream.restype = ct.c_int
    L.ftblas_launch_count.argtypes = []
    L.ftblas_launch_count.restype = I
    L.ftblas_profile.argtypes = [ct.c_int]
    L.ftblas_profile.restype = ct.c_int
    L.ftblas_profile_read.argtypes = [ct.POINTER(ct.c_double), ct.POINTER(ct.c_double),
                                      ct.POINTER(ct.c_int64)]
    L.ftblas_profile_read.restype = ct.c_int
    L.ftblas_tile_shape.argtypes = [ct.POINTER(ct.c_int32), ct.POINTER(ct.c_int32)]
    L.ftblas_tile_shape.restype = None
    L.ftblas_last_error.argtypes = []
    L.ftblas_last_error.restype = ct.c_char_p
    L.ftblas_release.argtypes = []
    L.ftblas_release.restype = ct.c_int
    L.ftblas_dgemm_ex.argtypes = common + [I, I, ct.c_int32, ct.POINTER(ftblas_err_report)]
    L.ftblas_dgemm_ex.restype = ct.c_int
    L.ftblas_report_reset.argtypes = []
    L.ftblas_report_reset.restype = ct.c_int
    L.ftblas_set_tile_policy.argtypes = [ct.c_int]
    L.ftblas_set_tile_policy.restype = ct.c_int
    L.ftblas_get_tile_policy.argtypes = []
    L.ftblas_get_tile_policy.restype = ct.c_int
    L.ftblas_set_checksum_mode.argtypes = [ct.c_int]
    L.ftblas_set_checksum_mode.restype = ct.c_int
    L.ftblas_get_checksum_mode.argtypes = []
    L.ftblas_get_checksum_mode.restype = ct.c_int
    L.ftblas_b_encoding_len.argtypes = [I, I]
    L.ftblas_b_encoding_len.restype = I
    L.ftblas_b_encoding_layout.argtypes = [I, I, ct.POINTER(I), ct.POINTER(I), ct.POINTER(I)]
    L.ftblas_b_encoding_layout.restype = ct.c_int
    L.ftblas_encode_b.argtypes = [ct.c_char, I, I, P, I, P]
    L.ftblas_encode_b.restype = ct.c_int
    L.ftblas_set_b_encoding.argtypes = [P, I, I]
    L.ftblas_set_b_encoding.restype = ct.c_int
    return L


lib = _load()

# Symbols include/ftblas.h declares (checked by tests/test_abi.py).
EXPORTS = ("ftblas_dgemm", "ftblas_dgemm_noft", "ftblas_dgemm_host", "ftblas_report_fetch",
           "ftblas_set_fault_plan", "ftblas_set_stream", "ftblas_launch_count",
           "ftblas_tile_shape", "ftblas_last_error", "ftblas_release", "ftblas_profile",
           "ftblas_profile_read", "ftblas_set_checksum_mode", "ftblas_get_checksum_mode",
           "ftblas_dgemm_ex", "ftblas_report_reset", "ftblas_set_tile_policy",
           "ftblas_get_tile_policy", "ftblas_b_encoding_len", "ftblas_b_encoding_layout",
           "ftblas_encode_b", "ftblas_set_b_encoding")

TILES = {"auto": 0, "full": 1, "pair": 2, "ws": 3}  # FTBLAS_TILES_*

REPORT_APPEND = 1  # FTBLAS_REPORT_APPEND
REUSE_A_ENCODE = 2  # FTBLAS_REUSE_A_ENCODE
B_ENCODED = 4  # FTBLAS_B_ENCODED

CHECKSUM_GEMM = 0   # FTBLAS_CHECKSUM_GEMM: checksum row/column by two DMMA GEMMs (default)
CHECKSUM_FUSED = 1  # FTBLAS_CHECKSUM_FUSED: accumulated in the main GEMM's mainloop
CHECKSUM_MODES = {"gemm": CHECKSUM_GEMM, "fused": CHECKSUM_FUSED}


def _ptr(x):
    """Device/host pointer of a torch tensor, numpy array, int or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):      # torch.Tensor
        return x.data_ptr()
    if hasattr(x, "ctypes"):        # numpy.ndarray
        return x.ctypes.data
    raise TypeError(type(x))


def _check(rc: int):
    if rc != 0:
        raise FtblasError(f"ftblas error {rc}: {lib.ftblas_last_error().decode()}")


class Report:
    """Host-side report: list of corrections (dicts) plus counters."""

    def __init__(self, capacity: int = 4096):
        self._buf = (ftblas_correction * max(1, capacity))()
        self.c = ftblas_err_report(ct.cast(self._buf, ct.POINTER(ftblas_correction)), capacity,
                                   0, 0, 0, 0)

    @property
    def count(self):
        return self.c.count

    @property
    def tiles_flagged(self):
        return self.c.tiles_flagged

    @property
    def rows_flagged(self):
        return self.c.rows_flagged

    @property
    def cols_flagged(self):
        return self.c.cols_flagged

    def entries(self):
        n = min(self.c.count, self.c.capacity)
        return [dict(tile_m=self._buf[q].tile_m, tile_n=self._buf[q].tile_n, i=self._buf[q].i,
                     j=self._buf[q].j, residual=self._buf[q].residual, kind=self._buf[q].kind)
                for q in range(n)]


def _tc(t: str) -> bytes:
    return t.encode() if isinstance(t, str) else t


def ftblas_dgemm(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, report=None):
    rep = ct.byref(report.c) if report is not None else None
    _check(lib.ftblas_dgemm(_tc(transA), _tc(transB), M, N, K, alpha, _ptr(A), lda, _ptr(B), ldb,
                            beta, _ptr(C), ldc, rep))
    return report


def ftblas_dgemm_ex(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, row_offset=0,
                    col_offset=0, append=False, report=None, reuse_a=False, b_encoded=False):
    rep = ct.byref(report.c) if report is not None else None
    flags = (REPORT_APPEND if append else 0) | (REUSE_A_ENCODE if reuse_a else 0) | \
        (B_ENCODED if b_encoded else 0)
    _check(lib.ftblas_dgemm_ex(_tc(transA), _tc(transB), M, N, K, alpha, _ptr(A), lda, _ptr(B), ldb,
                               beta, _ptr(C), ldc, row_offset, col_offset, flags, rep))
    return report


def ftblas_b_encoding_layout(N, K):
    """(off_nrm, off_max, total) in doubles of the op(B) encoding layout (include/ftblas.h)."""
    a, b, t = ct.c_int64(), ct.c_int64(), ct.c_int64()
    _check(lib.ftblas_b_encoding_layout(N, K, ct.byref(a), ct.byref(b), ct.byref(t)))
    return a.value, b.value, t.value


def ftblas_b_encoding_len(N, K) -> int:
    return lib.ftblas_b_encoding_len(N, K)


def ftblas_encode_b(transB, N, K, B, ldb, enc):
    _check(lib.ftblas_encode_b(_tc(transB), N, K, _ptr(B), ldb, _ptr(enc)))


def ftblas_set_b_encoding(enc, N=0, K=0):
    _check(lib.ftblas_set_b_encoding(_ptr(enc), N, K))


def ftblas_report_reset():
    _check(lib.ftblas_report_reset())


def ftblas_dgemm_noft(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc):
    _check(lib.ftblas_dgemm_noft(_tc(transA), _tc(transB), M, N, K, alpha, _ptr(A), lda, _ptr(B),
                                 ldb, beta, _ptr(C), ldc))


def ftblas_dgemm_host(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, report=None):
    rep = ct.byref(report.c) if report is not None else None
    _check(lib.ftblas_dgemm_host(_tc(transA), _tc(transB), M, N, K, alpha, _ptr(A), lda, _ptr(B),
                                 ldb, beta, _ptr(C), ldc, rep))
    return report


def ftblas_report_fetch(report):
    _check(lib.ftblas_report_fetch(ct.byref(report.c)))
    return report


def ftblas_set_fault_plan(i, j, bit):
    """i, j: int64 numpy arrays; bit: int32 numpy array (copied by the library)."""
    import numpy as np
    i = np.ascontiguousarray(i, dtype=np.int64)
    j = np.ascontiguousarray(j, dtype=np.int64)
    bit = np.ascontiguousarray(bit, dtype=np.int32)
    _check(lib.ftblas_set_fault_plan(len(i), i.ctypes.data, j.ctypes.data, bit.ctypes.data))


def ftblas_clear_fault_plan():
    _check(lib.ftblas_set_fault_plan(0, None, None, None))


def ftblas_set_checksum_mode(mode):
    """mode: CHECKSUM_GEMM / CHECKSUM_FUSED or the names 'gemm' / 'fused'."""
    _check(lib.ftblas_set_checksum_mode(CHECKSUM_MODES.get(mode, mode)))


def ftblas_set_tile_policy(policy):
    """policy: 'auto' | 'full' | 'pair' | 'ws' or the FTBLAS_TILES_* value."""
    _check(lib.ftblas_set_tile_policy(TILES.get(policy, policy)))


def ftblas_get_tile_policy() -> int:
    return lib.ftblas_get_tile_policy()


def ftblas_get_checksum_mode() -> int:
    return lib.ftblas_get_checksum_mode()


def ftblas_set_stream(stream):
    """stream: torch.cuda.Stream, raw cudaStream_t int, or None (default stream)."""
    h = getattr(stream, "cuda_stream", stream)
    _check(lib.ftblas_set_stream(h))


def ftblas_launch_count() -> int:
    return lib.ftblas_launch_count()


def ftblas_profile(enable: bool):
    _check(lib.ftblas_profile(1 if enable else 0))


def ftblas_profile_read():
    """(encode_ms, gemm_ms, gemm_launches) recorded since the last read."""
    a, b, n = ct.c_double(), ct.c_double(), ct.c_int64()
    _check(lib.ftblas_profile_read(ct.byref(a), ct.byref(b), ct.byref(n)))
    return a.value, b.value, n.value


def ftblas_tile_shape():
    a, b = ct.c_int32(), ct.c_int32()
    lib.ftblas_tile_shape(ct.byref(a), ct.byref(b))
    return a.value, b.value


def ftblas_release():
    _check(lib.ftblas_release())
