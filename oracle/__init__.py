"""CPU oracle for the ABFT DGEMM hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2305_02444_b200`` never imports it; the two share no code (the only
common module is ``synthetic``, which holds no arithmetic of the method).

The arithmetic lives in plain C (``ftblas_oracle.c``, binary64, ascending
sums, no FMA contraction); this file only marshals numpy arrays through
ctypes.  Each function cites the PAPER.md passage it follows in the C source.
Parity status: all functions pinned (tests/test_oracle_pins.py); none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ftblas_oracle.c")
_LIB = os.path.join(_HERE, "libftblas_oracle.so")

CFLAGS = ["-O2", "-fPIC", "-shared", "-std=c11", "-ffp-contract=off", "-fno-fast-math"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (``build()`` of __graft_entry__ calls this)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


class Correction(ct.Structure):
    _fields_ = [("tile_m", ct.c_int64), ("tile_n", ct.c_int64), ("i", ct.c_int64),
                ("j", ct.c_int64), ("residual", ct.c_double), ("kind", ct.c_int32),
                ("pad", ct.c_int32)]


class Stats(ct.Structure):
    _fields_ = [("count", ct.c_int64), ("tiles_flagged", ct.c_int64),
                ("rows_flagged", ct.c_int64), ("cols_flagged", ct.c_int64)]


_lib = None
_P = ct.POINTER(ct.c_double)
_I64 = ct.c_int64


def lib():
    global _lib
    if _lib is None:
        _lib = ct.CDLL(build())
        L = _lib
        L.ora_dot.restype = ct.c_double
        L.ora_dot.argtypes = [ct.c_int, ct.c_int, _I64, _P, _I64, _P, _I64, _I64, _I64]
        L.ora_absdot.restype = ct.c_double
        L.ora_absdot.argtypes = L.ora_dot.argtypes
        L.ora_dgemm.restype = None
        L.ora_dgemm.argtypes = [ct.c_int, ct.c_int, _I64, _I64, _I64, ct.c_double, _P, _I64, _P,
                                _I64, ct.c_double, _P, _I64, _I64, _I64, _I64, _I64]
        L.ora_flip.restype = ct.c_double
        L.ora_flip.argtypes = [ct.c_double, ct.c_int]
        L.ora_encode_a.restype = None
        L.ora_encode_a.argtypes = [ct.c_int, _I64, _P, _I64, _I64, _I64, _P, _P, _P]
        L.ora_encode_b.restype = None
        L.ora_encode_b.argtypes = [ct.c_int, _I64, _P, _I64, _I64, _I64, _P, _P, _P]
        L.ora_ref_checksums.restype = None
        L.ora_ref_checksums.argtypes = [ct.c_int, ct.c_int, _I64, ct.c_double, _P, _I64, _P, _I64,
                                        ct.c_double, _P, _I64, _I64, _I64, _I64, _I64, _P, _P,
                                        _P, _P, _P, _P]
        L.ora_verify_tile.restype = _I64
        L.ora_verify_tile.argtypes = [ct.c_int, ct.c_int, _I64, ct.c_double, _P, _I64, _P, _I64,
                                      ct.c_double, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64,
                                      _P, _I64, ct.POINTER(Correction), _I64, _I64,
                                      ct.POINTER(Stats)]
        L.ora_abft_dgemm.restype = _I64
        L.ora_abft_dgemm.argtypes = [ct.c_int, ct.c_int, _I64, _I64, _I64, ct.c_double, _P, _I64,
                                     _P, _I64, ct.c_double, _P, _I64, _I64, _I64, _I64,
                                     ct.POINTER(ct.c_int64), ct.POINTER(ct.c_int64),
                                     ct.POINTER(ct.c_int32), ct.POINTER(Correction), _I64,
                                     ct.POINTER(Stats), ct.POINTER(ct.c_uint8)]
    return _lib


def _buf(x: np.ndarray):
    """Pointer to the first element of a column-major array or padded view thereof."""
    assert x.dtype == np.float64
    assert x.flags.f_contiguous or (x.ndim == 2 and x.strides[0] == 8), "column-major expected"
    return x.ctypes.data_as(_P)


def _t(trans: str) -> int:
    t = trans.upper()
    if t not in ("N", "T", "C"):
        raise ValueError(trans)
    return 0 if t == "N" else 1


def ld_of(x: np.ndarray) -> int:
    return max(1, x.strides[1] // 8) if x.ndim == 2 and x.shape[1] > 1 else max(1, x.shape[0])


def dgemm(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, rows=None, cols=None):
    """C := alpha op(A) op(B) + beta C in place (optionally only rows/cols sub-block)."""
    i0, i1 = rows if rows else (0, M)
    j0, j1 = cols if cols else (0, N)
    lib().ora_dgemm(_t(transA), _t(transB), M, N, K, alpha, _buf(A), lda, _buf(B), ldb, beta,
                    _buf(C), ldc, i0, i1, j0, j1)
    return C


def dot(transA, transB, K, A, lda, B, ldb, i, j) -> float:
    return lib().ora_dot(_t(transA), _t(transB), K, _buf(A), lda, _buf(B), ldb, i, j)


def absdot(transA, transB, K, A, lda, B, ldb, i, j) -> float:
    return lib().ora_absdot(_t(transA), _t(transB), K, _buf(A), lda, _buf(B), ldb, i, j)


def flip(x: float, bit: int) -> float:
    return lib().ora_flip(x, bit)


def encode_a(transA, K, A, lda, i0, i1):
    ac = np.zeros(max(K, 1))
    mx = ct.c_double(0.0)
    rowabs = np.zeros(max(i1 - i0, 1))
    lib().ora_encode_a(_t(transA), K, _buf(A), lda, i0, i1, _buf(ac), ct.byref(mx), _buf(rowabs))
    return ac[:K], mx.value, rowabs[: i1 - i0]


def encode_b(transB, K, B, ldb, j0, j1):
    br = np.zeros(max(K, 1))
    mx = ct.c_double(0.0)
    colabs = np.zeros(max(j1 - j0, 1))
    lib().ora_encode_b(_t(transB), K, _buf(B), ldb, j0, j1, _buf(br), ct.byref(mx), _buf(colabs))
    return br[:K], mx.value, colabs[: j1 - j0]


def ref_checksums(transA, transB, K, alpha, A, lda, B, ldb, beta, C0, ldc, i0, i1, j0, j1, ac, br):
    m, n = i1 - i0, j1 - j0
    crow, ccol, c0row, c0col = (np.zeros(max(m, 1)), np.zeros(max(n, 1)),
                                np.zeros(max(m, 1)), np.zeros(max(n, 1)))
    ac = np.ascontiguousarray(ac if len(ac) else np.zeros(1))
    br = np.ascontiguousarray(br if len(br) else np.zeros(1))
    lib().ora_ref_checksums(_t(transA), _t(transB), K, alpha, _buf(A), lda, _buf(B), ldb, beta,
                            _buf(C0), ldc, i0, i1, j0, j1, _buf(ac), _buf(br), _buf(crow),
                            _buf(ccol), _buf(c0row), _buf(c0col))
    return crow[:m], ccol[:n], c0row[:m], c0col[:n]


def verify_tile(transA, transB, K, alpha, A, lda, B, ldb, beta, C0, ldc, i0, i1, j0, j1,
                tile_m, tile_n, Ct, cap=64):
    """Verify/locate/correct one computed tile Ct (m x n, col-major, corrected in place)."""
    rep = (Correction * max(cap, 1))()
    st = Stats()
    n = lib().ora_verify_tile(_t(transA), _t(transB), K, alpha, _buf(A), lda, _buf(B), ldb, beta,
                              _buf(C0), ldc, i0, i1, j0, j1, tile_m, tile_n, _buf(Ct),
                              Ct.shape[0], rep, cap, 0, ct.byref(st))
    return [_corr_tuple(rep[q]) for q in range(min(n, cap))], st


def _corr_tuple(c: Correction):
    return dict(tile_m=c.tile_m, tile_n=c.tile_n, i=c.i, j=c.j, residual=c.residual, kind=c.kind)


def abft_dgemm(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, *, tile_m=128,
               tile_n=128, faults=None, cap=None, tiles_only=None):
    """The whole hot path on CPU: returns (corrections list, stats); C corrected in place."""
    if faults is None:
        fi = np.zeros(0, np.int64); fj = np.zeros(0, np.int64); fb = np.zeros(0, np.int32)
    else:
        fi, fj, fb = (np.ascontiguousarray(faults[0], np.int64),
                      np.ascontiguousarray(faults[1], np.int64),
                      np.ascontiguousarray(faults[2], np.int32))
    cap = cap if cap is not None else max(16, 4 * len(fi))
    rep = (Correction * max(cap, 1))()
    st = Stats()
    to = None
    if tiles_only is not None:
        tiles_only = np.ascontiguousarray(tiles_only, dtype=np.uint8)
        to = tiles_only.ctypes.data_as(ct.POINTER(ct.c_uint8))
    lib().ora_abft_dgemm(_t(transA), _t(transB), M, N, K, alpha, _buf(A), lda, _buf(B), ldb, beta,
                         _buf(C), ldc, tile_m, tile_n, len(fi),
                         fi.ctypes.data_as(ct.POINTER(ct.c_int64)),
                         fj.ctypes.data_as(ct.POINTER(ct.c_int64)),
                         fb.ctypes.data_as(ct.POINTER(ct.c_int32)), rep, cap, ct.byref(st), to)
    return [_corr_tuple(rep[q]) for q in range(min(st.count, cap))], st
