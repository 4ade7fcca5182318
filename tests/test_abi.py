"""CPU-side checks of the boundary: the library builds/loads and exports every symbol
include/ftblas.h declares; argument errors follow the header (no GPU compute calls)."""
import ctypes as ct
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ftblas.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ftblas_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2305_02444_b200 import build
    build.build()
    from paper_2305_02444_b200 import ftblas
    return ftblas


def test_header_declares_expected_api():
    names = declared_functions()
    for n in ["ftblas_dgemm", "ftblas_dgemm_noft", "ftblas_dgemm_host", "ftblas_set_fault_plan",
              "ftblas_report_fetch", "ftblas_set_stream"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    L = ct.CDLL(lib.LIB_PATH)
    for n in declared_functions():
        assert hasattr(L, n), n
    assert set(lib.EXPORTS) == set(declared_functions())


def test_struct_abi_sizes(lib):
    assert ct.sizeof(lib.ftblas_correction) == 48
    assert ct.sizeof(lib.ftblas_err_report) == 48


def test_tile_shape(lib):
    assert lib.ftblas_tile_shape() == (lib.TILE_M, lib.TILE_N) == (128, 128)


@pytest.mark.parametrize("args,code", [
    (("X", "N", 4, 4, 4, 1.0, 8, 4, 8, 4, 0.0, 8, 4), -1),
    (("N", "Q", 4, 4, 4, 1.0, 8, 4, 8, 4, 0.0, 8, 4), -2),
    (("N", "N", -1, 4, 4, 1.0, 8, 4, 8, 4, 0.0, 8, 4), -3),
    (("N", "N", 4, -1, 4, 1.0, 8, 4, 8, 4, 0.0, 8, 4), -4),
    (("N", "N", 4, 4, -1, 1.0, 8, 4, 8, 4, 0.0, 8, 4), -5),
    (("N", "N", 4, 4, 4, 1.0, 8, 3, 8, 4, 0.0, 8, 4), -8),
    (("T", "N", 4, 4, 5, 1.0, 8, 4, 8, 5, 0.0, 8, 4), -8),
    (("N", "N", 4, 4, 4, 1.0, 8, 4, 8, 3, 0.0, 8, 4), -10),
    (("N", "T", 4, 5, 4, 1.0, 8, 4, 8, 4, 0.0, 8, 4), -10),
    (("N", "N", 4, 4, 4, 1.0, 8, 4, 8, 4, 0.0, 8, 3), -13),
    (("N", "N", 4, 4, 4, 1.0, 0, 4, 8, 4, 0.0, 8, 4), -7),
    (("N", "N", 4, 4, 4, 1.0, 8, 4, 0, 4, 0.0, 8, 4), -9),
    (("N", "N", 4, 4, 4, 1.0, 8, 4, 8, 4, 0.0, 0, 4), -12),
])
def test_argument_errors_launch_nothing(lib, args, code):
    """Invalid arguments return -p (BLAS xerbla numbering) before any CUDA call, so these
    run without a GPU; pointers are dummies never dereferenced."""
    ta, tb, M, N, K, al, A, lda, B, ldb, be, C, ldc = args
    A = A or None; B = B or None; C = C or None
    for fn in (lib.lib.ftblas_dgemm, lib.lib.ftblas_dgemm_noft):
        extra = (None,) if fn is lib.lib.ftblas_dgemm else ()
        rc = fn(ta.encode(), tb.encode(), M, N, K, al, A, lda, B, ldb, be, C, ldc, *extra)
        assert rc == code
    assert b"invalid argument" in lib.lib.ftblas_last_error()


def test_fault_plan_validation(lib):
    import numpy as np
    with pytest.raises(lib.FtblasError):
        lib.ftblas_set_fault_plan(np.array([1]), np.array([1]), np.array([64]))
    lib.ftblas_set_fault_plan(np.array([1, 2]), np.array([3, 4]), np.array([40, 62]))
    # at most FTBLAS_MAX_FLIPS_PER_TILE (4) flips per 128 x 128 tile; 4 in one tile is fine
    lib.ftblas_set_fault_plan(np.arange(4), np.arange(4), np.full(4, 50))
    with pytest.raises(lib.FtblasError):
        lib.ftblas_set_fault_plan(np.arange(5), np.arange(5), np.full(5, 50))
    with pytest.raises(lib.FtblasError):
        lib.ftblas_set_fault_plan(np.array([-1]), np.array([0]), np.array([50]))
    lib.ftblas_set_fault_plan(np.array([0, 130, 260, 390, 520]), np.zeros(5, np.int64), np.full(5, 50))
    lib.ftblas_clear_fault_plan()


def test_b_encoding_host_checks(lib):
    """FTBLAS_B_ENCODED needs a matching installed encoding (checked before any CUDA work); the
    layout of an N x K encoding: ceil(N/128) rows of Kp, then N norms, then the tile maxima."""
    import numpy as np
    with pytest.raises(lib.FtblasError):
        lib.ftblas_dgemm_ex("N", "N", 4, 4, 4, 1.0, 1, 4, 1, 4, 0.0, 1, 4, b_encoded=True)
    off_n, off_m, tot = lib.ftblas_b_encoding_layout(300, 90)
    assert (off_n, off_m, tot) == (3 * 96, 3 * 96 + 300, 3 * 96 + 300 + 4)
    assert lib.ftblas_b_encoding_len(300, 90) == tot and lib.ftblas_b_encoding_layout(128, 1)[0] == 32
    with pytest.raises(lib.FtblasError):
        lib.ftblas_encode_b("X", 4, 4, 1, 4, 1)
    lib.ftblas_set_b_encoding(None)


def test_product_has_no_oracle_or_cpu_fallback():
    """The product package never imports the oracle and has no CPU compute path."""
    pkg = os.path.join(ROOT, "paper_2305_02444_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in s and "from oracle" not in s, f
                assert "ftblas_oracle" not in s, f
                assert "numpy.matmul" not in s and "np.matmul" not in s and " @ " not in s, f


def test_checksum_mode_api(lib):
    """ftblas_set_checksum_mode accepts the two modes of the header and rejects others
    (host-side state only, no GPU)."""
    assert lib.ftblas_get_checksum_mode() == lib.CHECKSUM_GEMM  # default
    lib.ftblas_set_checksum_mode("fused")
    assert lib.ftblas_get_checksum_mode() == lib.CHECKSUM_FUSED
    with pytest.raises(lib.FtblasError):
        lib.ftblas_set_checksum_mode(7)
    assert lib.ftblas_get_checksum_mode() == lib.CHECKSUM_FUSED
    lib.ftblas_set_checksum_mode("gemm")
    assert lib.ftblas_get_checksum_mode() == lib.CHECKSUM_GEMM


@pytest.mark.parametrize("roff,coff,flags,code", [(64, 0, 0, -14), (-128, 0, 0, -14), (0, 5, 0, -15),
                                                  (0, 0, 4, -16)])
def test_ex_argument_errors(lib, roff, coff, flags, code):
    """ftblas_dgemm_ex rejects offsets that are not whole tiles and unknown flags before any
    CUDA call (so this runs without a GPU)."""
    rc = lib.lib.ftblas_dgemm_ex(b"N", b"N", 4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, roff, coff,
                                 flags, None)
    assert rc == code


def test_tile_policy_api(lib):
    """ftblas_set_tile_policy accepts the three policies of the header (host state only)."""
    assert lib.ftblas_get_tile_policy() == lib.TILES["auto"]
    for name in ("full", "pair", "auto"):
        lib.ftblas_set_tile_policy(name)
        assert lib.ftblas_get_tile_policy() == lib.TILES[name]
    with pytest.raises(lib.FtblasError):
        lib.ftblas_set_tile_policy(9)
    lib.ftblas_set_tile_policy("auto")
