"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  * error reports bit-exact: the same (tile, i, j) list (+ kind) and the same count;
  * corrected C within 4 (K+2) 2^-53 (|alpha| |A||B| + |beta| |C0|) elementwise.
Small cases compare every element; full-size configs compare the tiles the oracle can
compute (every faulty tile of configs[1], samples elsewhere) plus sampled elements.
"""
import numpy as np
import pytest

import oracle
import synthetic as syn
from tests._util import from_dev, gemm_bound, report_key, to_dev

pytestmark = pytest.mark.gpu


def _lib(mode, tiles="auto"):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_02444_b200 import ftblas
    ftblas.ftblas_set_stream(None)
    ftblas.ftblas_set_checksum_mode(mode)
    ftblas.ftblas_set_tile_policy(tiles)
    return ftblas


@pytest.fixture(params=[("gemm", "ws"), ("gemm", "pair"), ("gemm", "full"), ("fused", "full")],
                ids=["gemm-ws", "gemm-pair", "gemm-full", "fused-full"])
def ft(request):
    """The library in each checksum mode (checksum GEMMs / fused mainloop checksums) and CTA
    tiling (128 x 64 cluster-pair halves / 128 x 128 tiles)."""
    lib = _lib(*request.param)
    yield lib
    lib.ftblas_set_checksum_mode("gemm")
    lib.ftblas_set_tile_policy("auto")


@pytest.fixture
def ftd():
    """The library in its default checksum mode (full-size configs)."""
    return _lib("gemm")


def run_gpu(ft, w, d, *, plan=None, noft=False, offsets=(0, 0, 0)):
    A_t, pA = to_dev(d["A"], offsets[0])
    B_t, pB = to_dev(d["B"], offsets[1])
    C_t, pC = to_dev(d["C"], offsets[2])
    if plan is not None:
        ft.ftblas_set_fault_plan(*plan)
    else:
        ft.ftblas_clear_fault_plan()
    rep = ft.Report(8192)
    if noft:
        ft.ftblas_dgemm_noft(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"],
                             w.beta, pC, d["ldc"])
        import torch
        torch.cuda.synchronize()
        rep = None
    else:
        ft.ftblas_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"],
                        w.beta, pC, d["ldc"], rep)
    ft.ftblas_clear_fault_plan()
    return from_dev(C_t, d["C"], offsets[2]), rep


def run_oracle(w, d, plan=None, tiles_only=None):
    Cb = np.asfortranarray(syn.base_of(d["C"]).copy())
    Cv = Cb[: w.M, :]
    rep, st = oracle.abft_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, d["A"], d["lda"],
                                d["B"], d["ldb"], w.beta, Cv, d["ldc"], faults=plan,
                                cap=max(64, 4 * (0 if plan is None else len(plan[0]))),
                                tiles_only=tiles_only)
    return Cv, rep, st


def abs_product(w, d):
    opA = d["A"] if w.transA == "N" else d["A"].T
    opB = d["B"] if w.transB == "N" else d["B"].T
    return np.abs(opA) @ np.abs(opB)


def assert_close(w, d, C_gpu, C_ref, rows=None, cols=None):
    ab = abs_product(w, d)
    c0 = np.abs(d["C"]) if w.beta != 0 else np.zeros_like(ab)
    tol = gemm_bound(w.K, w.alpha, w.beta, ab, c0)
    err = np.abs(C_gpu - C_ref)
    bad = ~(err <= tol)
    assert not bad.any(), f"{bad.sum()} elements beyond tolerance; max err {err.max()}"


SMALL = [
    # (M, N, K, tA, tB, alpha, beta, dist, pad)
    (300, 260, 70, "N", "N", 1.0, 0.0, "uniform", 0),
    (300, 260, 70, "N", "T", 1.5, -0.5, "uniform", 0),
    (257, 129, 33, "T", "N", -1.0, 1.0, "normal", 0),
    (130, 390, 100, "T", "T", 0.75, 2.0, "uniform", 3),
    (128, 128, 16, "N", "N", 1.0, 0.0, "uniform", 0),
    (1, 1, 1, "N", "N", 2.0, 0.0, "uniform", 0),
    (5, 700, 9, "N", "T", 1.0, 1.0, "normal", 1),
    (700, 3, 17, "T", "N", 1.0, 0.0, "uniform", 0),
    # more than 128 verification tiles along N / M: checksum GEMMs in several column blocks
    (200, 16512, 40, "N", "T", 1.0, 0.5, "uniform", 0),
    (16600, 130, 40, "T", "N", -1.0, 0.0, "normal", 0),
]


@pytest.mark.parametrize("case", SMALL)
def test_fault_free_matches_oracle(ft, case):
    M, N, K, tA, tB, al, be, dist, pad = case
    w = syn.Workload("t", M, N, K, tA, tB, al, be, dist, True, seed=M * 7 + N + K)
    d = syn.make_inputs(w, pad=pad)
    C_gpu, rep = run_gpu(ft, w, d)
    C_ref, orep, st = run_oracle(w, d)
    assert rep.count == 0 and rep.tiles_flagged == 0 and orep == []
    assert_close(w, d, C_gpu, C_ref)
    C_nf, _ = run_gpu(ft, w, d, noft=True)
    assert_close(w, d, C_nf, C_ref)


@pytest.mark.parametrize("offsets", [(1, 0, 0), (0, 1, 1), (1, 1, 1)])
def test_misaligned_and_odd_ld(ft, offsets):
    """8-byte (non-vector) staging path: misaligned pointers and odd leading dimensions."""
    w = syn.Workload("t", 201, 150, 45, "N", "T", 1.25, -1.0, "uniform", True, seed=5)
    d = syn.make_inputs(w, pad=1)  # ld = rows + 1 (odd for even rows)
    plan = syn.fault_plan(w.M, w.N, 2, 9)
    C_gpu, rep = run_gpu(ft, w, d, plan=plan, offsets=offsets)
    C_ref, orep, _ = run_oracle(w, d, plan)
    assert report_key(rep.entries()) == report_key(orep)
    assert_close(w, d, C_gpu, C_ref)


@pytest.mark.parametrize("tA,tB", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
def test_injected_flips_reports_bit_exact(ft, tA, tB):
    w = syn.Workload("t", 390, 300, 130, tA, tB, 1.5, -0.5, "uniform", True, seed=11)
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, 9, 21)
    C_gpu, rep = run_gpu(ft, w, d, plan=plan)
    C_ref, orep, st = run_oracle(w, d, plan)
    assert rep.count == st.count == 9
    assert report_key(rep.entries()) == report_key(orep)
    assert (rep.tiles_flagged, rep.rows_flagged, rep.cols_flagged) == \
        (st.tiles_flagged, st.rows_flagged, st.cols_flagged)
    assert_close(w, d, C_gpu, C_ref)


def test_multiple_errors_in_one_tile(ft):
    """Two flips in one tile (distinct rows/cols) and two in one row: candidate path (kind 2).
    Tiles (1,1) and (0,1) put the two columns in different 64-column halves (the two CTAs of a
    pair tile): same row, and different rows."""
    w = syn.Workload("t", 256, 256, 64, "N", "N", 1.0, 0.0, "uniform", False, seed=3)
    d = syn.make_inputs(w)
    plan = (np.array([3, 40, 200, 200, 5, 70], np.int64), np.array([10, 55, 130, 250, 140, 230], np.int64),
            np.array([50, 58, 45, 61, 52, 44], np.int32))
    C_gpu, rep = run_gpu(ft, w, d, plan=plan)
    C_ref, orep, st = run_oracle(w, d, plan)
    assert report_key(rep.entries()) == report_key(orep)
    assert sorted((e["i"], e["j"]) for e in rep.entries()) == [(3, 10), (5, 140), (40, 55), (70, 230),
                                                               (200, 130), (200, 250)]
    assert_close(w, d, C_gpu, C_ref)


def test_four_flips_in_one_tile_same_thread(ft):
    """FTBLAS_MAX_FLIPS_PER_TILE (4) flips in one tile, three of them on elements one thread of
    the persistent kernel holds (same row, adjacent columns; the row below), plus a lone flip in
    another tile: every flip is applied (the per-thread hit list and its jump table), reports
    bit-exact vs the oracle (candidate path, kind 2), C within the tolerance."""
    w = syn.Workload("t", 256, 256, 96, "N", "N", 1.25, 0.5, "uniform", True, seed=8)
    d = syn.make_inputs(w)
    # (3, 8), (3, 10), (1, 8): fragment rows a = 1, 0 of row group g = 1 and columns (t = 0, e = 0 /
    # 1) of fragment column b = 1 -- one thread of MMA warp 0 in the 32 x 64 warp tiling
    plan = (np.array([3, 3, 1, 70, 200], np.int64), np.array([8, 10, 8, 100, 140], np.int64),
            np.array([53, 57, 61, 49, 55], np.int32))
    C_gpu, rep = run_gpu(ft, w, d, plan=plan)
    C_ref, orep, st = run_oracle(w, d, plan)
    assert report_key(rep.entries()) == report_key(orep)
    assert rep.count == st.count
    assert sorted((e["i"], e["j"]) for e in rep.entries()) == [(1, 8), (3, 8), (3, 10), (70, 100), (200, 140)]
    assert_close(w, d, C_gpu, C_ref)


@pytest.mark.parametrize("bit", [40, 47, 51, 52, 55, 60, 61, 62])
def test_each_bit_class(ft, bit):
    w = syn.Workload("t", 256, 256, 200, "N", "N", 1.0, 0.0, "normal", False, seed=bit)
    d = syn.make_inputs(w)
    rng = np.random.default_rng(bit)
    plan = (np.array([rng.integers(256)], np.int64), np.array([rng.integers(256)], np.int64),
            np.array([bit], np.int32))
    C_gpu, rep = run_gpu(ft, w, d, plan=plan)
    C_ref, orep, _ = run_oracle(w, d, plan)
    assert report_key(rep.entries()) == report_key(orep)
    assert rep.count == 1
    assert_close(w, d, C_gpu, C_ref)


def test_degenerate_shapes(ft):
    import torch
    # M == 0 / N == 0: no-op, empty report
    z = torch.zeros(4, dtype=torch.float64, device="cuda")
    rep = ft.Report(4)
    ft.ftblas_dgemm("N", "N", 0, 5, 3, 1.0, z, 1, z, 3, 0.0, z, 1, rep)
    assert rep.count == 0
    # K == 0: C := beta C;  alpha == 0: A, B not read (NULL)
    w = syn.Workload("t", 140, 70, 0, "N", "N", 1.0, 2.0, "uniform", True, seed=1)
    d = syn.make_inputs(w)
    C_t, pC = to_dev(d["C"])
    ft.ftblas_dgemm("N", "N", 140, 70, 0, 1.0, None, 140, None, 1, 2.0, pC, 140, rep)
    assert rep.count == 0
    assert np.array_equal(from_dev(C_t, d["C"]), 2.0 * d["C"])
    C_t, pC = to_dev(d["C"])
    ft.ftblas_dgemm("N", "N", 140, 70, 9, 0.0, None, 140, None, 9, -1.0, pC, 140, rep)
    assert np.array_equal(from_dev(C_t, d["C"]), -d["C"])


def test_beta_zero_ignores_nan_in_C(ft):
    w = syn.Workload("t", 150, 140, 20, "N", "N", 1.0, 0.0, "uniform", False, seed=2)
    d = syn.make_inputs(w)
    d["C"] = np.asfortranarray(np.full((150, 140), np.nan))
    C_gpu, rep = run_gpu(ft, w, d)
    assert np.isfinite(C_gpu).all() and rep.count == 0


@pytest.mark.parametrize("shape", ["c0", "blocks_nt", "blocks_ntn_ragged", "rowblocks"])
def test_host_buffer_entry_point(ft, shape):
    """The e2e call on host buffers: pipelined over column blocks (H2D / GEMM / D2H overlap),
    report accumulated over the blocks; must equal the oracle on the whole problem."""
    if shape == "c0":
        w = syn.CONFIGS[0]
    elif shape == "blocks_nt":   # 9 column tiles -> 8 blocks, transposed B (2-D row-slab copies)
        w = syn.Workload("hb", 300, 1100, 60, "N", "T", -0.75, 1.5, "uniform", True, seed=31, n_flips=7)
    elif shape == "blocks_ntn_ragged":  # ragged last tile, transposed A, beta = 0
        w = syn.Workload("hb2", 130, 390, 33, "T", "N", 2.0, 0.0, "normal", True, seed=32, n_flips=3)
    else:                        # 16 x 150 tiles: 2 row blocks x 8 column blocks, op(A) = A^T
        w = syn.Workload("hb3", 2048, 19200, 16, "T", "N", 1.0, -1.0, "uniform", True, seed=33, n_flips=9)
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, w.n_flips, w.seed)
    ft.ftblas_set_fault_plan(*plan)
    C = np.asfortranarray(d["C"].copy())
    rep = ft.Report(64)
    ft.ftblas_dgemm_host(w.transA, w.transB, w.M, w.N, w.K, w.alpha, np.asfortranarray(d["A"]),
                         d["lda"], np.asfortranarray(d["B"]), d["ldb"], w.beta, C, d["ldc"], rep)
    ft.ftblas_clear_fault_plan()
    C_ref, orep, _ = run_oracle(w, d, plan)
    assert report_key(rep.entries()) == report_key(orep)
    assert_close(w, d, C, C_ref)


@pytest.mark.parametrize("split", ["cols", "rows"])
def test_blocked_calls_with_offsets_and_append(ft, split):
    """ftblas_dgemm_ex on column blocks (the chunked broadcast path) or row blocks (shards)
    with a global fault plan and FTBLAS_REPORT_APPEND: the accumulated report must equal
    the oracle's report of the whole problem, and C must match."""
    import torch
    w = syn.Workload("blk", 400, 520, 70, "N", "N", 1.25, 0.5, "uniform", True, seed=23)
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, 6, 9)
    A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
    ft.ftblas_set_fault_plan(*plan)
    ft.ftblas_report_reset()
    if split == "cols":  # later blocks reuse the A encoding (FTBLAS_REUSE_A_ENCODE)
        for q, (c0, c1) in enumerate([(0, 256), (256, 384), (384, 520)]):
            ft.ftblas_dgemm_ex("N", "N", w.M, c1 - c0, w.K, w.alpha, pA, d["lda"], pB + 8 * c0 * d["ldb"],
                               d["ldb"], w.beta, pC + 8 * c0 * d["ldc"], d["ldc"], 0, c0, q > 0,
                               reuse_a=q > 0)
    else:
        for q, (r0, r1) in enumerate([(0, 128), (128, 400)]):
            ft.ftblas_dgemm_ex("N", "N", r1 - r0, w.N, w.K, w.alpha, pA + 8 * r0, d["lda"], pB, d["ldb"],
                               w.beta, pC + 8 * r0, d["ldc"], r0, 0, q > 0)
    rep = ft.ftblas_report_fetch(ft.Report(64))
    ft.ftblas_clear_fault_plan()
    C = from_dev(C_t, d["C"])
    C_ref, orep, st = run_oracle(w, d, plan)
    assert rep.count == st.count == 6
    assert report_key(rep.entries()) == report_key(orep)
    assert_close(w, d, C, C_ref)


def test_blocked_calls_growing_workspace(ft):
    """Column blocks of increasing width after ftblas_release(), later blocks asking to reuse
    the A encoding: the workspace grows on the second and third call (free + malloc), so the
    cached encoding must be dropped and A encoded again.  Report and C must
    equal the oracle's for the whole problem."""
    w = syn.Workload("grow", 384, 1024, 96, "N", "N", 1.0, -1.0, "uniform", True, seed=29)
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, 7, 13)
    A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
    ft.ftblas_release()
    ft.ftblas_set_fault_plan(*plan)
    ft.ftblas_report_reset()
    for q, (c0, c1) in enumerate([(0, 128), (128, 384), (384, 1024)]):
        ft.ftblas_dgemm_ex("N", "N", w.M, c1 - c0, w.K, w.alpha, pA, d["lda"], pB + 8 * c0 * d["ldb"],
                           d["ldb"], w.beta, pC + 8 * c0 * d["ldc"], d["ldc"], 0, c0, q > 0, reuse_a=q > 0)
    rep = ft.ftblas_report_fetch(ft.Report(64))
    ft.ftblas_clear_fault_plan()
    C = from_dev(C_t, d["C"])
    C_ref, orep, st = run_oracle(w, d, plan)
    assert rep.count == st.count == 7 and rep.tiles_flagged == st.tiles_flagged
    assert report_key(rep.entries()) == report_key(orep)
    assert_close(w, d, C, C_ref)


@pytest.mark.parametrize("tB", ["N", "T"])
def test_shared_b_encoding(ft, tB):
    """op(B)'s encoding computed in column slices (ftblas_encode_b, as the
    ranks of a sharded product do), assembled by shard.assemble_b_encoding and passed with
    FTBLAS_B_ENCODED: reports and C equal the oracle's, in two column blocks (the second reusing
    the A encoding), under every tiling."""
    import torch
    from paper_2305_02444_b200 import shard
    w = syn.Workload("benc", 300, 700, 90, "N", tB, 1.5, -0.5, "uniform", True, seed=41)
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, 5, 23)
    A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
    ft.ftblas_set_fault_plan(*plan)
    ft.ftblas_report_reset()
    ldb = d["ldb"]
    for q, (c0, c1) in enumerate([(0, 256), (256, 700)]):
        n = c1 - c0
        b_off = c0 * ldb if tB == "N" else c0
        pieces = []
        for t0, t1, nr in shard.b_encoding_slices(n, 3):
            piece = torch.zeros(max(1, ft.ftblas_b_encoding_len(nr, w.K)), dtype=torch.float64, device="cuda")
            if nr:
                off = b_off + (t0 * 128 * ldb if tB == "N" else t0 * 128)
                ft.ftblas_encode_b(tB, nr, w.K, pB + 8 * off, ldb, piece)
            pieces.append(piece)
        enc = torch.zeros(ft.ftblas_b_encoding_len(n, w.K), dtype=torch.float64, device="cuda")
        shard.assemble_b_encoding(pieces, n, w.K, ft.ftblas_b_encoding_layout, enc)
        ft.ftblas_set_b_encoding(enc, n, w.K)
        ft.ftblas_dgemm_ex("N", tB, w.M, n, w.K, w.alpha, pA, d["lda"], pB + 8 * b_off, ldb, w.beta,
                           pC + 8 * c0 * d["ldc"], d["ldc"], 0, c0, q > 0, reuse_a=q > 0, b_encoded=True)
        torch.cuda.synchronize()
        ft.ftblas_set_b_encoding(None)
    rep = ft.ftblas_report_fetch(ft.Report(64))
    ft.ftblas_clear_fault_plan()
    C = from_dev(C_t, d["C"])
    C_ref, orep, st = run_oracle(w, d, plan)
    assert rep.count == st.count == 5 and rep.tiles_flagged == st.tiles_flagged
    assert report_key(rep.entries()) == report_key(orep)
    assert_close(w, d, C, C_ref)


def _flip(x: float, bit: int) -> float:
    import struct
    b = struct.unpack("<Q", struct.pack("<d", x))[0] ^ (1 << bit)
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def test_gpu_subthreshold_flip_matches_oracle(ft):
    """Reading R10: flips too small for the round-off threshold (low mantissa bits) are left in
    C by both sides -- identical (empty) reports, C within the R9 tolerance of the oracle's C
    (which keeps the same flipped value) -- while large flips in the same run are corrected."""
    w = syn.Workload("sub", 256, 256, 200, "N", "T", 1.5, -0.5, "uniform", True, seed=61)
    d = syn.make_inputs(w)
    # one flip per tile: in three tiles a low mantissa bit whose change is >= 10x the R9
    # tolerance but <= 1e-10 (about 1/10 of the row threshold tau ~ 1e-9 here), bit 50 (far
    # above tau) in the fourth
    ab = abs_product(w, d)
    ii, jj, bits = [5, 140, 20, 200], [7, 30, 150, 222], []
    for i, j in zip(ii[:3], jj[:3]):
        acc = oracle.dot(w.transA, w.transB, w.K, d["A"], d["lda"], d["B"], d["ldb"], i, j)
        tol = 4 * (w.K + 2) * 2.0 ** -53 * (abs(w.alpha) * ab[i, j] + abs(w.beta) * abs(d["C"][i, j]))
        ok = [b for b in range(52) if 10 * tol <= abs(w.alpha * (_flip(acc, b) - acc)) <= 1e-10]
        assert ok, (i, j)
        bits.append(ok[-1])
    plan = (np.array(ii, np.int64), np.array(jj, np.int64), np.array(bits + [50], np.int32))
    C_gpu, rep = run_gpu(ft, w, d, plan=plan)
    C_ref, orep, st = run_oracle(w, d, plan)
    assert report_key(rep.entries()) == report_key(orep)
    assert [(e["i"], e["j"]) for e in rep.entries()] == [(200, 222)]
    assert_close(w, d, C_gpu, C_ref)
    # the sub-threshold flips really stayed (their change exceeds the R9 tolerance): compare
    # with the oracle's fault-free C
    C_clean, _, _ = run_oracle(w, d)
    for i, j, bit in zip(*[p.tolist() for p in plan]):
        tol = 4 * (w.K + 2) * 2.0 ** -53 * (abs(w.alpha) * ab[i, j] + abs(w.beta) * abs(d["C"][i, j]))
        if bit < 40:
            assert abs(C_gpu[i, j] - C_clean[i, j]) > tol, (i, j, bit)
        else:
            assert abs(C_gpu[i, j] - C_clean[i, j]) <= tol


def test_gpu_c0_bound_window_matches_oracle(ft):
    """Reading R4k: when the |beta| |C0| term dominates the threshold, flips whose change lies
    between the exact-sum threshold (sum |C0|) and the bound actually used (n up(max |C0|)) are
    not flagged -- by the kernel and, since round 2, by the oracle alike (round 1's oracle used
    the sum and flagged them); flips above the bound are corrected by both."""
    w = syn.Workload("win", 256, 256, 64, "N", "N", 1.0, 1.0, "uniform", True, seed=67)
    d = syn.make_inputs(w)
    scale = 1e-4  # operands small: |alpha| |A||B| << |beta| |C0| in the threshold
    d["A"] = np.asfortranarray(d["A"] * scale)
    d["B"] = np.asfortranarray(d["B"] * scale)
    opA, opB = d["A"], d["B"]
    acc = opA @ opB
    U = 2.0 ** -53
    K = w.K
    picks = []
    for (tm, tn) in [(0, 0), (0, 1), (1, 0), (1, 1)]:
        r0, c0 = 128 * tm, 128 * tn
        tile_c0 = np.abs(d["C"][r0:r0 + 128, c0:c0 + 128])
        rng = np.random.default_rng(tm * 2 + tn)
        for _ in range(2000):
            i, j = r0 + int(rng.integers(128)), c0 + int(rng.integers(128))
            rowabs = np.abs(opA[i, :]).sum()
            bmax = np.abs(opB[:, c0:c0 + 128]).sum(axis=1).max()
            colabs = np.abs(opB[:, j]).sum()
            amax = np.abs(opA[r0:r0 + 128, :]).sum(axis=0).max()
            t_sum_r = 4 * U * (K + 131) * (rowabs * bmax + tile_c0[i - r0, :].sum())
            t_max_r = 4 * U * (K + 131) * (rowabs * bmax + 128 * tile_c0[i - r0, :].max())
            t_sum_c = 4 * U * (K + 131) * (amax * colabs + tile_c0[:, j - c0].sum())
            t_max_c = 4 * U * (K + 131) * (amax * colabs + 128 * tile_c0[:, j - c0].max())
            lo, hi = 1.1 * max(t_sum_r, t_sum_c), 0.9 * min(t_max_r, t_max_c)
            bits = [b for b in range(53) if lo < abs(_flip(acc[i, j], b) - acc[i, j]) < hi]
            if bits:
                picks.append((i, j, bits[0]))
                break
    assert len(picks) >= 3, picks
    big = (60, 60, 55)  # and one flip far above every threshold, in tile (0, 0)
    plan = (np.array([p[0] for p in picks] + [big[0]], np.int64),
            np.array([p[1] for p in picks] + [big[1]], np.int64),
            np.array([p[2] for p in picks] + [big[2]], np.int32))
    C_gpu, rep = run_gpu(ft, w, d, plan=plan)
    C_ref, orep, st = run_oracle(w, d, plan)
    assert report_key(rep.entries()) == report_key(orep)
    assert [(e["i"], e["j"]) for e in rep.entries()] == [(60, 60)]
    assert_close(w, d, C_gpu, C_ref)


def test_ex_argument_errors(ft):
    with pytest.raises(ft.FtblasError):
        ft.ftblas_dgemm_ex("N", "N", 4, 4, 4, 1.0, 0, 4, 0, 4, 0.0, 0, 4, 64, 0)
    with pytest.raises(ft.FtblasError):
        ft.ftblas_dgemm_ex("N", "N", 4, 4, 4, 1.0, 0, 4, 0, 4, 0.0, 0, 4, 0, 5)


# ---------------------------------------------------------------- BASELINE configs
def test_config0_all_flips_corrected(ftd):
    w = syn.CONFIGS[0]
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, w.n_flips, w.seed)
    C_gpu, rep = run_gpu(ftd, w, d, plan=plan)
    C_ref, orep, st = run_oracle(w, d, plan)
    assert rep.count == st.count == w.n_flips
    assert report_key(rep.entries()) == report_key(orep)
    assert sorted((e["i"], e["j"]) for e in rep.entries()) == sorted(zip(*[p.tolist() for p in plan[:2]]))
    assert_close(w, d, C_gpu, C_ref)


def sampled_check(w, d, C_gpu, n=300, seed=0, extra=()):
    rng = np.random.default_rng(seed)
    pts = [(int(rng.integers(w.M)), int(rng.integers(w.N))) for _ in range(n)] + list(extra)
    for (i, j) in pts:
        acc = oracle.dot(w.transA, w.transB, w.K, d["A"], d["lda"], d["B"], d["ldb"], i, j)
        ab = oracle.absdot(w.transA, w.transB, w.K, d["A"], d["lda"], d["B"], d["ldb"], i, j)
        c0 = d["C"][i, j] if w.beta != 0 else 0.0
        ref = w.alpha * acc + (w.beta * c0 if w.beta != 0 else 0.0)
        tol = gemm_bound(w.K, w.alpha, w.beta, ab, abs(c0))
        assert abs(C_gpu[i, j] - ref) <= tol, (i, j, C_gpu[i, j], ref)


_PAR = {}


def _tile_plan(plan, r0, r1, c0, c1):
    if plan is None:
        return None
    i, j, bit = plan
    m = (i >= r0) & (i < r1) & (j >= c0) & (j < c1)
    return (i[m] - r0, j[m] - c0, bit[m])


def _oracle_tile(t):
    """The unchanged oracle on one verification tile as a stand-alone problem (a tile's
    verification reads only op(A) rows I, op(B) columns J and the C0 tile), shifted back to
    the caller's coordinates."""
    w, d, plan = _PAR["w"], _PAR["d"], _PAR["plan"]
    tm, tn = t
    r0, r1 = 128 * tm, min(w.M, 128 * tm + 128)
    c0, c1 = 128 * tn, min(w.N, 128 * tn + 128)
    A = d["A"][r0:r1, :] if w.transA == "N" else d["A"][:, r0:r1]
    B = d["B"][:, c0:c1] if w.transB == "N" else d["B"][c0:c1, :]
    C = np.asfortranarray(d["C"][r0:r1, c0:c1].copy())
    lda = d["lda"]
    ldb = d["ldb"]
    sub = _tile_plan(plan, r0, r1, c0, c1)
    rep, st = oracle.abft_dgemm(w.transA, w.transB, r1 - r0, c1 - c0, w.K, w.alpha, A, lda, B, ldb,
                                w.beta, C, r1 - r0, faults=sub, cap=64)
    ents = [dict(e, tile_m=tm, tile_n=tn, i=e["i"] + r0, j=e["j"] + c0) for e in rep]
    return tm, tn, C, ents


def oracle_tiles(w, d, plan, tiles):
    """Oracle results of the listed (tm, tn) tiles, in parallel over the host cores (fork:
    the inputs are shared copy-on-write)."""
    import multiprocessing as mp
    import os
    _PAR.update(w=w, d=d, plan=plan)
    procs = max(1, min(len(tiles), os.cpu_count() or 1))
    if procs == 1:
        return [_oracle_tile(t) for t in tiles]
    with mp.get_context("fork").Pool(procs) as pool:
        return pool.map(_oracle_tile, tiles, chunksize=1)


def check_tiles(w, d, C_gpu, results):
    opA = d["A"] if w.transA == "N" else d["A"].T
    opB = d["B"] if w.transB == "N" else d["B"].T
    for tm, tn, Ct, _ in results:
        r0, c0 = 128 * tm, 128 * tn
        r1, c1 = r0 + Ct.shape[0], c0 + Ct.shape[1]
        ab = np.abs(opA[r0:r1, :]) @ np.abs(opB[:, c0:c1])
        cc = np.abs(d["C"][r0:r1, c0:c1]) if w.beta != 0 else 0.0
        tol = gemm_bound(w.K, w.alpha, w.beta, ab, cc)
        bad = ~(np.abs(C_gpu[r0:r1, c0:c1] - Ct) <= tol)
        assert not bad.any(), (tm, tn, int(bad.sum()))


def check_full_config(ft, w, clean_tiles=64):
    """Full-size config: the fault-free run on `clean_tiles` random tiles and the injected run
    on EVERY faulty tile plus the same clean tiles are compared with the oracle tile by tile
    (whole tiles, elementwise bound; reports bit-exact on the faulty tiles), plus sampled
    single-element dots anywhere."""
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, w.n_flips, w.seed)
    ntm, ntn = -(-w.M // 128), -(-w.N // 128)
    faulty = sorted({(int(i) // 128, int(j) // 128) for i, j in zip(plan[0], plan[1])})
    rng = np.random.default_rng(w.seed + 1000)
    clean = []
    while len(clean) < min(clean_tiles, ntm * ntn - len(faulty)):
        t = (int(rng.integers(ntm)), int(rng.integers(ntn)))
        if t not in faulty and t not in clean:
            clean.append(t)
    # fault-free run: no report; the clean tiles equal the oracle's
    C_clean, rep0 = run_gpu(ft, w, d)
    assert rep0.count == 0 and rep0.tiles_flagged == 0
    res_clean = oracle_tiles(w, d, None, clean)
    check_tiles(w, d, C_clean, res_clean)
    sampled_check(w, d, C_clean, n=100)
    # injected run: every planned flip located and corrected; faulty tiles vs the oracle
    C_gpu, rep = run_gpu(ft, w, d, plan=plan)
    got = report_key(rep.entries())
    assert rep.count == w.n_flips
    assert sorted((g[2], g[3]) for g in got) == sorted(zip(plan[0].tolist(), plan[1].tolist()))
    res = oracle_tiles(w, d, plan, faulty)
    assert report_key([e for r in res for e in r[3]]) == got
    check_tiles(w, d, C_gpu, res)
    # the clean tiles are untouched by the injection (bitwise the fault-free run's)
    for tm, tn, Ct, _ in res_clean:
        sl = (slice(128 * tm, 128 * tm + Ct.shape[0]), slice(128 * tn, 128 * tn + Ct.shape[1]))
        assert np.array_equal(C_gpu[sl], C_clean[sl])
    sampled_check(w, d, C_gpu, n=100, seed=1, extra=list(zip(plan[0].tolist(), plan[1].tolist()))[:50])


def test_config1_4096_tn(ftd):
    check_full_config(ftd, syn.CONFIGS[1])


def test_config2_rank_k_update(ftd):
    check_full_config(ftd, syn.CONFIGS[2])


def test_config3_16384(ftd):
    check_full_config(ftd, syn.CONFIGS[3])


def test_config4_32768x16384(ftd):
    """configs[4] is quoted for an 8-GPU row-block shard; each shard runs the single-GPU call,
    so the whole problem on one GPU (17 GB of operands) checks the same kernels at full size."""
    check_full_config(ftd, syn.CONFIGS[4], clean_tiles=16)


def test_zero_fault_transparency_and_no_false_positives(ft):
    """Fault-free ftblas_dgemm is bitwise identical to ftblas_dgemm_noft (the checksum work is
    additive: same DMMA sequence and epilogue formula) and flags nothing, over random shapes
    (1..400 x 1..400 x 1..300, all transposes, random alpha / beta) -- the SPEC's
    zero-fault-transparency and checksum-identity criteria at desk scale."""
    import torch
    rng = np.random.default_rng(2024)
    for trial in range(24):
        M, N = (int(x) for x in rng.integers(1, 401, 2))
        K = int(rng.integers(1, 301))
        tA, tB = ("N", "T")[int(rng.integers(2))], ("N", "T")[int(rng.integers(2))]
        alpha = float(rng.choice([1.0, -1.0, 0.5, 2.5]))
        beta = float(rng.choice([0.0, 1.0, -0.5]))
        w = syn.Workload("zf", M, N, K, tA, tB, alpha, beta, "normal", True, seed=100 + trial)
        d = syn.make_inputs(w)
        A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"])
        C1_t, pC1 = to_dev(d["C"]); C2_t, pC2 = to_dev(d["C"])
        ft.ftblas_clear_fault_plan()
        rep = ft.Report(16)
        ft.ftblas_dgemm(tA, tB, M, N, K, alpha, pA, d["lda"], pB, d["ldb"], beta, pC1, d["ldc"], rep)
        ft.ftblas_dgemm_noft(tA, tB, M, N, K, alpha, pA, d["lda"], pB, d["ldb"], beta, pC2, d["ldc"])
        torch.cuda.synchronize()
        assert rep.count == 0 and rep.tiles_flagged == 0, (M, N, K, tA, tB)
        assert torch.equal(C1_t, C2_t), (M, N, K, tA, tB, alpha, beta)


@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("tiles", ["ws", "pair", "full"])
def test_many_faulted_tiles_leave_neighbours_clean(tB, tiles):
    """Regression: 100 faulted tiles (each with a long single-element recompute) next to clean
    tiles, K deep enough that CTAs of different tiles share SMs for a long time.  Every flag
    must come from a planned flip: exactly one kind-1 correction per faulted tile, no other
    tile flagged, and C bitwise equal to the fault-free run (the corrected elements are
    recomputed, all others untouched).  (Pair CTAs with setmaxnreg failed this for NT.)"""
    import torch
    ft = _lib("gemm", tiles)
    try:
        w = syn.Workload("t", 2048, 2048, 2048, "N", tB, 1.5, -0.5, "uniform", True, seed=5)
        d = syn.make_inputs(w)
        plan = syn.fault_plan(w.M, w.N, 100, 17)
        C_clean, rep0 = run_gpu(ft, w, d)
        assert rep0.count == 0
        ft.ftblas_set_fault_plan(*plan)
        for _ in range(3):
            C_t, pC = to_dev(d["C"], 0)
            A_t, pA = to_dev(d["A"], 0)
            B_t, pB = to_dev(d["B"], 0)
            rep = ft.Report(8192)
            ft.ftblas_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"],
                            w.beta, pC, d["ldc"], rep)
            torch.cuda.synchronize()
            got = sorted((e["i"], e["j"], e["kind"]) for e in rep.entries())
            want = sorted((int(i), int(j), 1) for i, j in zip(plan[0], plan[1]))
            assert rep.count == 100 and rep.tiles_flagged == 100 and got == want
            C_gpu = from_dev(C_t, d["C"], 0)
            changed = np.argwhere(C_gpu != C_clean)
            assert {(int(i), int(j)) for i, j in changed} <= {(i, j) for i, j, _ in want}
            if len(changed):
                ii, jj = changed[:, 0], changed[:, 1]
                ab = abs_product(w, d)[ii, jj]
                tol = gemm_bound(w.K, w.alpha, w.beta, ab, np.abs(d["C"][ii, jj]))
                assert (np.abs(C_gpu[ii, jj] - C_clean[ii, jj]) <= tol).all()
    finally:
        ft.ftblas_clear_fault_plan()
        ft.ftblas_set_tile_policy("auto")


@pytest.mark.parametrize("tiles", ["ws", "pair", "full"])
def test_deep_k_faulted_tiles_no_spurious_flags(tiles):
    """The case that corrupted accumulators of concurrently running tiles when a K-long one-warp
    recomputation ran beside DMMA mainloops (4096^3 NT, 100 flips: ~10 extra tiles and hundreds
    of extra rows / columns flagged): with the recomputation deferred to
    correct_kernel, exactly the 100 planned flips are flagged (one row, one column each) and
    located, in each of 3 repetitions."""
    import torch
    ft = _lib("gemm", tiles)
    try:
        w = syn.Workload("t", 4096, 4096, 4096, "N", "T", 1.5, -0.5, "uniform", True, seed=5)
        d = syn.make_inputs(w)
        plan = syn.fault_plan(w.M, w.N, 100, 17)
        A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"])
        want = sorted((int(i), int(j), 1) for i, j in zip(plan[0], plan[1]))
        ft.ftblas_set_fault_plan(*plan)
        for _ in range(3):
            C_t, pC = to_dev(d["C"])
            rep = ft.Report(4096)
            ft.ftblas_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"],
                            w.beta, pC, d["ldc"], rep)
            torch.cuda.synchronize()
            assert (rep.count, rep.tiles_flagged, rep.rows_flagged, rep.cols_flagged) == (100, 100, 100, 100)
            assert sorted((e["i"], e["j"], e["kind"]) for e in rep.entries()) == want
    finally:
        ft.ftblas_clear_fault_plan()
        ft.ftblas_set_tile_policy("auto")


@pytest.mark.parametrize("tB", ["N", "T"])
def test_noft_pair_stress_matches_ft(tB):
    """The non-FT pair-tile kernel (the same producer / cluster-free structure as the FT pair
    kernel that once produced corrupted tiles) against the FT kernel at 2048^3, 5 repetitions:
    bitwise equal to the FT output wherever no flip was planned (same mainloop and epilogue
    formula), the planned elements within the bound of the FT (corrected) values, and every
    repetition bitwise identical."""
    import torch
    ft = _lib("gemm", "pair")
    try:
        w = syn.Workload("t", 2048, 2048, 2048, "N", tB, 1.5, -0.5, "uniform", True, seed=9)
        d = syn.make_inputs(w)
        plan = syn.fault_plan(w.M, w.N, 100, 19)
        C_ft, rep = run_gpu(ft, w, d, plan=plan)
        assert rep.count == 100
        mask = np.ones_like(C_ft, dtype=bool)
        mask[plan[0], plan[1]] = False
        ab = abs_product(w, d)[plan[0], plan[1]]
        tol = gemm_bound(w.K, w.alpha, w.beta, ab, np.abs(d["C"][plan[0], plan[1]]))
        first = None
        for _ in range(5):
            C_nf, _ = run_gpu(ft, w, d, noft=True)
            assert np.array_equal(C_nf[mask], C_ft[mask])
            assert (np.abs(C_nf[plan[0], plan[1]] - C_ft[plan[0], plan[1]]) <= tol).all()
            if first is None:
                first = C_nf
            assert np.array_equal(C_nf, first)
        sampled_check(w, d, first, n=200, seed=3)
    finally:
        ft.ftblas_clear_fault_plan()
        ft.ftblas_set_tile_policy("auto")


def test_host_entry_4x4_blocks_bitwise_equal_device():
    """The e2e entry at a size that takes the 4 x 4 block pipeline (16384^2 x 4096, beta != 0 so
    C0 blocks are uploaded too, 200 flips): C and the report equal the single device call's
    bitwise (blocks are whole 128 x 128 tiles, so every tile does the same arithmetic)."""
    import torch
    ft = _lib("gemm")
    w = syn.Workload("hb4", 16384, 16384, 4096, "N", "N", 1.0, 0.5, "uniform", True, seed=41, n_flips=200)
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, w.n_flips, w.seed)
    C_dev, rep_dev = run_gpu(ft, w, d, plan=plan)
    ft.ftblas_set_fault_plan(*plan)
    C = np.asfortranarray(d["C"].copy())
    rep = ft.Report(512)
    ft.ftblas_dgemm_host(w.transA, w.transB, w.M, w.N, w.K, w.alpha, np.asfortranarray(d["A"]),
                         d["lda"], np.asfortranarray(d["B"]), d["ldb"], w.beta, C, d["ldc"], rep)
    ft.ftblas_clear_fault_plan()
    torch.cuda.synchronize()
    assert rep.count == rep_dev.count == w.n_flips
    assert report_key(rep.entries()) == report_key(rep_dev.entries())
    assert np.array_equal(C, C_dev)


@pytest.mark.parametrize("tA,tB,K", [("N", "N", 8192), ("T", "T", 8192), ("N", "T", 16384)])
def test_host_entry_ksplit_first_block(tA, tB, K):
    """The e2e entry at depths that run pipeline row block 0 in k parts (16384^2 x K, 4 x 4
    blocks: 2 parts at K = 8192, 4 at 16384; beta != 0, 150 flips): same report as the single
    device call, C within the elementwise bound of it (the split blocks sum in another order;
    every other block is bitwise equal)."""
    import torch
    ft = _lib("gemm")
    w = syn.Workload("hb5", 16384, 16384, K, tA, tB, 1.25, -0.5, "uniform", True, seed=43, n_flips=150)
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, w.n_flips, w.seed)
    C_dev, rep_dev = run_gpu(ft, w, d, plan=plan)
    ft.ftblas_set_fault_plan(*plan)
    C = np.asfortranarray(d["C"].copy())
    rep = ft.Report(512)
    ft.ftblas_dgemm_host(w.transA, w.transB, w.M, w.N, w.K, w.alpha, np.asfortranarray(d["A"]),
                         d["lda"], np.asfortranarray(d["B"]), d["ldb"], w.beta, C, d["ldc"], rep)
    ft.ftblas_clear_fault_plan()
    torch.cuda.synchronize()
    assert rep.count == rep_dev.count == w.n_flips
    assert report_key(rep.entries()) == report_key(rep_dev.entries())
    # row block 0 of the 4 x 4 pipeline (rows [0, 4096)) is computed in k parts; every other
    # row block bitwise; row block 0 within the bound, checked on a 4096 x 1024 column slice
    # per column block (|A||B| of the full slab would be a 16384-wide dense product)
    assert np.array_equal(C[4096:, :], C_dev[4096:, :])
    opA = d["A"] if tA == "N" else d["A"].T
    opB = d["B"] if tB == "N" else d["B"].T
    absA = np.abs(opA[:4096, :])
    for c0 in range(0, 16384, 4096):
        cs = slice(c0, c0 + 1024)
        ab = absA @ np.abs(opB[:, cs])
        tol = gemm_bound(w.K, w.alpha, w.beta, ab, np.abs(d["C"][:4096, cs]))
        assert (np.abs(C[:4096, cs] - C_dev[:4096, cs]) <= 2 * tol).all()
    del C, C_dev, d
