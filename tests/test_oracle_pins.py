"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these re-types the oracle's formula: they use exact integer / rational
arithmetic (Python int, fractions.Fraction), closed forms, IEEE-754 bit
manipulation via ``struct``, hand-worked golden fixtures from PAPER.md
section II.A and SPEC.md examples, invariants, and brute force on tiny inputs.
A dropped term, wrong sign/index or transposed operand in oracle/ftblas_oracle.c
fails at least one of them.
"""
import json
import math
import os
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synthetic as syn

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U = 2.0 ** -53


def F(x):
    return np.asfortranarray(np.array(x, dtype=np.float64))


def op_exact(X, trans):
    """op(X) as a list of lists of Fractions (X is a stored col-major array)."""
    rows = [[Fraction(float(v)) for v in r] for r in X.tolist()]
    if trans == "N":
        return rows
    return [list(c) for c in zip(*rows)]


def gemm_exact(tA, tB, alpha, A, B, beta, C):
    a, b = op_exact(A, tA), op_exact(B, tB)
    M, K, N = len(a), len(b), len(b[0]) if b else C.shape[1]
    out = [[None] * N for _ in range(M)]
    for i in range(M):
        for j in range(N):
            s = sum((a[i][k] * b[k][j] for k in range(K)), Fraction(0))
            c0 = Fraction(float(C[i, j])) if beta != 0 else Fraction(0)
            out[i][j] = Fraction(alpha) * s + Fraction(beta) * c0
    return out


def absprod(tA, tB, A, B):
    a, b = op_exact(A, tA), op_exact(B, tB)
    M, K, N = len(a), len(b), len(b[0])
    return [[float(sum(abs(a[i][k]) * abs(b[k][j]) for k in range(K))) for j in range(N)]
            for i in range(M)]


def rand_case(rng, M, N, K, tA, tB, dist="uniform", pad=0, beta_c=True):
    w = syn.Workload("t", M, N, K, tA, tB, 1.0, 0.0, dist, beta_c, int(rng.integers(1 << 30)))
    d = syn.make_inputs(w, pad=pad)
    return d


# ----------------------------------------------------------------- DGEMM definition
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("pad", [0, 3])
def test_dgemm_exact_integers(tA, tB, pad):
    """Small-integer operands: every product and partial sum is an exact binary64 integer,
    so the oracle must equal exact integer arithmetic bit for bit (pins indices/transposes)."""
    rng = np.random.default_rng(7)
    for (M, N, K) in [(1, 1, 1), (3, 5, 2), (7, 4, 9), (17, 13, 33)]:
        w = syn.Workload("t", M, N, K, tA, tB, 2.0, -3.0, "int", True, int(rng.integers(1 << 30)))
        d = syn.make_inputs(w, pad=pad, dist="int")
        C = d["C"].copy(order="F")
        exact = gemm_exact(tA, tB, 2.0, d["A"], d["B"], -3.0, d["C"])
        Cbuf = np.asfortranarray(np.zeros((d["ldc"], N)))
        Cbuf[:M, :] = C
        oracle.dgemm(tA, tB, M, N, K, 2.0, d["A"], d["lda"], d["B"], d["ldb"], -3.0,
                     Cbuf, d["ldc"])
        got = Cbuf[:M, :]
        for i in range(M):
            for j in range(N):
                assert got[i, j] == float(exact[i][j]), (tA, tB, M, N, K, i, j)


@pytest.mark.parametrize("tA,tB", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
def test_dgemm_rational_bound(tA, tB):
    """Tiny random reals vs exact rational arithmetic: the DGEMM error bound
    |C - C_exact| <= (K+2) u (|alpha||A||B| + |beta||C0|) holds elementwise."""
    rng = np.random.default_rng(11)
    for (M, N, K) in [(2, 3, 4), (4, 4, 7), (5, 2, 16)]:
        d = rand_case(rng, M, N, K, tA, tB)
        alpha, beta = 1.5, -0.5
        exact = gemm_exact(tA, tB, alpha, d["A"], d["B"], beta, d["C"])
        ab = absprod(tA, tB, d["A"], d["B"])
        C = d["C"].copy(order="F")
        oracle.dgemm(tA, tB, M, N, K, alpha, d["A"], d["lda"], d["B"], d["ldb"], beta, C, M)
        for i in range(M):
            for j in range(N):
                err = abs(Fraction(C[i, j]) - exact[i][j])
                bound = (K + 2) * U * (abs(alpha) * ab[i][j] + abs(beta) * abs(d["C"][i, j]))
                assert float(err) <= bound * 1.0000001


def test_dgemm_special_cases():
    rng = np.random.default_rng(3)
    d = rand_case(rng, 6, 5, 4, "N", "N")
    # beta == 0: C is not read (NaN input ignored), BLAS semantics.
    C = np.full((6, 5), np.nan, order="F")
    oracle.dgemm("N", "N", 6, 5, 4, 1.0, d["A"], 6, d["B"], 4, 0.0, C, 6)
    assert np.isfinite(C).all()
    # alpha == 0, beta == 1: C unchanged bit for bit.
    C0 = d["C"].copy(order="F")
    C1 = C0.copy(order="F")
    oracle.dgemm("N", "N", 6, 5, 4, 0.0, d["A"], 6, d["B"], 4, 1.0, C1, 6)
    assert np.array_equal(C0, C1)
    # identity: op(A) = I  =>  C = B exactly.
    eye = np.asfortranarray(np.eye(4))
    Bm = d["B"]
    C2 = np.zeros((4, 5), order="F")
    oracle.dgemm("N", "N", 4, 5, 4, 1.0, eye, 4, Bm, 4, 0.0, C2, 4)
    assert np.array_equal(C2, Bm)
    # K == 0: C := beta*C.
    C3 = C0.copy(order="F")
    oracle.dgemm("N", "N", 6, 5, 0, 1.0, d["A"], 6, d["B"], 1, 2.0, C3, 6)
    assert np.array_equal(C3, 2.0 * C0)


def test_dgemm_vs_independent_blas():
    """An independent implementation (numpy/OpenBLAS matmul) agrees within the bound."""
    rng = np.random.default_rng(5)
    M, N, K = 70, 45, 130
    d = rand_case(rng, M, N, K, "T", "N", dist="normal")
    C = d["C"].copy(order="F")
    oracle.dgemm("T", "N", M, N, K, -1.25, d["A"], d["lda"], d["B"], d["ldb"], 0.75, C, M)
    ref = -1.25 * (d["A"].T @ d["B"]) + 0.75 * d["C"]
    bound = 2 * (K + 2) * U * (1.25 * (np.abs(d["A"].T) @ np.abs(d["B"])) + 0.75 * np.abs(d["C"]))
    assert (np.abs(C - ref) <= bound).all()


def test_dot_and_absdot_closed_form():
    # A = ones(1,K), B = (1..K)^T  =>  dot = K(K+1)/2 exactly; absdot same for positive data;
    # with alternating signs dot = -K/2 (K even) and absdot = K(K+1)/2.
    K = 100
    A = np.asfortranarray(np.ones((1, K)))
    B = np.asfortranarray(np.arange(1, K + 1, dtype=np.float64).reshape(K, 1))
    assert oracle.dot("N", "N", K, A, 1, B, K, 0, 0) == K * (K + 1) / 2
    s = np.asfortranarray(np.array([[(-1.0) ** k for k in range(K)]]))
    assert oracle.dot("N", "N", K, s, 1, np.asfortranarray(np.ones((K, 1))), K, 0, 0) == 0.0
    Bs = np.asfortranarray((np.arange(1, K + 1) * (-1.0) ** np.arange(K)).reshape(K, 1))
    assert oracle.dot("N", "N", K, A, 1, Bs, K, 0, 0) == -K / 2
    assert oracle.absdot("N", "N", K, A, 1, Bs, K, 0, 0) == K * (K + 1) / 2


# ----------------------------------------------------------------- fault model
@pytest.mark.parametrize("x,bit", [(1.0, 51), (1.0, 52), (1.0, 62), (0.5, 62), (-3.25, 40),
                                   (1e-300, 60), (123.456, 63), (0.0, 45)])
def test_flip_matches_ieee_bits(x, bit):
    (b,) = struct.unpack("<Q", struct.pack("<d", x))
    (y,) = struct.unpack("<d", struct.pack("<Q", b ^ (1 << bit)))
    got = oracle.flip(x, bit)
    assert struct.pack("<d", got) == struct.pack("<d", y)


def test_flip_golden():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["bitflip"]
    assert oracle.flip(g["x"], g["bit"]) == g["y"]
    assert oracle.flip(1.0, 52) == 0.5          # exponent LSB: 2^0 -> 2^-1
    assert math.isinf(oracle.flip(1.0, 62))    # exponent 0x3FF -> 0x7FF, mantissa 0
    assert oracle.flip(0.5, 62) == 2.0 ** 1023  # exponent 0x3FE -> 0x7FE


# ----------------------------------------------------------------- encoding (section II.A)
def test_encode_spec_examples():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    A = F(g["encode_a"]["A"])
    ac, mx, rowabs = oracle.encode_a("N", 2, A, 2, 0, 2)
    assert ac.tolist() == g["encode_a"]["a_col"]
    assert mx == 6.0 and rowabs.tolist() == [3.0, 7.0]
    Bm = F(g["encode_b"]["B"])
    br, mx, colabs = oracle.encode_b("N", 2, Bm, 2, 0, 2)
    assert br.tolist() == g["encode_b"]["b_row"]
    assert mx == 7.0 and colabs.tolist() == [4.0, 6.0]
    cc = g["c_checksums"]
    C0 = F(cc["C"])
    Z = np.asfortranarray(np.zeros((2, 2)))
    crow, ccol, c0row, c0col = oracle.ref_checksums(
        "N", "N", 2, 1.0, Z, 2, Z, 2, cc["beta"], C0, 2, 0, 2, 0, 2, np.zeros(2), np.zeros(2))
    assert ccol.tolist() == cc["c_col"] and crow.tolist() == cc["c_row"]
    assert c0row.tolist() == [2.0, 2.0] and c0col.tolist() == [2.0, 2.0]


@pytest.mark.parametrize("tA", ["N", "T"])
def test_encode_exact_integers(tA):
    rng = np.random.default_rng(13)
    M, K = 11, 9
    w = syn.Workload("t", M, 3, K, tA, "N", 1, 0, "int", False, 99)
    d = syn.make_inputs(w, pad=2, dist="int")
    a = op_exact(d["A"], tA)
    for (i0, i1) in [(0, M), (2, 7), (10, 11)]:
        ac, mx, rowabs = oracle.encode_a(tA, K, d["A"], d["lda"], i0, i1)
        for k in range(K):
            assert ac[k] == float(sum(a[i][k] for i in range(i0, i1)))
        assert mx == max(float(sum(abs(a[i][k]) for i in range(i0, i1))) for k in range(K))
        for i in range(i0, i1):
            assert rowabs[i - i0] == float(sum(abs(a[i][k]) for k in range(K)))
    # B side with the transposed storage
    wb = syn.Workload("t", 3, M, K, "N", "T", 1, 0, "int", False, 98)
    db = syn.make_inputs(wb, dist="int")
    b = op_exact(db["B"], "T")
    br, mx, colabs = oracle.encode_b("T", K, db["B"], db["ldb"], 1, 6)
    for k in range(K):
        assert br[k] == float(sum(b[k][j] for j in range(1, 6)))
    assert mx == max(float(sum(abs(b[k][j]) for j in range(1, 6))) for k in range(K))
    for j in range(1, 6):
        assert colabs[j - 1] == float(sum(abs(b[k][j]) for k in range(K)))


def test_checksum_golden_cf():
    """C^f = A^c B^r = [[C, Ce],[e^T C, .]], hand-worked fixture."""
    g = json.load(open(os.path.join(GOLD, "huang_abraham_2x2.json")))
    A, Bm = F(g["A"]), F(g["B"])
    C = np.asfortranarray(np.zeros((2, 2)))
    oracle.dgemm("N", "N", 2, 2, 2, 1.0, A, 2, Bm, 2, 0.0, C, 2)
    assert C.tolist() == g["C"]
    ac, _, _ = oracle.encode_a("N", 2, A, 2, 0, 2)
    br, _, _ = oracle.encode_b("N", 2, Bm, 2, 0, 2)
    assert ac.tolist() == g["eT_A"] and br.tolist() == g["B_e"]
    crow, ccol, _, _ = oracle.ref_checksums("N", "N", 2, 1.0, A, 2, Bm, 2, 0.0, C, 2,
                                            0, 2, 0, 2, ac, br)
    assert crow.tolist() == g["C_e"] and ccol.tolist() == g["eT_C"]
    assert [g["Cf"][0][2], g["Cf"][1][2]] == g["C_e"] and g["Cf"][2][:2] == g["eT_C"]


@pytest.mark.parametrize("tA,tB", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
def test_checksum_invariants_exact(tA, tB):
    """e^T C = (e^T A) B and C e = A (B e) (+ the beta C0 sums), exactly, on integer data
    where no rounding occurs -- pins ref_checksums independently of its own formula."""
    rng = np.random.default_rng(17)
    M, N, K = 9, 8, 6
    w = syn.Workload("t", M, N, K, tA, tB, 1, 0, "int", True, int(rng.integers(1 << 30)))
    d = syn.make_inputs(w, dist="int")
    for alpha, beta in [(1.0, 0.0), (2.0, -1.0), (-1.0, 3.0)]:
        exact = gemm_exact(tA, tB, alpha, d["A"], d["B"], beta, d["C"])
        for (i0, i1, j0, j1) in [(0, M, 0, N), (2, 5, 1, 8), (8, 9, 0, 3)]:
            ac, _, _ = oracle.encode_a(tA, K, d["A"], d["lda"], i0, i1)
            br, _, _ = oracle.encode_b(tB, K, d["B"], d["ldb"], j0, j1)
            crow, ccol, c0row, c0col = oracle.ref_checksums(
                tA, tB, K, alpha, d["A"], d["lda"], d["B"], d["ldb"], beta, d["C"], d["ldc"],
                i0, i1, j0, j1, ac, br)
            for i in range(i0, i1):
                assert crow[i - i0] == float(sum(exact[i][j] for j in range(j0, j1)))
                want = sum(abs(d["C"][i, j]) for j in range(j0, j1)) if beta != 0 else 0.0
                assert c0row[i - i0] == want
            for j in range(j0, j1):
                assert ccol[j - j0] == float(sum(exact[i][j] for i in range(i0, i1)))


# ----------------------------------------------------------------- verify / locate / correct
def clean_tile(d, tA, tB, M, N, K, alpha, beta):
    C = d["C"].copy(order="F")
    oracle.dgemm(tA, tB, M, N, K, alpha, d["A"], d["lda"], d["B"], d["ldb"], beta, C, M)
    return C


def test_spec_single_additive_error():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["single_error"]
    n = g["n"]
    ones = np.asfortranarray(np.ones((n, n)))
    Ct = np.asfortranarray(np.full((n, n), g["clean_value"]))
    Ct[g["i"], g["j"]] += g["delta"]
    rep, st = oracle.verify_tile("N", "N", n, 1.0, ones, n, ones, n, 0.0, ones, n,
                                 0, n, 0, n, 0, 0, Ct)
    assert len(rep) == 1 and st.tiles_flagged == 1
    assert (rep[0]["i"], rep[0]["j"], rep[0]["kind"]) == (g["i"], g["j"], 1)
    assert rep[0]["residual"] == g["delta"]
    assert (Ct == g["clean_value"]).all()


@pytest.mark.parametrize("tA,tB", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
@pytest.mark.parametrize("dist", ["uniform", "normal"])
def test_no_false_positives(tA, tB, dist):
    """Fault-free: the round-off threshold never flags (many shapes, ragged tiles)."""
    rng = np.random.default_rng(19)
    for trial in range(6):
        M, N = (int(x) for x in rng.integers(1, 300, size=2))
        K = int(rng.integers(1, 400))
        d = rand_case(rng, M, N, K, tA, tB, dist=dist)
        alpha, beta = [(1.0, 0.0), (1.5, -0.5), (-1.0, 1.0)][trial % 3]
        C = d["C"].copy(order="F")
        rep, st = oracle.abft_dgemm(tA, tB, M, N, K, alpha, d["A"], d["lda"], d["B"], d["ldb"],
                                    beta, C, d["ldc"], tile_m=64, tile_n=96)
        assert rep == [] and st.tiles_flagged == 0 and st.rows_flagged == 0
        assert np.array_equal(C, clean_tile(d, tA, tB, M, N, K, alpha, beta))


@pytest.mark.parametrize("bit", list(range(40, 63)))
def test_every_flip_bit_located_and_corrected(bit):
    """Single flips of each bit in [40,62] (incl. Inf/NaN-producing exponent flips) are
    located at exactly (i,j) and the corrected C is bitwise the fault-free C."""
    rng = np.random.default_rng(100 + bit)
    M, N, K = 150, 140, 96
    d = rand_case(rng, M, N, K, "N", "T")
    alpha, beta = 1.5, -0.5
    clean = clean_tile(d, "N", "T", M, N, K, alpha, beta)
    i, j = int(rng.integers(M)), int(rng.integers(N))
    C = d["C"].copy(order="F")
    rep, st = oracle.abft_dgemm("N", "T", M, N, K, alpha, d["A"], d["lda"], d["B"], d["ldb"], beta,
                                C, d["ldc"], tile_m=128, tile_n=128,
                                faults=(np.array([i]), np.array([j]), np.array([bit])))
    assert [(r["i"], r["j"], r["kind"], r["tile_m"], r["tile_n"]) for r in rep] == \
        [(i, j, 1, i // 128, j // 128)]
    assert np.array_equal(C, clean)


def test_plan_of_flips_all_corrected_and_within_paper_bound():
    """BASELINE configs[0] shape (256^3, 4 flips) on the oracle: all detected/located/corrected,
    result within 4 K 2^-53 (|A||B|)_ij of the exact product (checked on sampled entries)."""
    w = syn.CONFIGS[0]
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, w.n_flips, w.seed)
    C = d["C"].copy(order="F")
    rep, st = oracle.abft_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, d["A"], d["lda"],
                                d["B"], d["ldb"], w.beta, C, d["ldc"], faults=plan)
    got = sorted((r["i"], r["j"]) for r in rep)
    assert got == sorted(zip(plan[0].tolist(), plan[1].tolist()))
    assert st.count == w.n_flips
    rng = np.random.default_rng(0)
    pts = list(zip(plan[0].tolist(), plan[1].tolist())) + \
        [(int(rng.integers(w.M)), int(rng.integers(w.N))) for _ in range(12)]
    for (i, j) in pts:
        exact = sum(Fraction(float(d["A"][i, k])) * Fraction(float(d["B"][k, j])) for k in range(w.K))
        ab = float(sum(abs(Fraction(float(d["A"][i, k])) * Fraction(float(d["B"][k, j])))
                       for k in range(w.K)))
        assert abs(float(Fraction(C[i, j]) - exact)) <= 4 * w.K * U * ab


def test_two_errors_one_tile_distinct_rows_cols():
    rng = np.random.default_rng(23)
    M, N, K = 64, 64, 50
    d = rand_case(rng, M, N, K, "N", "N")
    clean = clean_tile(d, "N", "N", M, N, K, 1.0, 0.0)
    C = d["C"].copy(order="F")
    plan = (np.array([3, 40]), np.array([10, 55]), np.array([50, 58]))
    rep, st = oracle.abft_dgemm("N", "N", M, N, K, 1.0, d["A"], M, d["B"], K, 0.0, C, M,
                                faults=plan)
    assert sorted((r["i"], r["j"], r["kind"]) for r in rep) == [(3, 10, 2), (40, 55, 2)]
    assert st.rows_flagged == 2 and st.cols_flagged == 2
    assert np.array_equal(C, clean)


def test_two_errors_same_row():
    rng = np.random.default_rng(29)
    M, N, K = 64, 64, 50
    d = rand_case(rng, M, N, K, "T", "N")
    clean = clean_tile(d, "T", "N", M, N, K, 1.0, 0.0)
    C = d["C"].copy(order="F")
    plan = (np.array([7, 7]), np.array([1, 60]), np.array([55, 47]))
    rep, st = oracle.abft_dgemm("T", "N", M, N, K, 1.0, d["A"], d["lda"], d["B"], d["ldb"], 0.0,
                                C, M, faults=plan)
    assert sorted((r["i"], r["j"]) for r in rep) == [(7, 1), (7, 60)]
    assert np.array_equal(C, clean)


def test_tiny_brute_force_all_positions():
    """Brute force over every element of a tiny problem: each single flip is corrected."""
    rng = np.random.default_rng(31)
    M, N, K = 5, 4, 3
    d = rand_case(rng, M, N, K, "N", "N")
    clean = clean_tile(d, "N", "N", M, N, K, 2.0, 0.5)
    for i in range(M):
        for j in range(N):
            C = d["C"].copy(order="F")
            rep, _ = oracle.abft_dgemm("N", "N", M, N, K, 2.0, d["A"], M, d["B"], K, 0.5, C, M,
                                       tile_m=3, tile_n=3,
                                       faults=(np.array([i]), np.array([j]), np.array([61])))
            assert [(r["i"], r["j"]) for r in rep] == [(i, j)]
            assert np.array_equal(C, clean)


def test_sensitivity_large_perturbation_detected():
    """Any perturbation >= 1e3 x the threshold scale is flagged (additive, via verify_tile)."""
    rng = np.random.default_rng(37)
    M, N, K = 40, 30, 200
    d = rand_case(rng, M, N, K, "N", "N")
    clean = clean_tile(d, "N", "N", M, N, K, 1.0, 0.0)
    for trial in range(20):
        i, j = int(rng.integers(M)), int(rng.integers(N))
        rowscale = np.abs(d["A"][i, :]).sum() * np.abs(d["B"]).sum(axis=1).max()
        delta = 1e3 * 4 * U * (K + N + 3) * rowscale * (1 if trial % 2 else -1)
        Ct = clean.copy(order="F")
        Ct[i, j] += delta
        rep, st = oracle.verify_tile("N", "N", K, 1.0, d["A"], M, d["B"], K, 0.0, d["C"], M,
                                     0, M, 0, N, 0, 0, Ct)
        assert [(r["i"], r["j"]) for r in rep] == [(i, j)]
        assert np.array_equal(Ct, clean)


def test_tiles_only_subset_matches_full():
    rng = np.random.default_rng(41)
    M, N, K = 200, 170, 30
    d = rand_case(rng, M, N, K, "N", "N")
    plan = syn.fault_plan(M, N, 3, 5, tile_m=64, tile_n=64)
    Cf = d["C"].copy(order="F")
    rep_full, _ = oracle.abft_dgemm("N", "N", M, N, K, 1.0, d["A"], M, d["B"], K, 0.0, Cf, M,
                                    tile_m=64, tile_n=64, faults=plan)
    ntm, ntn = -(-M // 64), -(-N // 64)
    mask = np.zeros(ntm * ntn, np.uint8)
    for i, j in zip(plan[0], plan[1]):
        mask[(j // 64) * ntm + i // 64] = 1
    Cs = d["C"].copy(order="F")
    rep_sub, _ = oracle.abft_dgemm("N", "N", M, N, K, 1.0, d["A"], M, d["B"], K, 0.0, Cs, M,
                                   tile_m=64, tile_n=64, faults=plan, tiles_only=mask)
    assert [(r["i"], r["j"]) for r in rep_sub] == [(r["i"], r["j"]) for r in rep_full]
