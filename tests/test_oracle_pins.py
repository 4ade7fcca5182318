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
    # R4k: n * up(max |C0|), up(1.0) = 1 + 2^-20 (high word 0x3ff00000 + 1, low word 0)
    assert c0row.tolist() == [2.0 * (1 + 2.0 ** -20)] * 2 and c0col.tolist() == [2.0 * (1 + 2.0 ** -20)] * 2


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
                want = c0_bound_indep([d["C"][i, j] for j in range(j0, j1)]) if beta != 0 else 0.0
                assert c0row[i - i0] == want
            for j in range(j0, j1):
                assert ccol[j - j0] == float(sum(exact[i][j] for i in range(i0, i1)))
                want = c0_bound_indep([d["C"][i, j] for i in range(i0, i1)]) if beta != 0 else 0.0
                assert c0col[j - j0] == want


def up_indep(m: float) -> float:
    """Smallest double with a zero low 32-bit word strictly above |m| (struct, not the oracle)."""
    bits = struct.unpack("<Q", struct.pack("<d", abs(m)))[0]
    hi = (bits >> 32) & 0x7FFFFFFF
    if hi >= 0x7FF00000:
        return math.inf
    return struct.unpack("<d", struct.pack("<Q", (hi + 1) << 32))[0]


def c0_bound_indep(vals) -> float:
    """Reading R4k: n * up(max |v|) (NaN / Inf -> +Inf)."""
    if any(math.isnan(v) or math.isinf(v) for v in vals):
        return math.inf
    return len(vals) * up_indep(max(abs(v) for v in vals))


def test_c0_bounds_nonuniform_integers():
    """The |C0| terms of the threshold (c0row, c0col) on non-uniform integer data with a
    distinct maximum per row and column, negatives and zeros: equal to the independent
    definition and >= the exact sums sum |C0| they bound (a wrong index, range or a row/column
    swap changes the maxima here)."""
    rng = np.random.default_rng(43)
    M, N = 13, 11
    C0 = np.asfortranarray(rng.integers(-9, 10, size=(M, N)).astype(np.float64))
    C0[3, :] = 0.0
    C0[:, 5] *= 1000.0
    C0[7, 2] = -2.0 ** 40
    Z = np.asfortranarray(np.zeros((M, N)))
    for (i0, i1, j0, j1) in [(0, M, 0, N), (2, 9, 1, 7), (12, 13, 4, 11)]:
        _, _, c0row, c0col = oracle.ref_checksums("N", "N", 1, 1.0, Z, M, Z, 1, 0.5, C0, M,
                                                  i0, i1, j0, j1, np.zeros(1), np.zeros(1))
        for i in range(i0, i1):
            row = [float(C0[i, j]) for j in range(j0, j1)]
            assert c0row[i - i0] == c0_bound_indep(row)
            assert c0row[i - i0] >= sum(abs(v) for v in row)
        for j in range(j0, j1):
            col = [float(C0[i, j]) for i in range(i0, i1)]
            assert c0col[j - j0] == c0_bound_indep(col)
            assert c0col[j - j0] >= sum(abs(v) for v in col)
    # an Inf in C0 makes the bound infinite; beta = 0 ignores C0 entirely
    C0[1, 1] = math.inf
    _, _, c0row, c0col = oracle.ref_checksums("N", "N", 1, 1.0, Z, M, Z, 1, 2.0, C0, M,
                                              0, M, 0, N, np.zeros(1), np.zeros(1))
    assert math.isinf(c0row[1]) and math.isinf(c0col[1]) and math.isfinite(c0row[0])
    _, _, c0row, c0col = oracle.ref_checksums("N", "N", 1, 1.0, Z, M, Z, 1, 0.0, C0, M,
                                              0, M, 0, N, np.zeros(1), np.zeros(1))
    assert (c0row == 0).all() and (c0col == 0).all()


def tau_exact(d, tA, tB, K, alpha, beta, i0, i1, j0, j1, i=None, j=None):
    """Row (i given) or column (j given) threshold of reading R4/R4k from exact sums."""
    a, b = op_exact(d["A"], tA), op_exact(d["B"], tB)
    if i is not None:
        n = j1 - j0
        rowabs = sum(abs(a[i][k]) for k in range(K))
        bmax = max(sum(abs(b[k][jj]) for jj in range(j0, j1)) for k in range(K))
        c0 = Fraction(c0_bound_indep([float(d["C"][i, jj]) for jj in range(j0, j1)])) if beta else 0
        return 4 * Fraction(U) * (K + n + 3) * (abs(Fraction(alpha)) * rowabs * bmax + abs(Fraction(beta)) * c0)
    m = i1 - i0
    colabs = sum(abs(b[k][j]) for k in range(K))
    amax = max(sum(abs(a[ii][k]) for ii in range(i0, i1)) for k in range(K))
    c0 = Fraction(c0_bound_indep([float(d["C"][ii, j]) for ii in range(i0, i1)])) if beta else 0
    return 4 * Fraction(U) * (K + m + 3) * (abs(Fraction(alpha)) * amax * colabs + abs(Fraction(beta)) * c0)


@pytest.mark.parametrize("tA,tB", [("N", "T"), ("T", "N")])
def test_threshold_pinned_within_one_percent(tA, tB):
    """tau (reading R4/R4k) is pinned to +-1 %: an additive perturbation of 0.99 tau is not
    flagged, one of 1.01 tau is, separately for the row and the column threshold (computed
    here from exact sums).  A tau off by a factor >= 1.01 either way, a dropped term or a
    row / column mix-up fails."""
    rng = np.random.default_rng(47)
    M, N, K = 40, 36, 50
    alpha, beta = 1.5, -0.5
    w = syn.Workload("t", M, N, K, tA, tB, alpha, beta, "uniform", True, int(rng.integers(1 << 30)))
    d = syn.make_inputs(w)
    clean = clean_tile(d, tA, tB, M, N, K, alpha, beta)
    for trial in range(3):
        i, j = int(rng.integers(M)), int(rng.integers(N))
        tr = float(tau_exact(d, tA, tB, K, alpha, beta, 0, M, 0, N, i=i))
        tc = float(tau_exact(d, tA, tB, K, alpha, beta, 0, M, 0, N, j=j))
        for delta in (0.99 * tr, 1.01 * tr, 0.99 * tc, 1.01 * tc):
            for sign in (1.0, -1.0):
                Ct = clean.copy(order="F")
                Ct[i, j] += sign * delta
                rep, st = oracle.verify_tile(tA, tB, K, alpha, d["A"], d["lda"], d["B"], d["ldb"], beta,
                                             d["C"], d["ldc"], 0, M, 0, N, 0, 0, Ct)
                assert st.rows_flagged == (1 if delta > tr else 0), (delta / tr, trial)
                assert st.cols_flagged == (1 if delta > tc else 0), (delta / tc, trial)
                if delta > min(tr, tc):  # located (single flag pair or candidate recompute)
                    assert [(r["i"], r["j"]) for r in rep] == [(i, j)]
                    assert np.array_equal(Ct, clean)
                else:
                    assert rep == []


def flip_indep(x: float, bit: int) -> float:
    b = struct.unpack("<Q", struct.pack("<d", x))[0] ^ (1 << bit)
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def test_subthreshold_flip_window():
    """Reading R10: a flip whose change is below the row and column thresholds is not
    flagged (indistinguishable from rounding) and stays in C, within tau of
    the fault-free value; flips of the same element above twice the thresholds are located and
    corrected.  Sweeps every bit 0..62 of one element and checks each against exact tau."""
    rng = np.random.default_rng(53)
    M, N, K = 48, 40, 64
    alpha, beta = 1.5, -0.5
    w = syn.Workload("t", M, N, K, "N", "T", alpha, beta, "uniform", True, 4242)
    d = syn.make_inputs(w)
    clean = clean_tile(d, "N", "T", M, N, K, alpha, beta)
    i, j = 17, 23
    a, b = op_exact(d["A"], "N"), op_exact(d["B"], "T")
    acc = float(sum(a[i][k] * b[k][j] for k in range(K)))  # |exact - fl(acc)| << tau
    tr = float(tau_exact(d, "N", "T", K, alpha, beta, 0, M, 0, N, i=i))
    tc = float(tau_exact(d, "N", "T", K, alpha, beta, 0, M, 0, N, j=j))
    tmin = min(tr, tc)
    below = above = 0
    for bit in range(63):
        delta = abs(alpha * (flip_indep(acc, bit) - acc))
        if 0.5 * tmin < delta < 2.0 * max(tr, tc):
            continue  # within a factor 2 of a threshold: pinned by the 1 % test above
        C = d["C"].copy(order="F")
        rep, st = oracle.abft_dgemm("N", "T", M, N, K, alpha, d["A"], d["lda"], d["B"], d["ldb"], beta,
                                    C, d["ldc"], tile_m=64, tile_n=64,
                                    faults=(np.array([i]), np.array([j]), np.array([bit])))
        mask = np.ones_like(C, dtype=bool)
        mask[i, j] = False
        assert np.array_equal(C[mask], clean[mask])
        if delta <= 0.5 * tmin:
            below += 1
            assert rep == [] and st.tiles_flagged == 0
            assert abs(C[i, j] - clean[i, j]) <= tr and abs(C[i, j] - clean[i, j]) <= tc
            if delta > 4 * K * U * abs(alpha) * 64:  # above the per-element bound: really stays
                assert C[i, j] != clean[i, j]
        else:
            above += 1
            assert [(r["i"], r["j"], r["kind"]) for r in rep] == [(i, j, 1)]
            assert C[i, j] == clean[i, j]
    assert below >= 10 and above >= 20


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
