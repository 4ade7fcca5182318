/*
 * oracle/ftblas_oracle.c -- CPU ORACLE FOR THE ABFT DGEMM HOT PATH.
 *
 *   TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 *   bench.py's cpu_baseline / --impl reference legs may load this library.
 *   The product path (paper_2305_02444_b200, libftblas.so) never links,
 *   loads or calls it, and this file shares no code with it.
 *
 * Plain, slow, obviously correct.  Every floating-point quantity is binary64,
 * every sum runs in ascending index order, no blocking, no fusion, compiled
 * with -ffp-contract=off (no fused multiply-add contraction).
 *
 * What is computed (PAPER.md = /root/reference/PAPER.md; readings R1..R9 are
 * listed in DESIGN.md section 3):
 *   ora_dgemm        C := alpha*op(A)*op(B) + beta*C, the BLAS DGEMM definition
 *                    (PAPER.md section "Optimizing DGEMV"/"Implementation of DGEMM",
 *                    lines 799 and 823; op(A) in {A, A^T}).
 *   ora_encode_a/b   Huang-Abraham checksum encoding A^c = [A; e^T A],
 *                    B^r = [B, B e] restricted to one verification tile
 *                    (section II.A "Algorithm-Based Fault Tolerance", line 516).
 *   ora_ref_checksums  the checksum row/column of C^f = A^c B^r (line 516) with the
 *                    beta*C term folded in ("encoding of C^c and C^r is fused with the
 *                    matrix scaling routine C = beta C", section V.B).
 *   ora_verify_tile  compare C against C^r, C^c: "if the difference exceeds the
 *                    round-off threshold" (line 517), locate the erroneous row from the
 *                    row checksum and column from the column checksum (line 540),
 *                    correct one error per verification interval (line 521).
 *   ora_abft_dgemm   the whole hot path over all tiles, with seeded bit flips
 *                    injected into the accumulator ("An element of matrix C is randomly
 *                    selected for modification", section VI.C).
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py
 * (exact integer/rational arithmetic, closed forms, invariants, SPEC examples).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

#define U_ROUND (1.0 / 9007199254740992.0) /* u = 2^-53, unit roundoff of binary64 */

/* ---- storage accessors: column-major BLAS layout, element (r,c) at p[r + c*ld] ---- */
static double opA(const double *A, i64 lda, int tA, i64 i, i64 k) {
    return tA ? A[k + i * lda] : A[i + k * lda];
}
static double opB(const double *B, i64 ldb, int tB, i64 k, i64 j) {
    return tB ? B[j + k * ldb] : B[k + j * ldb];
}

/* Accumulator of one element: sum_k op(A)(i,k) * op(B)(k,j), k ascending. */
double ora_dot(int tA, int tB, i64 K, const double *A, i64 lda, const double *B, i64 ldb,
               i64 i, i64 j) {
    double s = 0.0;
    for (i64 k = 0; k < K; k++) s += opA(A, lda, tA, i, k) * opB(B, ldb, tB, k, j);
    return s;
}

/* sum_k |op(A)(i,k)| * |op(B)(k,j)| -- the (|A||B|)_ij of the error bounds. */
double ora_absdot(int tA, int tB, i64 K, const double *A, i64 lda, const double *B, i64 ldb,
                  i64 i, i64 j) {
    double s = 0.0;
    for (i64 k = 0; k < K; k++) s += fabs(opA(A, lda, tA, i, k)) * fabs(opB(B, ldb, tB, k, j));
    return s;
}

/* BLAS epilogue of one element: alpha*acc + beta*c0; beta == 0 means C is not read. */
static double epilogue(double alpha, double acc, double beta, double c0) {
    return beta == 0.0 ? alpha * acc : alpha * acc + beta * c0;
}

/* C[i0:i1, j0:j1] := alpha*op(A)*op(B) + beta*C  -- the DGEMM definition, triple loop. */
void ora_dgemm(int tA, int tB, i64 M, i64 N, i64 K, double alpha, const double *A, i64 lda,
               const double *B, i64 ldb, double beta, double *C, i64 ldc,
               i64 i0, i64 i1, i64 j0, i64 j1) {
    (void)M; (void)N;
    for (i64 j = j0; j < j1; j++)
        for (i64 i = i0; i < i1; i++) {
            double acc = ora_dot(tA, tB, K, A, lda, B, ldb, i, j);
            C[i + j * ldc] = epilogue(alpha, acc, beta, C[i + j * ldc]);
        }
}

/* Fault model: flip bit `bit` (0 = LSB of the mantissa, 63 = sign) of a binary64. */
double ora_flip(double x, int bit) {
    uint64_t b;
    memcpy(&b, &x, 8);
    b ^= (uint64_t)1 << bit;
    memcpy(&x, &b, 8);
    return x;
}

/* Encoding of the A side for row block I = [i0,i1):  A^c's extra row e^T A (line 516).
 *   ac[k]      = sum_{i in I} op(A)(i,k)
 *   *acabsmax  = max_k sum_{i in I} |op(A)(i,k)|      (threshold ingredient, reading R4)
 *   rowabs[i]  = sum_k |op(A)(i0+i,k)|                 (threshold ingredient, reading R4) */
void ora_encode_a(int tA, i64 K, const double *A, i64 lda, i64 i0, i64 i1,
                  double *ac, double *acabsmax, double *rowabs) {
    double mx = 0.0;
    for (i64 k = 0; k < K; k++) {
        double s = 0.0, sa = 0.0;
        for (i64 i = i0; i < i1; i++) {
            double a = opA(A, lda, tA, i, k);
            s += a;
            sa += fabs(a);
        }
        ac[k] = s;
        if (sa > mx) mx = sa;
    }
    *acabsmax = mx;
    for (i64 i = i0; i < i1; i++) {
        double sa = 0.0;
        for (i64 k = 0; k < K; k++) sa += fabs(opA(A, lda, tA, i, k));
        rowabs[i - i0] = sa;
    }
}

/* Encoding of the B side for column block J = [j0,j1):  B^r's extra column B e (line 516).
 *   br[k]      = sum_{j in J} op(B)(k,j)
 *   *brabsmax  = max_k sum_{j in J} |op(B)(k,j)|
 *   colabs[j]  = sum_k |op(B)(k,j0+j)| */
void ora_encode_b(int tB, i64 K, const double *B, i64 ldb, i64 j0, i64 j1,
                  double *br, double *brabsmax, double *colabs) {
    double mx = 0.0;
    for (i64 k = 0; k < K; k++) {
        double s = 0.0, sa = 0.0;
        for (i64 j = j0; j < j1; j++) {
            double b = opB(B, ldb, tB, k, j);
            s += b;
            sa += fabs(b);
        }
        br[k] = s;
        if (sa > mx) mx = sa;
    }
    *brabsmax = mx;
    for (i64 j = j0; j < j1; j++) {
        double sa = 0.0;
        for (i64 k = 0; k < K; k++) sa += fabs(opB(B, ldb, tB, k, j));
        colabs[j - j0] = sa;
    }
}

/* Reference checksums of the C tile (I,J), i.e. the border of C^f = A^c B^r (line 516),
 * with beta*C0 encoded alongside (line 558):
 *   crow[i] = alpha * sum_k op(A)(i,k) br[k]  + beta * sum_{j in J} C0(i,j)     (C e)
 *   ccol[j] = alpha * sum_k ac[k] op(B)(k,j)  + beta * sum_{i in I} C0(i,j)     (e^T C)
 * and the bounds of the absolute C0 sums used by the threshold (readings R4, R4k):
 *   c0row[i] = |J| * up(max_{j in J} |C0(i,j)|)  >=  sum_{j in J} |C0(i,j)|,
 *   c0col[j] = |I| * up(max_{i in I} |C0(i,j)|)  >=  sum_{i in I} |C0(i,j)|,
 * up(x) = the binary64 whose high 32-bit word is that of x plus one and whose low word is
 * zero (the smallest such double above x; +Inf when x is Inf/NaN or in the top binade step).
 * beta == 0: C0 is not read and the C0 terms are 0. */
/* High 32-bit word of |x| (sign cleared): integer maxima of it order non-negative doubles. */
static uint32_t abs_hi(double x) {
    uint64_t b;
    memcpy(&b, &x, 8);
    return (uint32_t)(b >> 32) & 0x7fffffffu;
}
/* n * up(m) for the maximum high word h of |C0| over n elements (reading R4k). */
double ora_c0_bound(i64 n, uint32_t h) {
    if (h >= 0x7ff00000u) return INFINITY;
    uint64_t b = (uint64_t)(h + 1u) << 32;
    double up;
    memcpy(&up, &b, 8);
    return (double)n * up;
}

void ora_ref_checksums(int tA, int tB, i64 K, double alpha, const double *A, i64 lda,
                       const double *B, i64 ldb, double beta, const double *C0, i64 ldc,
                       i64 i0, i64 i1, i64 j0, i64 j1, const double *ac, const double *br,
                       double *crow, double *ccol, double *c0row, double *c0col) {
    for (i64 i = i0; i < i1; i++) {
        double r = 0.0;
        for (i64 k = 0; k < K; k++) r += opA(A, lda, tA, i, k) * br[k];
        double c = 0.0;
        uint32_t h = 0;
        if (beta != 0.0)
            for (i64 j = j0; j < j1; j++) {
                c += C0[i + j * ldc];
                if (abs_hi(C0[i + j * ldc]) > h) h = abs_hi(C0[i + j * ldc]);
            }
        crow[i - i0] = beta == 0.0 ? alpha * r : alpha * r + beta * c;
        c0row[i - i0] = beta == 0.0 ? 0.0 : ora_c0_bound(j1 - j0, h);
    }
    for (i64 j = j0; j < j1; j++) {
        double s = 0.0;
        for (i64 k = 0; k < K; k++) s += ac[k] * opB(B, ldb, tB, k, j);
        double c = 0.0;
        uint32_t h = 0;
        if (beta != 0.0)
            for (i64 i = i0; i < i1; i++) {
                c += C0[i + j * ldc];
                if (abs_hi(C0[i + j * ldc]) > h) h = abs_hi(C0[i + j * ldc]);
            }
        ccol[j - j0] = beta == 0.0 ? alpha * s : alpha * s + beta * c;
        c0col[j - j0] = beta == 0.0 ? 0.0 : ora_c0_bound(i1 - i0, h);
    }
}

/* One correction record (same field order as the product's ftblas_correction). */
typedef struct {
    i64 tile_m, tile_n; /* verification tile coordinates */
    i64 i, j;           /* 0-based element of C */
    double residual;    /* row-checksum residual d_i of the flagged row (informational) */
    int32_t kind;       /* 1: single error at (flagged row) x (flagged column); 2: candidate recompute */
    int32_t pad;
} ora_correction;

typedef struct {
    i64 count;         /* corrections found (entries beyond capacity are dropped) */
    i64 tiles_flagged; /* tiles with at least one flagged row or column */
    i64 rows_flagged;  /* total flagged rows */
    i64 cols_flagged;  /* total flagged columns */
} ora_stats;

/* Threshold (readings R4, R4k):  tau = 4 u (K + n + 3) * rho,  rho an upper bound of the
 * absolute checksum |alpha| (|A||B| e)_i + |beta| (|C0| e)_i built from norms and the
 * rounded-up |C0| maxima (c0row / c0col above).  The flag test is written !(x <= tau) so
 * that NaN/Inf residuals are flagged. */
static int flagged(double resid, double tau) { return !(fabs(resid) <= tau); }

/* Verify one tile, locate and correct (lines 517, 540, 521; readings R5-R7).
 * Ct: the computed tile (col-major, ld = ldt), corrected in place.  C0: the original C
 * (only read when beta != 0).  Returns the number of corrections appended to rep. */
i64 ora_verify_tile(int tA, int tB, i64 K, double alpha, const double *A, i64 lda,
                    const double *B, i64 ldb, double beta, const double *C0, i64 ldc,
                    i64 i0, i64 i1, i64 j0, i64 j1, i64 tile_m, i64 tile_n,
                    double *Ct, i64 ldt, ora_correction *rep, i64 rep_cap, i64 rep_base,
                    ora_stats *st) {
    i64 m = i1 - i0, n = j1 - j0;
    double *ac = malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
    double *br = malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
    double *rowabs = malloc(sizeof(double) * (size_t)m), *colabs = malloc(sizeof(double) * (size_t)n);
    double *crow = malloc(sizeof(double) * (size_t)m), *ccol = malloc(sizeof(double) * (size_t)n);
    double *c0row = malloc(sizeof(double) * (size_t)m), *c0col = malloc(sizeof(double) * (size_t)n);
    double *drow = malloc(sizeof(double) * (size_t)m), *dcol = malloc(sizeof(double) * (size_t)n);
    int *frow = calloc((size_t)m, sizeof(int)), *fcol = calloc((size_t)n, sizeof(int));
    double acmax, brmax;
    ora_encode_a(tA, K, A, lda, i0, i1, ac, &acmax, rowabs);
    ora_encode_b(tB, K, B, ldb, j0, j1, br, &brmax, colabs);
    ora_ref_checksums(tA, tB, K, alpha, A, lda, B, ldb, beta, C0, ldc, i0, i1, j0, j1, ac, br,
                      crow, ccol, c0row, c0col);
    i64 nr = 0, nc = 0, ri = -1, cj = -1;
    for (i64 i = 0; i < m; i++) {
        double s = 0.0;
        for (i64 j = 0; j < n; j++) s += Ct[i + j * ldt];
        drow[i] = s - crow[i];
        double tau = 4.0 * U_ROUND * (double)(K + n + 3) *
                     (fabs(alpha) * rowabs[i] * brmax + fabs(beta) * c0row[i]);
        if (flagged(drow[i], tau)) { frow[i] = 1; nr++; ri = i; }
    }
    for (i64 j = 0; j < n; j++) {
        double s = 0.0;
        for (i64 i = 0; i < m; i++) s += Ct[i + j * ldt];
        dcol[j] = s - ccol[j];
        double tau = 4.0 * U_ROUND * (double)(K + m + 3) *
                     (fabs(alpha) * acmax * colabs[j] + fabs(beta) * c0col[j]);
        if (flagged(dcol[j], tau)) { fcol[j] = 1; nc++; cj = j; }
    }
    i64 found = 0;
    if (nr > 0 || nc > 0) {
        st->tiles_flagged++;
        st->rows_flagged += nr;
        st->cols_flagged += nc;
        if (nr == 1 && nc == 1) {
            /* Single error: row from C^r, column from C^c (line 540).  Corrected by
             * recomputing the element (reading R6). */
            i64 i = i0 + ri, j = j0 + cj;
            double y = epilogue(alpha, ora_dot(tA, tB, K, A, lda, B, ldb, i, j), beta,
                                beta == 0.0 ? 0.0 : C0[i + j * ldc]);
            Ct[ri + cj * ldt] = y;
            if (rep_base + found < rep_cap) {
                ora_correction *e = &rep[rep_base + found];
                e->tile_m = tile_m; e->tile_n = tile_n; e->i = i; e->j = j;
                e->residual = drow[ri]; e->kind = 1; e->pad = 0;
            }
            found++;
        } else {
            /* Several flags (reading R7): candidates = (flagged rows, or all rows if none)
             * x (flagged columns, or all columns if none); each candidate is recomputed and
             * replaced when it differs from the recomputation beyond its rounding bound. */
            for (i64 jj = 0; jj < n; jj++) {
                if (nc > 0 && !fcol[jj]) continue;
                for (i64 ii = 0; ii < m; ii++) {
                    if (nr > 0 && !frow[ii]) continue;
                    i64 i = i0 + ii, j = j0 + jj;
                    double c0 = beta == 0.0 ? 0.0 : C0[i + j * ldc];
                    double y = epilogue(alpha, ora_dot(tA, tB, K, A, lda, B, ldb, i, j), beta, c0);
                    double e = 4.0 * U_ROUND * (double)(K + 3) *
                               (fabs(alpha) * ora_absdot(tA, tB, K, A, lda, B, ldb, i, j) +
                                fabs(beta) * fabs(c0));
                    if (flagged(Ct[ii + jj * ldt] - y, e)) {
                        Ct[ii + jj * ldt] = y;
                        if (rep_base + found < rep_cap) {
                            ora_correction *r = &rep[rep_base + found];
                            r->tile_m = tile_m; r->tile_n = tile_n; r->i = i; r->j = j;
                            r->residual = drow[ii]; r->kind = 2; r->pad = 0;
                        }
                        found++;
                    }
                }
            }
        }
    }
    free(ac); free(br); free(rowabs); free(colabs); free(crow); free(ccol);
    free(c0row); free(c0col); free(drow); free(dcol); free(frow); free(fcol);
    return found;
}

/* Compute one tile of the hot path: accumulator, injected flips, epilogue -> Ct. */
void ora_compute_tile(int tA, int tB, i64 K, double alpha, const double *A, i64 lda,
                      const double *B, i64 ldb, double beta, const double *C0, i64 ldc,
                      i64 i0, i64 i1, i64 j0, i64 j1, i64 nflt, const i64 *fi, const i64 *fj,
                      const int32_t *fbit, double *Ct, i64 ldt) {
    for (i64 j = j0; j < j1; j++)
        for (i64 i = i0; i < i1; i++) {
            double acc = ora_dot(tA, tB, K, A, lda, B, ldb, i, j);
            for (i64 f = 0; f < nflt; f++)
                if (fi[f] == i && fj[f] == j) acc = ora_flip(acc, fbit[f]);
            Ct[(i - i0) + (j - j0) * ldt] = epilogue(alpha, acc, beta,
                                                     beta == 0.0 ? 0.0 : C0[i + j * ldc]);
        }
}

/* The whole hot path: C := alpha op(A) op(B) + beta C with ABFT on every tile_m x tile_n
 * tile, flips (fi, fj, fbit) injected into the accumulator before the epilogue.
 * Tiles are visited column of tiles by column of tiles (tile_n outer, tile_m inner).
 * If tiles_only != NULL, only the tiles with tiles_only[tn * ntm + tm] != 0 are computed
 * (the others are left untouched) -- used to check sampled tiles at full size. */
i64 ora_abft_dgemm(int tA, int tB, i64 M, i64 N, i64 K, double alpha, const double *A,
                   i64 lda, const double *B, i64 ldb, double beta, double *C, i64 ldc,
                   i64 tile_m, i64 tile_n, i64 nflt, const i64 *fi, const i64 *fj,
                   const int32_t *fbit, ora_correction *rep, i64 rep_cap, ora_stats *st,
                   const uint8_t *tiles_only) {
    memset(st, 0, sizeof(*st));
    i64 ntm = (M + tile_m - 1) / tile_m, ntn = (N + tile_n - 1) / tile_n;
    double *Ct = malloc(sizeof(double) * (size_t)(tile_m * tile_n));
    i64 total = 0;
    for (i64 tn = 0; tn < ntn; tn++)
        for (i64 tm = 0; tm < ntm; tm++) {
            if (tiles_only && !tiles_only[tn * ntm + tm]) continue;
            i64 i0 = tm * tile_m, i1 = i0 + tile_m < M ? i0 + tile_m : M;
            i64 j0 = tn * tile_n, j1 = j0 + tile_n < N ? j0 + tile_n : N;
            ora_compute_tile(tA, tB, K, alpha, A, lda, B, ldb, beta, C, ldc, i0, i1, j0, j1,
                             nflt, fi, fj, fbit, Ct, tile_m);
            total += ora_verify_tile(tA, tB, K, alpha, A, lda, B, ldb, beta, C, ldc, i0, i1, j0,
                                     j1, tm, tn, Ct, tile_m, rep, rep_cap, total, st);
            for (i64 j = j0; j < j1; j++)
                for (i64 i = i0; i < i1; i++) C[i + j * ldc] = Ct[(i - i0) + (j - j0) * tile_m];
        }
    free(Ct);
    st->count = total;
    return total;
}
