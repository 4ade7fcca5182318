/*
 * ftblas.h -- C ABI of the B200-native fault-tolerant DGEMM (libftblas.so).
 *
 * The operation (PAPER.md = the FT-BLAS paper text, /root/reference/PAPER.md):
 *   C := alpha * op(A) * op(B) + beta * C,   op(X) = X or X^T,
 * the Level-3 BLAS DGEMM (PAPER.md "Implementation of DGEMM", line 823; the
 * op() convention as stated for DGEMV, line 799), in binary64, column-major
 * BLAS storage: element (r, c) of a matrix with leading dimension ld lives at
 * p[r + c*ld].
 *
 * Fault tolerance (ftblas_dgemm only): Huang-Abraham algorithm-based fault
 * tolerance (section II.A; fusion: section V.B, line
 * 558): checksums A^c = [A; e^T A] and B^r = [B, B e] are encoded per
 * verification tile (FTBLAS_TILE_M x FTBLAS_TILE_N block of C), the checksum
 * row e^T C = (e^T A) B and column C e = A (B e) of the product are formed on
 * the FP64 tensor cores (ftblas_set_checksum_mode: as two checksum GEMMs
 * before the main GEMM -- the default -- or accumulated in the same mainloop
 * as the MMA), and the epilogue of the GEMM kernel compares them with the
 * computed tile, flags any row/column whose difference "exceeds the round-off
 * threshold" (line 517), locates the erroneous element at the intersection of
 * the flagged row and column (line 540) and corrects it before C is stored.
 * The detection threshold, the multi-flag rule and the correction rule are the
 * readings R4-R7 of DESIGN.md section 3.
 *
 * Conventions for every entry point:
 *   - A, B, C are DEVICE pointers (cudaMalloc'ed or torch CUDA storage) on the
 *     current CUDA device, except in ftblas_dgemm_host where they are HOST
 *     pointers.  The caller owns all memory; the library owns only its
 *     internal workspace and report buffers (freed by ftblas_release).
 *   - transA/transB: 'N'/'n' (op(X) = X) or 'T'/'t'/'C'/'c' (op(X) = X^T).
 *   - op(A) is M x K: A is M x K (lda >= max(1,M)) for 'N', K x M (lda >= max(1,K)) for 'T'.
 *     op(B) is K x N: B is K x N (ldb >= max(1,K)) for 'N', N x K (ldb >= max(1,N)) for 'T'.
 *     C is M x N, ldc >= max(1,M).
 *   - beta == 0: C is not read on input (may hold NaN); alpha == 0: A and B are
 *     not read.  M == 0 or N == 0: no-op.
 *   - Work is enqueued on the stream set by ftblas_set_stream (default: the
 *     legacy default stream).  Calls are asynchronous unless they take a
 *     non-NULL report (see below).
 *   - Return value: 0 on success; -p if argument p (1-based, BLAS xerbla
 *     numbering) is invalid; FTBLAS_ERR_CUDA (1000) on a CUDA error, with the
 *     message available from ftblas_last_error().  Nothing is launched when an
 *     argument is invalid.
 *   - Not thread-safe: one host thread drives the library per process (one
 *     process per GPU).
 */
#ifndef FTBLAS_H
#define FTBLAS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FTBLAS_TILE_M 128 /* verification tile rows (one CTA tile of C) */
#define FTBLAS_TILE_N 128 /* verification tile columns */
#define FTBLAS_ERR_CUDA 1000

/* One corrected element of C.  Field order/size is ABI (48 bytes). */
typedef struct ftblas_correction {
    int64_t tile_m;   /* verification tile row index    (= i / FTBLAS_TILE_M) */
    int64_t tile_n;   /* verification tile column index (= j / FTBLAS_TILE_N) */
    int64_t i, j;     /* 0-based row / column of the corrected element of C */
    double residual;  /* row-checksum residual d_i of row i (sum_j C_ij - (C e)_i) */
    int32_t kind;     /* 1: exactly one row and one column flagged in the tile -> their
                         intersection (Huang-Abraham location);
                         2: several flags -> candidate recomputation (reading R7) */
    int32_t pad;
} ftblas_correction;

/* Error report of one ftblas_dgemm call.  entries/capacity are supplied by the
 * caller (HOST memory, may be NULL/0); the library fills the rest.  Entries are
 * unordered (tiles run concurrently); sort by (tile_n, tile_m, j, i) to compare. */
typedef struct ftblas_err_report {
    ftblas_correction *entries; /* in: host array of `capacity` records (caller-owned) */
    int64_t capacity;           /* in */
    int64_t count;              /* out: corrections made (may exceed capacity: truncated) */
    int64_t tiles_flagged;      /* out: tiles with >= 1 flagged row or column */
    int64_t rows_flagged;       /* out: flagged rows summed over tiles */
    int64_t cols_flagged;       /* out: flagged columns summed over tiles */
} ftblas_err_report;

/* ABFT DGEMM (the hot path).  Device pointers.  If err_report != NULL the call
 * synchronizes the stream and fills *err_report; if NULL it is fully
 * asynchronous and the report can be read later with ftblas_report_fetch.
 * Corrections are applied to C in both cases.  Faults from the plan installed
 * by ftblas_set_fault_plan are injected into the accumulator before
 * verification (test/benchmark harness; empty plan = no injection). */
int ftblas_dgemm(char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha,
                 const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                 double *C, int64_t ldc, ftblas_err_report *err_report);

/* ftblas_dgemm on a block of a larger problem (sharded / chunked callers).  The call's C
 * is the block of the caller's C starting at (row_offset, col_offset), both >= 0 and
 * multiples of FTBLAS_TILE_M / FTBLAS_TILE_N (else -14 / -15).  Report entries (i, j,
 * tile_m, tile_n) are given in the caller's coordinates, and the fault plan of
 * ftblas_set_fault_plan is read in the caller's coordinates (entries outside the block are
 * ignored).  flags: FTBLAS_REPORT_APPEND -- append to the device report instead of resetting
 * it (clear it with ftblas_report_reset); FTBLAS_REUSE_A_ENCODE -- the caller guarantees that
 * op(A) (same pointer, lda, M, K, transA) is unchanged since the previous FT call, whose A
 * checksum encoding is then reused if still cached (column blocks of one product); other
 * FTBLAS_B_ENCODED -- see ftblas_set_b_encoding; other bits -> -16. */
#define FTBLAS_REPORT_APPEND 1
#define FTBLAS_REUSE_A_ENCODE 2
#define FTBLAS_B_ENCODED 4 /* op(B)'s encoding comes from ftblas_set_b_encoding (see below) */
int ftblas_dgemm_ex(char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha,
                    const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                    double *C, int64_t ldc, int64_t row_offset, int64_t col_offset, int32_t flags,
                    ftblas_err_report *err_report);

/* Shared op(B) encoding (sharded products: the B-side encoding -- w_J = op(B) e_J of every
 * column tile J, the column 1-norms and the tile maxima of reading R4 --
 * depends on op(B) only, so the ranks of a row-sharded product can each encode a slice of the
 * column tiles and exchange the slices instead of every rank encoding all of op(B); PAPER.md
 * section V.B: the packed B is shared and its checksum reduced once).
 *   ftblas_b_encoding_layout: the encoding of an op(B) with N columns and inner dimension K is
 *     *total doubles: [0, *off_nrm) the ceil(N/128) vectors w_J of Kp = max(32, ceil(K/32) 32)
 *     doubles each (zero for k >= K), [*off_nrm, *off_nrm + N) the column norms,
 *     [*off_max, *off_max + ceil(N/128)) the tile maxima.  Columns [c0, c1) of whole tiles of an
 *     encoding are the encoding of those columns, section by section.  Returns 0, -1 / -2 for
 *     N / K < 0.  ftblas_b_encoding_len returns *total (or -1).
 *   ftblas_encode_b: op(B) (K x N; B, ldb as for ftblas_dgemm; device pointers) -> enc (caller-
 *     owned device buffer of ftblas_b_encoding_len(N, K) doubles), stream-ordered on the library
 *     stream.  Returns 0; -1 transB, -2 N < 0, -3 K < 0, -4 B NULL, -5 ldb, -6 enc NULL;
 *     FTBLAS_ERR_CUDA.
 *   ftblas_set_b_encoding: install enc (an encoding of an N x K op(B); NULL uninstalls) for
 *     ftblas_dgemm_ex calls with FTBLAS_B_ENCODED, which use it in place of encoding their op(B)
 *     (their N and K must match, else -16).  The caller keeps enc alive and unchanged while such
 *     calls are in flight. */
int64_t ftblas_b_encoding_len(int64_t N, int64_t K);
int ftblas_b_encoding_layout(int64_t N, int64_t K, int64_t *off_nrm, int64_t *off_max, int64_t *total);
int ftblas_encode_b(char transB, int64_t N, int64_t K, const double *B, int64_t ldb, double *enc);
int ftblas_set_b_encoding(const double *enc, int64_t N, int64_t K);

/* Clear the device report (stream-ordered; for FTBLAS_REPORT_APPEND sequences). */
int ftblas_report_reset(void);

/* The same DGEMM without fault tolerance (same tiles and mainloop, no checksums,
 * no verification, no injection): the baseline for the FT overhead. */
int ftblas_dgemm_noft(char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha,
                      const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                      double *C, int64_t ldc);

/* ftblas_dgemm on HOST buffers (end-to-end path): copies op(A), op(B) and C
 * (if beta != 0) host->device, runs the ABFT DGEMM, copies C device->host and
 * synchronizes.  Pipelined over blocks of whole 128 x 128 tiles (uploads, block
 * GEMMs and downloads on three streams); for deep K the first row block runs in
 * k parts accumulated with beta = 1 (the fault plan applies to the last parts, so
 * the report equals the one-call report; those blocks' C can differ from
 * ftblas_dgemm's in rounding order, within the usual bound).  err_report as
 * above (may be NULL).  Pinned host memory gives the full PCIe bandwidth;
 * pageable memory works but is slower. */
int ftblas_dgemm_host(char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha,
                      const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                      double *C, int64_t ldc, ftblas_err_report *err_report);

/* Read the report of the most recent ftblas_dgemm call (synchronizes the stream). */
int ftblas_report_fetch(ftblas_err_report *err_report);

/* Install a fault-injection plan for subsequent ftblas_dgemm calls: n single-bit
 * flips, flip k toggles bit bit[k] (0..63) of the accumulator of element
 * (i[k], j[k]) of C (0-based, 0 <= i < M, 0 <= j < N of the call) before the
 * epilogue.  Host arrays, copied.  n == 0 clears the plan.  Plans are matched
 * against the M x N of each call; entries outside it are ignored.  At most
 * FTBLAS_MAX_FLIPS_PER_TILE flips may fall into one FTBLAS_TILE_M x FTBLAS_TILE_N
 * tile (the persistent kernel keeps a tile's hits in a 4-entry shared-memory list); a plan
 * with more returns -1 and leaves the installed plan unchanged.  Returns -1 for
 * n < 0, -2 for NULL arrays or negative coordinates, -4 for a bit outside 0..63. */
#define FTBLAS_MAX_FLIPS_PER_TILE 4
int ftblas_set_fault_plan(int64_t n, const int64_t *i, const int64_t *j, const int32_t *bit);

/* Where the checksum row/column of C (the border of C^f = A^c B^r, PAPER.md
 * line 516) is computed by subsequent ftblas_dgemm calls:
 *   FTBLAS_CHECKSUM_GEMM  (default): R = op(A) (B e_J) for every column tile J and
 *       S = (e_I^T A) op(B) for every row tile I as two DMMA GEMMs (M x ceil(N/128)
 *       and N x ceil(M/128)) before the main GEMM; the main kernel's mainloop is
 *       the plain one and its epilogue verifies against R, S.
 *   FTBLAS_CHECKSUM_FUSED: accumulated in the main kernel's mainloop from the
 *       operand fragments of the MMA (DFMA next to the DMMA stream).
 * Both give the same verification, reports and corrections up to rounding of
 * the checksum (covered by the threshold, R4).  Returns 0, or -1 for
 * an unknown mode. */
#define FTBLAS_CHECKSUM_GEMM 0
#define FTBLAS_CHECKSUM_FUSED 1
int ftblas_set_checksum_mode(int mode);
int ftblas_get_checksum_mode(void);

/* CTA tiling of the GEMM kernels (a performance choice; results, reports and the 128 x 128
 * verification tile are the same):
 *   FTBLAS_TILES_AUTO (default): for K <= 2048 FTBLAS_TILES_WS (ftblas_dgemm with at least
 *       one tile per SM) or FTBLAS_TILES_PAIR (ftblas_dgemm_noft, fewer tiles), else
 *       FTBLAS_TILES_FULL;
 *   FTBLAS_TILES_FULL: one CTA per 128 x 128 tile (8 MMA warps of 64 x 32, one CTA per SM);
 *   FTBLAS_TILES_PAIR: two CTAs per tile, each a 128 x 64 half (8 MMA warps of 32 x 32, two
 *       CTAs per SM so one CTA's epilogue overlaps another's mainloop); for ftblas_dgemm the halves form a
 *       thread-block cluster and exchange their row sums through distributed shared memory.
 *   FTBLAS_TILES_WS: persistent kernel, one CTA per SM walking its tiles: 8 MMA warps
 *       (TMA-fed DMMA mainloop; at the end of a tile they form out = alpha acc + beta C0 and
 *       the checksum sums in registers, with C0 and out passed through tensor memory, and
 *       verify the tile), 4 epilogue warps (C0 in, verified tile out, location) overlapping the
 *       next tile's mainloop, 1 TMA producer thread.
 * The fused checksum mode always uses FTBLAS_TILES_FULL.  Returns 0, or -1 for an unknown
 * policy. */
#define FTBLAS_TILES_AUTO 0
#define FTBLAS_TILES_FULL 1
#define FTBLAS_TILES_PAIR 2
#define FTBLAS_TILES_WS 3
int ftblas_set_tile_policy(int policy);
int ftblas_get_tile_policy(void);

/* Stream for subsequent calls (a cudaStream_t passed as void*; NULL = default stream). */
int ftblas_set_stream(void *stream);

/* Number of kernels the library launched since load (for launch accounting). */
int64_t ftblas_launch_count(void);

/* Per-kernel device timing (for roofline accounting in bench.py).  enable != 0:
 * subsequent ftblas_dgemm / ftblas_dgemm_noft calls record CUDA events on the
 * library stream around each kernel launch; enable == 0 stops recording.
 * ftblas_profile_read synchronizes, returns the summed device milliseconds of
 * the checksum stage (encode kernel + checksum GEMMs in FTBLAS_CHECKSUM_GEMM
 * mode) and of the main GEMM kernel and the number of GEMM calls
 * recorded since the last read, and clears the record.  Any output pointer may
 * be NULL. */
int ftblas_profile(int enable);
int ftblas_profile_read(double *encode_ms, double *gemm_ms, int64_t *gemm_launches);

/* Verification tile shape (FTBLAS_TILE_M, FTBLAS_TILE_N). */
void ftblas_tile_shape(int32_t *tile_m, int32_t *tile_n);

/* Message of the last error (static storage, never NULL). */
const char *ftblas_last_error(void);

/* Free the library's device workspace (it is re-allocated on demand). */
int ftblas_release(void);

#ifdef __cplusplus
}
#endif
#endif /* FTBLAS_H */
