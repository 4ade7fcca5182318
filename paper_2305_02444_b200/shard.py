"""Row-block sharding of the ABFT DGEMM over the GPUs of one node.

BASELINE.json north_star: "C is partitioned in row blocks across 1/2/4/8 GPUs ..., with
B broadcast once over NVLink via NCCL and per-shard checksums verified locally".
Rank r owns rows [r0, r1) of op(A) and of C (whole verification tiles, so a tile never
straddles two GPUs and its checksums are verified on the GPU that computed it).  The only
exchange of the step is the broadcast of op(B) from ``src``; every rank then runs the
single-GPU C-ABI call ``ftblas_dgemm`` on its shard.  torch.distributed is plumbing here
(process group + NCCL broadcast); all arithmetic runs in libftblas.so.

The GEMM call is a parameter so the host-side logic (ranges, plan slicing, broadcast,
report merging) can be exercised on CPU with the gloo backend.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TILE_M = 128
TILE_N = 128


def shard_rows(M: int, world: int, rank: int, align: int = TILE_M) -> tuple:
    """Rows [r0, r1) of op(A)/C owned by ``rank``: contiguous blocks of whole tiles."""
    tiles = -(-M // align)
    per, rem = divmod(tiles, world)
    t0 = rank * per + min(rank, rem)
    t1 = t0 + per + (1 if rank < rem else 0)
    return min(M, t0 * align), min(M, t1 * align)


def shard_plan(plan, r0: int, r1: int):
    """Restrict a global fault plan (i, j, bit) to rows [r0, r1), shifted to shard-local rows."""
    if plan is None:
        return None
    i, j, b = (np.asarray(p) for p in plan)
    sel = (i >= r0) & (i < r1)
    return (i[sel] - r0).astype(np.int64), j[sel].astype(np.int64), b[sel].astype(np.int32)


@dataclass
class ShardResult:
    rank: int
    rows: tuple
    corrections: list      # report entries with GLOBAL row indices and tile_m
    count: int
    tiles_flagged: int


def broadcast_b(B, src: int = 0, group=None):
    """Broadcast op(B) storage (a torch tensor) from ``src`` to every rank (NCCL on GPUs)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(B, src=src, group=group)
    return B


def chunk_bounds(N: int, chunks: int, align: int = TILE_N) -> list:
    """Column blocks [c0, c1) of whole verification tiles covering [0, N), as even as possible."""
    tiles = -(-N // align)
    chunks = max(1, min(chunks, tiles))
    per, rem = divmod(tiles, chunks)
    out, t0 = [], 0
    for c in range(chunks):
        t1 = t0 + per + (1 if c < rem else 0)
        out.append((min(N, t0 * align), min(N, t1 * align)))
        t0 = t1
    return out


def broadcast_chunk_bounds(m: int, N: int, sms: int = 148, waves=(1, 2, 4)) -> list:
    """Column blocks [c0, c1) of whole tiles for the overlapped op(B) broadcast of a rank with m
    rows: a geometric schedule of about 1, 2, 4 waves of 128 x 128 tiles, then the rest.  Only
    the first (one-wave) block's broadcast is exposed; each later block has the previous
    block's GEMM to arrive in, and every block is (close to) whole waves, since each block is
    one GEMM launch and a partial last wave idles SMs."""
    rows = -(-m // TILE_M)
    cols = -(-N // TILE_N)
    out, c = [], 0
    for w in waves:
        take = max(1, (w * sms) // rows)
        if c + take >= cols:
            break
        out.append((c * TILE_N, (c + take) * TILE_N))
        c += take
    out.append((c * TILE_N, N))
    return out


def b_encoding_slices(n: int, world: int) -> list:
    """Per rank, the column tiles [t0, t1) of an n-column op(B) it encodes, and its column count."""
    ntn = -(-n // TILE_N)
    out = []
    for r in range(world):
        t0, t1 = shard_rows(ntn, world, r, align=1)
        out.append((t0, t1, max(0, min(n, t1 * TILE_N) - t0 * TILE_N)))
    return out


def assemble_b_encoding(pieces, n: int, K: int, layout, out):
    """The encoding of an n-column op(B) (``layout(n, K)`` = (off_nrm, off_max, total), the
    library's section layout) assembled in ``out`` from the per-rank encodings ``pieces[r]`` of
    the column tiles ``b_encoding_slices(n, len(pieces))[r]``: section by section (the w_J rows,
    the column norms, the tile maxima), a copy only -- every value is tile- or column-local."""
    kp = layout(TILE_N, K)[0]  # one tile: the w_J section is exactly Kp doubles
    o_n, o_m, _ = layout(n, K)
    for (t0, t1, nr), piece in zip(b_encoding_slices(n, len(pieces)), pieces):
        if nr == 0:
            continue
        p_n, p_m, _ = layout(nr, K)
        out[t0 * kp: t1 * kp] = piece[: (t1 - t0) * kp]
        out[o_n + t0 * TILE_N: o_n + t0 * TILE_N + nr] = piece[p_n: p_n + nr]
        out[o_m + t0: o_m + t1] = piece[p_m: p_m + (t1 - t0)]
    return out


def shared_b_encoding(encoder, transB, n: int, K: int, B, ldb: int, *, rank: int, world: int,
                      group=None):
    """op(B)'s encoding (n columns; B: flat column-major storage of this op(B)'s columns, a torch
    tensor) computed once across the ranks: rank r encodes its slice of the column tiles
    (``encoder.encode(transB, nr, K, B_slice, ldb, piece)``, ftblas_encode_b in production) and
    the slices are all-gathered (one collective) and assembled section by section on every rank.
    ``encoder.layout(n, K)`` is the library's layout (ftblas_b_encoding_layout) and
    ``encoder.empty(len)`` allocates a float64 tensor where the collective runs."""
    import torch.distributed as dist
    slices = b_encoding_slices(n, world)
    lmax = max(encoder.layout(nr, K)[2] if nr else 0 for _, _, nr in slices) or 1
    t0, _, nr = slices[rank]
    piece = encoder.empty(lmax)
    piece.zero_()
    if nr:
        c0 = t0 * TILE_N
        view = B[c0 * ldb:] if transB in ("N", "n") else B[c0:]
        encoder.encode(transB, nr, K, view, ldb, piece)
    gathered = encoder.empty(world * lmax)
    dist.all_gather_into_tensor(gathered, piece, group=group)
    pieces = [gathered[r * lmax:(r + 1) * lmax] for r in range(world)]
    return assemble_b_encoding(pieces, n, K, encoder.layout, encoder.empty(encoder.layout(n, K)[2]))


def sharded_dgemm(gemm, transA, transB, M, N, K, alpha, A_shard, lda, B, ldb, beta, C_shard, ldc,
                  *, rank: int, world: int, src: int = 0, group=None, broadcast: bool = True,
                  chunks=1, encoder=None):
    """One sharded step on this rank.

    ``gemm(transA, transB, m, n, K, alpha, A, lda, B, ldb, beta, C, ldc, col_offset, append)``
    is the single-device call on the column block [col_offset, col_offset + n) of this rank's
    C (``ftblas.ftblas_dgemm_ex`` in production: reports in block-global column coordinates,
    ``append`` keeps the device report of the earlier blocks).  A_shard holds this rank's rows
    of op(A) (for transA='N' an (r1-r0) x K block, lda >= r1-r0; for 'T' a K x (r1-r0) block),
    C_shard its (r1-r0) x N rows of C as flat column-major storage (ld ``ldc``), B the flat
    column-major storage of B (ld ``ldb``).

    The exchange of the step is the broadcast of op(B) from ``src``.  With ``chunks`` > 1 (a
    count, or an explicit list of column blocks such as ``broadcast_chunk_bounds`` -- the same
    list on every rank, since each block is one collective) and
    transB = 'N' (column blocks of op(B) are contiguous in B) it is split into column blocks
    of whole tiles, all posted asynchronously on the communication stream; the GEMM of block
    c waits only for block c, so the broadcast of the later blocks overlaps the DMMA work of
    the earlier ones.  With an ``encoder`` (see ``shared_b_encoding``) each block's op(B)
    encoding is computed once across the ranks and passed to ``gemm`` as ``b_enc`` (else every
    rank encodes all of op(B) inside its GEMM calls).  Returns this rank's rows range.
    """
    def run(q, n, b_view, c_view, c0, append):
        kw = {}
        if encoder is not None and multi:
            kw["b_enc"] = shared_b_encoding(encoder, transB, n, K, b_view, ldb, rank=rank, world=world,
                                            group=group)
        gemm(transA, transB, m, n, K, alpha, A_shard, lda, b_view, ldb, beta, c_view, ldc, c0, append, **kw)

    r0, r1 = shard_rows(M, world, rank)
    m = r1 - r0
    multi = broadcast and world > 1
    bounds = chunks if isinstance(chunks, (list, tuple)) else chunk_bounds(N, chunks)
    if multi and len(bounds) > 1 and transB in ("N", "n"):
        import torch.distributed as dist
        works = [dist.broadcast(B[c0 * ldb: c1 * ldb], src=src, group=group, async_op=True)
                 for (c0, c1) in bounds]
        for q, (c0, c1) in enumerate(bounds):
            if rank != src:
                works[q].wait()  # NCCL: the compute stream waits for block q, the host does not
            run(q, c1 - c0, B[c0 * ldb:], C_shard[c0 * ldc:], c0, q > 0)
        if rank == src:
            for w in works:
                w.wait()
        return r0, r1
    if multi:
        broadcast_b(B, src, group)
    run(0, N, B, C_shard, 0, False)
    return r0, r1


def globalize(entries, r0: int):
    """Shard-local report entries -> global row / tile coordinates (r0 is tile aligned)."""
    out = []
    for e in entries:
        e = dict(e)
        e["i"] = int(e["i"]) + r0
        e["tile_m"] = int(e["tile_m"]) + r0 // TILE_M
        out.append(e)
    return out


def gather_reports(entries, group=None):
    """All ranks' (global) report entries, concatenated on every rank (object all-gather)."""
    import torch.distributed as dist
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return list(entries)
    bucket = [None] * dist.get_world_size(group)
    dist.all_gather_object(bucket, list(entries), group=group)
    return [e for part in bucket for e in part]
