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


def sharded_dgemm(gemm, transA, transB, M, N, K, alpha, A_shard, lda, B, ldb, beta, C_shard, ldc,
                  *, rank: int, world: int, src: int = 0, group=None, broadcast: bool = True,
                  report=None):
    """One sharded step on this rank.

    ``gemm(transA, transB, m, N, K, alpha, A, lda, B, ldb, beta, C, ldc, report)`` is the
    single-device call (``ftblas.ftblas_dgemm`` in production).  A_shard holds this rank's
    rows of op(A) (for transA='N' an (r1-r0) x K block, lda >= r1-r0; for 'T' a K x (r1-r0)
    block), C_shard its (r1-r0) x N rows of C.  Returns the local rows range.
    """
    r0, r1 = shard_rows(M, world, rank)
    if broadcast:
        broadcast_b(B, src, group)
    m = r1 - r0
    gemm(transA, transB, m, N, K, alpha, A_shard, lda, B, ldb, beta, C_shard, ldc, report)
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
