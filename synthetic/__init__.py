"""Seeded synthetic workloads shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no products, no checksums, no
thresholds): only random draws, BLAS storage shapes and the fault-plan sampler.
It is the one piece of code both sides may import (the oracle and the CUDA
path share nothing else).

Workloads follow BASELINE.json ``configs`` (the paper's own benchmarks use
random square matrices "ranging from 2048^2 to 10240^2", §VI.A, and
inject errors into "an element of matrix C ... randomly selected", §VI.C).
All matrices are column-major (Fortran order) numpy float64 arrays, exactly
the storage a BLAS caller hands to ``ftblas_dgemm``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# Fault model of BASELINE.json: single-bit flips with bit index uniform in [40, 62]
# (mantissa bits 40..51 and exponent bits 52..62 of an IEEE-754 binary64).
BIT_LO, BIT_HI = 40, 62

# Verification tile of the method (one CTA tile of C); see DESIGN.md §2.
TILE_M, TILE_N = 128, 128


@dataclass
class Workload:
    name: str
    M: int
    N: int
    K: int
    transA: str = "N"
    transB: str = "N"
    alpha: float = 1.0
    beta: float = 0.0
    dist: str = "uniform"   # "uniform" (U[-1,1]) or "normal" (N(0,1)) for A and B
    c_init: bool = False    # C drawn U[-1,1] (else zeros; beta==0 never reads C)
    seed: int = 0
    n_flips: int = 0
    shard_gpus: tuple = (1,)
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def flops(self) -> float:
        return 2.0 * self.M * self.N * self.K


# BASELINE.json configs[0..4], restated as data.
CONFIGS = [
    Workload("c0_256_ft", 256, 256, 256, "N", "N", 1.0, 0.0, "uniform", False, 0, 4,
             note="4 flips, all must be detected/located/corrected"),
    Workload("c1_4096_tn", 4096, 4096, 4096, "N", "T", 1.5, -0.5, "uniform", True, 1, 100,
             note="fault-free run plus 100 flips over distinct tiles"),
    Workload("c2_rankk_16384x256", 16384, 16384, 256, "N", "N", -1.0, 1.0, "uniform", True, 2, 32,
             shard_gpus=(1, 8), note="LU trailing-update shape, small K"),
    Workload("c3_16384_sharded", 16384, 16384, 16384, "N", "N", 1.0, 0.0, "normal", False, 3, 500,
             shard_gpus=(1, 2, 4, 8), note="row-block sharded C, B broadcast"),
    Workload("c4_32768x16384_8gpu", 32768, 32768, 16384, "N", "N", 1.0, 1.0, "uniform", True, 4, 300,
             shard_gpus=(8,), note="8-GPU row-block shard, sustained injection"),
]
CONFIG_BY_NAME = {w.name: w for w in CONFIGS}


def stored_shape(op_rows: int, op_cols: int, trans: str) -> tuple:
    """Shape of the stored (column-major) array whose op() is op_rows x op_cols."""
    return (op_rows, op_cols) if trans.upper() == "N" else (op_cols, op_rows)


def _draw(rng: np.random.Generator, rows: int, cols: int, dist: str, ld: int | None = None) -> np.ndarray:
    ld = rows if ld is None else ld
    if dist == "uniform":
        flat = rng.uniform(-1.0, 1.0, size=ld * cols)
    elif dist == "normal":
        flat = rng.standard_normal(size=ld * cols)
    elif dist == "int":          # small integers: products and sums are exact in binary64
        flat = rng.integers(-8, 9, size=ld * cols).astype(np.float64)
    else:
        raise ValueError(dist)
    full = flat.reshape((ld, cols), order="F")
    return full[:rows, :] if ld != rows else full


def make_inputs(w: Workload, *, pad: int = 0, dist: str | None = None) -> dict:
    """Draw op(A) (M x K), op(B) (K x N) and C (M x N) storage for workload ``w``.

    Draw order from ``default_rng(seed)``: A, then B, then C.  ``pad`` adds
    that many rows of leading-dimension padding (ld = rows + pad) to exercise
    lda/ldb/ldc > rows.
    """
    rng = np.random.default_rng(w.seed)
    d = dist or w.dist
    ar, ac = stored_shape(w.M, w.K, w.transA)
    br, bc = stored_shape(w.K, w.N, w.transB)
    A = _draw(rng, ar, ac, d, ar + pad)
    B = _draw(rng, br, bc, d, br + pad)
    if w.c_init:
        C = _draw(rng, w.M, w.N, "uniform" if d != "int" else "int", w.M + pad)
    else:
        C = np.zeros((w.M + pad, w.N), order="F")[: w.M, :]
    return dict(A=A, B=B, C=C, lda=max(1, ar + pad), ldb=max(1, br + pad), ldc=max(1, w.M + pad))


def base_of(x: np.ndarray) -> np.ndarray:
    """The full (ld x cols) column-major buffer behind a (possibly padded) matrix view."""
    own = x.base
    if own is None or x.ndim != 2:
        return x
    ld = x.strides[1] // 8 if x.shape[1] > 1 else x.shape[0]
    if own.ndim == 1 and ld > 0 and own.size == ld * x.shape[1]:
        return own.reshape((ld, x.shape[1]), order="F")
    if own.ndim == 2 and own.shape[1] == x.shape[1]:
        return own
    return x


def fault_plan(M: int, N: int, n: int, seed: int, *, tile_m: int = TILE_M, tile_n: int = TILE_N,
               distinct_tiles: bool = True, bit_lo: int = BIT_LO, bit_hi: int = BIT_HI):
    """Seeded single-bit-flip plan over the M x N output: arrays (i, j, bit), int64/int32.

    (i, j) uniform over C; with ``distinct_tiles`` a draw landing in an already
    used verification tile is redrawn (the paper's error model corrects "one
    error in each verification interval", §II.A).
    Elements are always distinct.  Sorted by (tile_n, tile_m, j, i) so the
    order is canonical.
    """
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x5EED_F1]))
    n_tiles = -(-M // tile_m) * -(-N // tile_n)
    if distinct_tiles and n > n_tiles:
        raise ValueError(f"{n} flips cannot occupy distinct tiles ({n_tiles} tiles)")
    if n > M * N:
        raise ValueError("more flips than elements")
    used_tiles, used_elems = set(), set()
    out_i, out_j, out_b = [], [], []
    while len(out_i) < n:
        i = int(rng.integers(0, M))
        j = int(rng.integers(0, N))
        b = int(rng.integers(bit_lo, bit_hi + 1))
        t = (i // tile_m, j // tile_n)
        if (i, j) in used_elems or (distinct_tiles and t in used_tiles):
            continue
        used_elems.add((i, j))
        used_tiles.add(t)
        out_i.append(i)
        out_j.append(j)
        out_b.append(b)
    order = sorted(range(n), key=lambda q: (out_j[q] // tile_n, out_i[q] // tile_m, out_j[q], out_i[q]))
    return (np.array([out_i[q] for q in order], dtype=np.int64),
            np.array([out_j[q] for q in order], dtype=np.int64),
            np.array([out_b[q] for q in order], dtype=np.int32))
