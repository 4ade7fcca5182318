"""Helpers shared by the GPU tests: device copies of column-major numpy storage and
comparison utilities.  No arithmetic of the method lives here."""
from __future__ import annotations

import numpy as np

import synthetic as syn

U = 2.0 ** -53


def full_buffer(x: np.ndarray) -> np.ndarray:
    """The (ld x cols) Fortran buffer behind a possibly padded column-major view."""
    b = syn.base_of(x)
    if b.ndim == 1:
        return x
    return b


def to_dev(x: np.ndarray, offset: int = 0):
    """Copy column-major storage (incl. ld padding) to a CUDA tensor; returns (tensor, ptr).
    ``offset`` elements of slack before the data produce a misaligned pointer."""
    import torch
    full = np.asfortranarray(full_buffer(x))
    flat = full.reshape(-1, order="F")
    t = torch.zeros(flat.size + offset, dtype=torch.float64, device="cuda")
    t[offset:].copy_(torch.from_numpy(flat.copy()))
    return t, t.data_ptr() + 8 * offset


def from_dev(t, like: np.ndarray, offset: int = 0) -> np.ndarray:
    full = full_buffer(like)
    host = t[offset:].cpu().numpy().reshape(full.shape, order="F")
    return host[: like.shape[0], : like.shape[1]]


def gemm_bound(K, alpha, beta, absAB, absC0):
    """Elementwise tolerance of BASELINE north_star: 4 K 2^-53 (|A||B|)_ij, extended to the
    alpha/beta epilogue: 4 (K+2) u (|alpha| (|A||B|)_ij + |beta| |C0_ij|)."""
    return 4.0 * (K + 2) * U * (abs(alpha) * absAB + abs(beta) * absC0)


def report_key(entries):
    return sorted((int(e["tile_m"]), int(e["tile_n"]), int(e["i"]), int(e["j"]), int(e["kind"]))
                  for e in entries)
