"""Magnitude pruning ("remove all connections whose weights are lower
than fixed threshold"; "Pruning makes weight matrix W sparse").

Reading C-10: BASELINE.json configs state a *density* d, so the kept set is
an exact count n_keep = floor(d * n + 0.5) of the largest |w| over the whole
layer, ties at the threshold broken toward the lower row-major linear index
(i.e. the first n_keep entries of a stable sort of -|W| in row-major order).
"""
from __future__ import annotations

import numpy as np


def n_keep_for(density: float, n: int) -> int:
    """floor(d*n + 0.5), computed in binary64 like every consumer of the
    configs (C-10)."""
    return int(np.floor(float(density) * float(n) + 0.5))


def prune_mask_sorted(W: np.ndarray, density: float) -> np.ndarray:
    """Definition of the kept set: stable sort of -|W| (row-major), keep first
    n_keep.  O(n log n); used for small matrices and as the pin of the fast
    form below."""
    flat = np.abs(W.astype(np.float32)).ravel()
    n_keep = n_keep_for(density, flat.size)
    order = np.argsort(-flat.astype(np.float64), kind="stable")
    mask = np.zeros(flat.size, dtype=bool)
    mask[order[:n_keep]] = True
    return mask.reshape(W.shape)


def prune_mask(W: np.ndarray, density: float) -> np.ndarray:
    """Same set as prune_mask_sorted, computed by threshold:
    t = the n_keep-th largest |w|; keep every |w| > t, then the first
    n_keep - count(|w| > t) entries with |w| == t in row-major order."""
    flat = np.abs(W.astype(np.float32)).ravel()
    n = flat.size
    n_keep = n_keep_for(density, n)
    mask = np.zeros(n, dtype=bool)
    if n_keep <= 0:
        return mask.reshape(W.shape)
    if n_keep >= n:
        mask[:] = True
        return mask.reshape(W.shape)
    t = np.partition(flat, n - n_keep)[n - n_keep]   # n_keep-th largest value
    above = flat > t
    need = n_keep - int(above.sum())
    eq_idx = np.flatnonzero(flat == t)[:need]
    mask = above
    mask[eq_idx] = True
    return mask.reshape(W.shape)
