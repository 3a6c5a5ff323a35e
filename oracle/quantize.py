"""Weight sharing / quantization: "If r bits are used for
quantization, we use at most (2^r - 1) distinct non-zero values along with 0
in quantized values, and each entry of the val vector is a r bit index to the
corresponding cluster centre. The cluster centre values are stored in the
codebook."

Readings:
  C-04 (Reading A): the codebook has 2^r entries; index 0 is the value 0.0 and
       is reserved for padding entries; indices 1..2^r-1 are the non-zero
       centres.  Real weights are never assigned index 0.
  C-05: the centres follow BASELINE.json config C1: "32 centroids linearly
       initialised over [min,max] of surviving weights, nearest-centroid
       assignment" -- no Lloyd refinement.  Grid computed in binary64, stored
       as fp32: C[j] = fp32(lo + (hi - lo) * (j - 1) / (2^r - 2)), j >= 1.
  C-07: assignment = argmin_{j>=1} |w - C[j]| in binary64 over the fp32 centres,
       ties to the smaller j.  lo == hi gives duplicate centres; the smallest
       j wins.  No kept weights -> lo = hi = 0.

Variant: 1-D Lloyd k-means refinement of the
same 2^r - 1 centres ("similar valued non-zero entries of val are clustered",
P:L244).  Reading C-33: start from the C-05 grid; per iteration assign every
kept weight to its nearest centre in binary64 (ties to the smaller index),
then move each non-empty centre to the binary64 mean of its weights, summed
in row-major order; an empty centre stays where it is; stop after 50
iterations or when no centre moved by more than 1e-7 * max(|lo|, |hi|).  The
stored codebook is fp32(centre); the final assignment is C-07 over the stored
fp32 centres.
"""
from __future__ import annotations

import numpy as np


def linear_codebook(kept: np.ndarray, r: int) -> np.ndarray:
    """fp32 codebook of 2^r entries, entry 0 == 0.0 (C-04, C-05)."""
    n = 1 << r
    cb = np.zeros(n, dtype=np.float32)
    if kept.size == 0:
        return cb
    lo = float(np.min(kept.astype(np.float64)))
    hi = float(np.max(kept.astype(np.float64)))
    denom = float(n - 2) if n > 2 else 1.0
    for j in range(1, n):
        cb[j] = np.float32(lo + (hi - lo) * (j - 1) / denom)
    return cb


def lloyd_codebook(kept: np.ndarray, r: int, iters: int = 50, tol: float = 1e-7) -> np.ndarray:
    """fp32 codebook of 2^r entries, entry 0 == 0.0, centres refined by 1-D
    Lloyd iterations from the linear grid (C-33)."""
    n = 1 << r
    cb = np.zeros(n, dtype=np.float32)
    if kept.size == 0:
        return cb
    v = kept.astype(np.float64)
    lo, hi = float(np.min(v)), float(np.max(v))
    denom = float(n - 2) if n > 2 else 1.0
    c = np.array([lo + (hi - lo) * (j - 1) / denom for j in range(1, n)], dtype=np.float64)
    eps = tol * max(abs(lo), abs(hi))
    for _ in range(iters):
        # nearest centre, binary64, ties -> smaller index (argmin returns the first)
        idx = np.empty(v.size, dtype=np.int64)
        for s in range(0, v.size, 1 << 20):
            idx[s:s + (1 << 20)] = np.argmin(np.abs(v[s:s + (1 << 20), None] - c[None, :]), axis=1)
        # bincount adds the weights one by one in array (row-major) order
        sums = np.bincount(idx, weights=v, minlength=c.size)
        cnt = np.bincount(idx, minlength=c.size)
        new = c.copy()
        nz = cnt > 0
        new[nz] = sums[nz] / cnt[nz]
        moved = float(np.max(np.abs(new - c)))
        c = new
        if moved <= eps:
            break
    cb[1:] = c.astype(np.float32)
    return cb


def assign(values: np.ndarray, codebook: np.ndarray, chunk: int = 1 << 20) -> np.ndarray:
    """Nearest non-zero centre, binary64 distances, ties -> smaller index
    (np.argmin returns the first minimum).  Returns uint8 indices in 1..2^r-1."""
    cand = codebook[1:].astype(np.float64)
    v = values.astype(np.float64)
    out = np.empty(v.size, dtype=np.int64)
    for s in range(0, v.size, chunk):
        d = np.abs(v[s:s + chunk, None] - cand[None, :])
        out[s:s + chunk] = np.argmin(d, axis=1) + 1
    return out.astype(np.uint16 if codebook.size > 256 else np.uint8)
