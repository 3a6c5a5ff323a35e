"""CSR with relative column index:

  "if val(i) is the first non-zero entry of any particular row, then
   col_ind(i) is set to the corresponding column number; else col_ind(i) is
   set to the number of columns between the current non-zero and the last
   non-zero entry of the row.  If more than 2^k zeros appear before a non-zero
   entry, we add a zero in both the val and the col_ind vectors."
  Example (k=2): "Since the first non-zero column of second row exceeds 4, we
   pad a zero at the fourth location of both val and col_ind."

Readings:
  C-01 zero-gap: g = number of columns strictly between this entry and the
       previous one (previous = -1 at row start); decode c = prev + g + 1.
  C-02 pad when g > 2^k - 1; a pad is (val index 0, gap 2^k - 1) and advances
       the column by 2^k; repeat until the residual gap fits.
  C-03 the first entry of a row is padded the same way.
A token is the pair (val symbol, gap symbol).  Pads are tokens with val 0.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def encode_row(cols: List[int], vals: List[int], k: int) -> Tuple[List[int], List[int]]:
    """Pure-Python definition for one row (small cases and pins)."""
    cap = (1 << k) - 1
    out_v: List[int] = []
    out_g: List[int] = []
    prev = -1
    for c, q in zip(cols, vals):
        g = c - prev - 1
        while g > cap:
            out_v.append(0)
            out_g.append(cap)
            prev += 1 << k
            g -= 1 << k
        out_v.append(q)
        out_g.append(g)
        prev = c
    return out_v, out_g


def decode_row(val_syms: List[int], gap_syms: List[int]) -> List[Tuple[int, int]]:
    """Alg. 1 line 7 "abs_col <- prefix sum of dec_col" under C-01:
    c_j = c_{j-1} + g_j + 1, c_{-1} = -1.  Returns (col, val symbol) per token,
    pads included."""
    out = []
    prev = -1
    for q, g in zip(val_syms, gap_syms):
        c = prev + g + 1
        out.append((c, q))
        prev = c
    return out


def encode_matrix(mask: np.ndarray, q: np.ndarray, k: int):
    """Relative-index every row of a pruned, quantized matrix.

    mask: bool (rows x cols) kept set; q: integer index matrix (same shape,
    meaningful where mask).  Returns (val_tokens, gap_tokens, row_tokens) with
    rows concatenated in order and row_tokens[i] = token count of row i.

    Vectorised form of encode_row: an entry with zero-gap g is preceded by
    g // 2^k pads and carries residual gap g % 2^k (the while-loop of C-02
    subtracts 2^k exactly g // 2^k times)."""
    rows, cols = mask.shape
    rr, cc = np.nonzero(mask)                       # row-major order
    qv = q[rr, cc].astype(np.int64)
    # previous column in the same row (-1 at each row start)
    prev = np.empty_like(cc)
    prev[1:] = cc[:-1]
    first = np.ones(cc.size, dtype=bool)
    first[1:] = rr[1:] != rr[:-1]
    prev[first] = -1
    g = cc - prev - 1
    npad = g >> k
    resid = g & ((1 << k) - 1)
    cap = (1 << k) - 1
    per_entry = npad + 1
    total = int(per_entry.sum())
    val_t = np.zeros(total, dtype=np.int64)
    gap_t = np.full(total, cap, dtype=np.int64)
    ends = np.cumsum(per_entry) - 1                # position of each real token
    val_t[ends] = qv
    gap_t[ends] = resid
    row_tokens = np.bincount(rr, weights=per_entry, minlength=rows).astype(np.int64)
    return val_t, gap_t, row_tokens
