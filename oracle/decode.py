"""Row-wise decode of an encoded layer: Algorithm 1 lines 4-8:

  <val_begin(i), col_begin(i)> <- row_ptr(i); <val_end(i), col_end(i)> <- row_ptr(i+1)
  dec_val(i) <- Huffman decoding of val between val_begin(i) and val_end(i)
  dec_col(i) <- Huffman decoding of col_ind between col_begin(i) and col_end(i)
  abs_col(i) <- prefix sum of dec_col(i)              (C-01: c = prev + g + 1)
  abs_val(i)[j] <- C[dec_val(i)[j]]

Plain bit-by-bit canonical decoding (oracle/huffman.CanonicalDecoder).  Pure
Python: use `rows=` to decode a sample of rows of a large layer.
"""
from __future__ import annotations

from typing import Iterable, List, Optional, Tuple

import numpy as np

from . import cdni, huffman, relindex


def decode_row_tokens(layer: cdni.Layer, i: int, vdec=None, gdec=None) -> List[Tuple[int, int, float]]:
    """Tokens of row i as (abs_col, val symbol, value), pads included."""
    vdec = vdec or huffman.CanonicalDecoder(layer.val_lengths)
    gdec = gdec or huffman.CanonicalDecoder(layer.gap_lengths)
    vb, gb = layer.row_ptr[i]
    ve, ge = layer.row_ptr[i + 1]
    dec_val = vdec.decode_range(layer.val_bytes, int(vb), int(ve))
    dec_col = gdec.decode_range(layer.gap_bytes, int(gb), int(ge))
    if len(dec_val) != len(dec_col):
        raise cdni.CDNIError("malformed", f"row {i}: {len(dec_val)} val vs {len(dec_col)} col tokens")
    out = []
    for c, q in relindex.decode_row(dec_val, dec_col):
        if c >= layer.stored_cols:
            raise cdni.CDNIError("malformed", f"row {i}: column {c} >= {layer.stored_cols}")
        out.append((c, q, float(layer.codebook[q])))
    return out


def decode_layer(layer: cdni.Layer, rows: Optional[Iterable[int]] = None):
    """Returns arrays (row, col, sym, val) of every token of the selected
    stored rows in stored token order, pads included.  Row and column are the
    stored matrix's: for a blocked layer (Alg. 2, C-34) the block index and
    the position inside the flattened block (cdni.Layer.unflatten maps them
    back to the weight matrix)."""
    vdec = huffman.CanonicalDecoder(layer.val_lengths)
    gdec = huffman.CanonicalDecoder(layer.gap_lengths)
    R, C, S, V = [], [], [], []
    for i in (range(layer.stored_rows) if rows is None else rows):
        for c, q, v in decode_row_tokens(layer, i, vdec, gdec):
            R.append(i); C.append(c); S.append(q); V.append(v)
    return (np.array(R, dtype=np.int64), np.array(C, dtype=np.int64),
            np.array(S, dtype=np.int64), np.array(V, dtype=np.float32))


def decode_dense(layer: cdni.Layer) -> np.ndarray:
    """decompress: dense fp32 W_q with W_q[row, c] = C[sym] for sym != 0."""
    r, c, s, v = decode_layer(layer)
    W = np.zeros((layer.rows, layer.cols), dtype=np.float32)
    real = s != 0
    wr, wc = layer.unflatten(r[real], c[real])   # Alg. 2 l.10-13 for a blocked layer
    W[wr, wc] = v[real]
    return W
