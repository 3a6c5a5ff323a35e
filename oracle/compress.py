"""Compression pipeline (Fig. 1a-1e): prune -> CSR -> relative
column index -> quantize -> Huffman-code both streams -> row_ptr 2-tuples.

`compress_layer` returns the CDNI layer plus the pre-encoding artefacts the
tests compare against (kept mask, index matrix, token streams).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Optional

import numpy as np

from . import cdni, huffman, prune, quantize, relindex


@dataclasses.dataclass
class Compressed:
    layer: cdni.Layer
    mask: np.ndarray          # kept set (rows x cols) bool
    q: np.ndarray             # codebook index per entry (0 where pruned)
    val_tokens: np.ndarray    # token streams, rows concatenated, pads included
    gap_tokens: np.ndarray
    row_tokens: np.ndarray    # token count per stored row (weight row, or block of M' when blocked)

    def dense_q(self) -> np.ndarray:
        """prune∘quantize(W): kept weights replaced by their centres (fp32)."""
        return np.where(self.mask, self.layer.codebook[self.q], np.float32(0)).astype(np.float32)


def _freqs(tokens: np.ndarray) -> Dict[int, int]:
    if tokens.size == 0:
        return {}
    cnt = np.bincount(tokens)
    return {int(s): int(c) for s, c in enumerate(cnt) if c > 0}


def to_blocked(A: np.ndarray, bh: int, bw: int) -> np.ndarray:
    """The modified matrix M' of Alg. 2 (C-34): block (bi, bj) of A
    flattened row-major into stored row bi * (cols/bw) + bj."""
    rows, cols = A.shape
    return (A.reshape(rows // bh, bh, cols // bw, bw).transpose(0, 2, 1, 3)
            .reshape((rows // bh) * (cols // bw), bh * bw))


def compress_layer(W: np.ndarray, density: float, r: int, k: int,
                   bias: Optional[np.ndarray] = None, quantizer: str = "linear",
                   bh: int = 1, bw: Optional[int] = None) -> Compressed:
    """bh x bw != 1 x cols stores the block-contiguous container of Alg. 2:
    pruning and quantization are those of the weight matrix, relative
    indexing, Huffman coding and row_ptr run over the rows of M' (C-34)."""
    W = np.asarray(W, dtype=np.float32)
    rows, cols = W.shape
    mask = prune.prune_mask(W, density)                       # P:L55, C-10
    kept_vals = W[mask]                                       # row-major order
    if quantizer == "linear":
        cb = quantize.linear_codebook(kept_vals, r)           # P:L244-246, C-04/05
    elif quantizer == "kmeans":
        cb = quantize.lloyd_codebook(kept_vals, r)            # P:L244, C-33
    else:
        raise ValueError(f"unknown quantizer {quantizer!r}")
    q = np.zeros(W.shape, dtype=np.int64)
    q[mask] = quantize.assign(kept_vals, cb)                  # nearest centre, C-07
    bw = cols if bw is None else bw
    blocked = not (bh == 1 and bw == cols)
    if blocked and (rows % bh or cols % bw):
        raise ValueError(f"block {bh}x{bw} does not tile {rows}x{cols} (C-34)")
    smask, sq = (to_blocked(mask, bh, bw), to_blocked(q, bh, bw)) if blocked else (mask, q)
    vt, gt, row_tokens = relindex.encode_matrix(smask, sq, k)   # P:L236-243 (over M' rows, Alg. 2)
    vlen = huffman.code_lengths(_freqs(vt))                   # P:L71-72, C-14/15
    glen = huffman.code_lengths(_freqs(gt))
    vbytes, vbits, voffs = huffman.encode(vt, huffman.canonical_codes(vlen))
    gbytes, gbits, goffs = huffman.encode(gt, huffman.canonical_codes(glen))
    # row_ptr 2-tuples: start bit of each row in (val, col_ind)
    nst = smask.shape[0]
    row_start_tok = np.zeros(nst + 1, dtype=np.int64)
    np.cumsum(row_tokens, out=row_start_tok[1:])
    rp = np.zeros((nst + 1, 2), dtype=np.int64)
    for stream, offs, total in ((0, voffs, vbits), (1, goffs, gbits)):
        ext = np.append(offs, total)
        rp[:, stream] = ext[row_start_tok]
    layer = cdni.Layer(rows, cols, k, r, cb, vlen, glen, rp, vbytes, gbytes,
                       None if bias is None else np.asarray(bias, dtype=np.float32), bh, bw)
    return Compressed(layer, mask, q, vt, gt, row_tokens)
