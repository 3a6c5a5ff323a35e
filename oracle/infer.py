"""Dense-definition inference (fp64) for FC and CONV layers.

FC (Eq. 1-2):  b = W a + v,  b_i = sum_j W_ij a_j + v_i, with W the
decoded (pruned, quantized) matrix.  Alg. 1 computes exactly this product row by
row (reading C-31), so the oracle is the plain definition in fp64.

CONV: "the dot products between the filters and local regions of
the input can be formulated as a matrix-matrix multiplication, by flattening
out the local regions of the input to individual columns and the layer weights
to rows".  K order is (r, s, c), channel fastest, per group (C-18).  The
product runs CONV on bf16 tensor cores with fp32 accumulation (config C4), so
the oracle rounds the input and the weights to bf16 (RNE) first and then does
the product in fp64 (C-21).  LRN/max-pool are the paper's "fixed functions"
(Table 4 rows norm*/pool*); LRN constants follow reading C-20; both are pinned by the hand-computed cases in tests/golden/lrn_maxpool_hand.txt.

Activation layout in the oracle: image-major [B][features] (FC) and NHWC (CONV).
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def relu(x: np.ndarray) -> np.ndarray:
    return np.maximum(x, 0.0)


def fc_forward(Wq, a: np.ndarray, bias=None, apply_relu: bool = False) -> np.ndarray:
    """y[b, i] = sum_j Wq[i, j] a[b, j] + v[i] in fp64.  Wq may be a dense array
    or a scipy.sparse matrix (a library product is allowed as a step)."""
    a64 = np.asarray(a, dtype=np.float64)
    try:
        import scipy.sparse as sp
        if sp.issparse(Wq):
            y = (Wq.astype(np.float64) @ a64.T).T
        else:
            y = a64 @ np.asarray(Wq, dtype=np.float64).T
    except ImportError:  # pragma: no cover
        y = a64 @ np.asarray(Wq, dtype=np.float64).T
    y = np.asarray(y)
    if bias is not None:
        y = y + np.asarray(bias, dtype=np.float64)[None, :]
    return relu(y) if apply_relu else y


def fc_forward_blocked(layer, a: np.ndarray, bias=None, apply_relu: bool = False) -> np.ndarray:
    """Algorithm 2 step by step, fp64: for every stored row i of a
    block-contiguous layer (C-34) decode it (l.4-8), arrange the values as the
    bh x bw block (l.9), and add block @ a[:, col_id:col_id+bw] into
    y[:, row_id:row_id+bh] (l.10-12; MKL_CSRMM of the paper = a plain product)."""
    from . import decode  # local: decode imports nothing from here
    a64 = np.asarray(a, dtype=np.float64)
    y = np.zeros((a64.shape[0], layer.rows), dtype=np.float64)
    nbj = layer.cols // layer.bw
    for i in range(layer.stored_rows):
        blk = np.zeros(layer.bh * layer.bw, dtype=np.float64)
        for c, q, v in decode.decode_row_tokens(layer, i):
            if q != 0:
                blk[c] = v
        blk = blk.reshape(layer.bh, layer.bw)
        col_id = (i % nbj) * layer.bw
        row_id = (i // nbj) * layer.bh
        y[:, row_id:row_id + layer.bh] += a64[:, col_id:col_id + layer.bw] @ blk.T
    if bias is not None:
        y = y + np.asarray(bias, dtype=np.float64)[None, :]
    return relu(y) if apply_relu else y


def fc_abs_scale(Wq, a: np.ndarray, bias=None) -> np.ndarray:
    """sum_j |W_ij a_j| + |v_i|: the natural scale of each output's rounding
    error (used to report the elementwise error metric)."""
    a64 = np.abs(np.asarray(a, dtype=np.float64))
    try:
        import scipy.sparse as sp
        if sp.issparse(Wq):
            y = (abs(Wq).astype(np.float64) @ a64.T).T
        else:
            y = a64 @ np.abs(np.asarray(Wq, dtype=np.float64)).T
    except ImportError:  # pragma: no cover
        y = a64 @ np.abs(np.asarray(Wq, dtype=np.float64)).T
    y = np.asarray(y)
    if bias is not None:
        y = y + np.abs(np.asarray(bias, dtype=np.float64))[None, :]
    return y


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 (ties to even), returned as fp32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) >> 16) << 16
    return (u & 0xFFFFFFFF).astype(np.uint32).view(np.float32)


def conv_out_hw(h: int, k: int, stride: int, pad: int) -> int:
    return (h + 2 * pad - k) // stride + 1


def im2col(x: np.ndarray, kh: int, kw: int, stride: int, pad: int,
           c0: int, cg: int) -> Tuple[np.ndarray, int, int]:
    """Patches [B*Ho*Wo][kh*kw*cg] of channels [c0, c0+cg), K = (r*kw+s)*cg + c."""
    B, H, W, C = x.shape
    Ho, Wo = conv_out_hw(H, kh, stride, pad), conv_out_hw(W, kw, stride, pad)
    xp = np.zeros((B, H + 2 * pad, W + 2 * pad, cg), dtype=x.dtype)
    xp[:, pad:pad + H, pad:pad + W, :] = x[..., c0:c0 + cg]
    cols = np.empty((B, Ho, Wo, kh, kw, cg), dtype=x.dtype)
    for r in range(kh):
        for s in range(kw):
            cols[:, :, :, r, s, :] = xp[:, r:r + stride * Ho:stride, s:s + stride * Wo:stride, :]
    return cols.reshape(B * Ho * Wo, kh * kw * cg), Ho, Wo


def conv_forward(x: np.ndarray, Wq: np.ndarray, bias, kh: int, kw: int, stride: int,
                 pad: int, groups: int, apply_relu: bool = True, bf16: bool = True,
                 chunk: int = 8) -> np.ndarray:
    """NHWC conv via im2col + fp64 GEMM.  Wq: [M][kh*kw*C/groups]."""
    B, H, W, C = x.shape
    M = Wq.shape[0]
    cg, mg = C // groups, M // groups
    xin = bf16_round(x) if bf16 else np.asarray(x, dtype=np.float32)
    w = (bf16_round(Wq) if bf16 else np.asarray(Wq, dtype=np.float32)).astype(np.float64)
    Ho, Wo = conv_out_hw(H, kh, stride, pad), conv_out_hw(W, kw, stride, pad)
    out = np.empty((B, Ho, Wo, M), dtype=np.float64)
    for b0 in range(0, B, chunk):
        xb = xin[b0:b0 + chunk].astype(np.float64)
        nb = xb.shape[0]
        for g in range(groups):
            cols, _, _ = im2col(xb, kh, kw, stride, pad, g * cg, cg)
            y = cols @ w[g * mg:(g + 1) * mg].T
            out[b0:b0 + nb, :, :, g * mg:(g + 1) * mg] = y.reshape(nb, Ho, Wo, mg)
    if bias is not None:
        out += np.asarray(bias, dtype=np.float64)[None, None, None, :]
    return relu(out) if apply_relu else out


def conv_direct(x: np.ndarray, Wq: np.ndarray, kh: int, kw: int, stride: int, pad: int,
                groups: int) -> np.ndarray:
    """Direct convolution loop nest (fp64, no bias): used only to pin im2col."""
    B, H, W, C = x.shape
    M = Wq.shape[0]
    cg, mg = C // groups, M // groups
    w = Wq.astype(np.float64).reshape(M, kh, kw, cg)
    Ho, Wo = conv_out_hw(H, kh, stride, pad), conv_out_hw(W, kw, stride, pad)
    xp = np.zeros((B, H + 2 * pad, W + 2 * pad, C))
    xp[:, pad:pad + H, pad:pad + W, :] = x
    out = np.zeros((B, Ho, Wo, M))
    for m in range(M):
        g = m // mg
        for oh in range(Ho):
            for ow in range(Wo):
                patch = xp[:, oh * stride:oh * stride + kh, ow * stride:ow * stride + kw, g * cg:(g + 1) * cg]
                out[:, oh, ow, m] = np.einsum("brsc,rsc->b", patch, w[m])
    return out


LRN_N, LRN_ALPHA, LRN_BETA, LRN_K = 5, 1e-4, 0.75, 2.0   # C-20 (constants are the reading; the implementation is pinned by tests/golden/lrn_maxpool_hand.txt)


def lrn(x: np.ndarray) -> np.ndarray:
    """Cross-channel LRN over NHWC: b_c = a_c (k + alpha/n sum_{|c'-c|<=2} a_c'^2)^-beta."""
    x = np.asarray(x, dtype=np.float64)
    C = x.shape[-1]
    sq = x * x
    acc = np.zeros_like(x)
    half = LRN_N // 2
    for c in range(C):
        lo, hi = max(0, c - half), min(C - 1, c + half)
        acc[..., c] = sq[..., lo:hi + 1].sum(axis=-1)
    return x * np.power(LRN_K + (LRN_ALPHA / LRN_N) * acc, -LRN_BETA)


def maxpool(x: np.ndarray, k: int = 3, s: int = 2) -> np.ndarray:
    """k x k / stride s max-pool, no padding (AlexNet pool1/2/5, C-19)."""
    B, H, W, C = x.shape
    Ho, Wo = (H - k) // s + 1, (W - k) // s + 1
    out = np.full((B, Ho, Wo, C), -np.inf, dtype=x.dtype)
    for r in range(k):
        for q in range(k):
            out = np.maximum(out, x[:, r:r + s * Ho:s, q:q + s * Wo:s, :])
    return out


def alexnet_layer_shapes(image_hw: int = 227, image_c: int = 3):
    """(name, out elements per image) for the 13 rows of Table 4
    from the C-19 geometry; OUT(i,B) = 4 bytes x elements x B."""
    from synth import ALEXNET_CONV, ALEXNET_FC
    rows = []
    h, c = image_hw, image_c
    for cv in ALEXNET_CONV:
        h = conv_out_hw(h, cv.kh, cv.stride, cv.pad)
        c = cv.out_ch
        rows.append((cv.name, h * h * c))
        if cv.lrn:
            rows.append(("norm" + cv.name[-1], h * h * c))
        if cv.pool:
            h = (h - 3) // 2 + 1
            rows.append(("pool" + cv.name[-1], h * h * c))
    for fc in ALEXNET_FC:
        rows.append((fc.name, fc.rows))
    return rows
