"""CDNI container ("bit-exact format"; the paper's stored model
is Fig. 1e: two Huffman bitstreams plus row_ptr 2-tuples of start
bit addresses).

Layout (all integers little-endian):
  "CDNI"  u16 version(=1)  u32 layer_count
  per layer:
    u32 rows, u32 cols, u32 bh, u32 bw          (unblocked: bh=1, bw=cols)
      blocked (Alg. 2, reading C-34): rows % bh == 0, cols % bw
      == 0; the streams hold the "modified matrix" M' whose stored row
      i = bi * (cols/bw) + bj is block (bi, bj) flattened row-major (element
      (r, c) of the block at position r*bw + c); row_ptr has one entry per
      stored row (+1) and relative indexing runs along the stored rows
    u8 k, u8 r
    u16 n_codebook, n_codebook x f32           (codebook C, index 0 = 0.0)
    u16 n_val_syms, n x (u16 symbol, u8 length)  (val-stream Huffman lengths)
    u16 n_gap_syms, n x (u16 symbol, u8 length)  (gap-stream Huffman lengths)
    (stored_rows+1) x (u64 val_bit, u64 gap_bit) (row_ptr 2-tuples)
    val stream: ceil(row_ptr[rows].val / 8) bytes
    gap stream: ceil(row_ptr[rows].gap / 8) bytes
    u8 has_bias, [rows x f32]
Symbol tables are written in ascending symbol order; codes are rebuilt
canonically from the lengths (C-17).
"""
from __future__ import annotations

import dataclasses
import struct
from typing import Dict, List, Optional

import numpy as np

MAGIC = b"CDNI"
VERSION = 1


class CDNIError(ValueError):
    def __init__(self, kind: str, msg: str = ""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


@dataclasses.dataclass
class Layer:
    rows: int
    cols: int
    k: int
    r: int
    codebook: np.ndarray                 # fp32, 2^r entries
    val_lengths: Dict[int, int]
    gap_lengths: Dict[int, int]
    row_ptr: np.ndarray                  # (rows+1, 2) int64 bit offsets
    val_bytes: bytes
    gap_bytes: bytes
    bias: Optional[np.ndarray] = None    # fp32 rows
    bh: int = 1
    bw: int = 0

    def __post_init__(self):
        if self.bw == 0:
            self.bw = self.cols

    @property
    def blocked(self) -> bool:
        return not (self.bh == 1 and self.bw == self.cols)

    @property
    def stored_rows(self) -> int:
        """Rows of the stored matrix: the weight rows, or the blocks of M' (C-34)."""
        return (self.rows // self.bh) * (self.cols // self.bw) if self.blocked else self.rows

    @property
    def stored_cols(self) -> int:
        return self.bh * self.bw if self.blocked else self.cols

    def unflatten(self, i, p):
        """(weight row, weight column) of position p of stored row i (Alg. 2
        lines 11-13: col_id = (i % (cols/bw)) * bw, row_id = (i / (cols/bw)) * bh)."""
        if not self.blocked:
            return i, p
        nbj = self.cols // self.bw
        i = np.asarray(i)
        p = np.asarray(p)
        return (i // nbj) * self.bh + p // self.bw, (i % nbj) * self.bw + p % self.bw


def _table(lengths: Dict[int, int]) -> bytes:
    out = [struct.pack("<H", len(lengths))]
    for s in sorted(lengths):
        out.append(struct.pack("<HB", s, lengths[s]))
    return b"".join(out)


def serialize(layers: List[Layer]) -> bytes:
    out = [MAGIC, struct.pack("<HI", VERSION, len(layers))]
    for L in layers:
        out.append(struct.pack("<IIII", L.rows, L.cols, L.bh, L.bw))
        out.append(struct.pack("<BB", L.k, L.r))
        cb = np.asarray(L.codebook, dtype="<f4")
        out.append(struct.pack("<H", cb.size))
        out.append(cb.tobytes())
        out.append(_table(L.val_lengths))
        out.append(_table(L.gap_lengths))
        rp = np.asarray(L.row_ptr, dtype="<u8").reshape(L.stored_rows + 1, 2)
        out.append(rp.tobytes())
        nv = (int(rp[-1, 0]) + 7) // 8
        ng = (int(rp[-1, 1]) + 7) // 8
        assert len(L.val_bytes) == nv and len(L.gap_bytes) == ng
        out.append(L.val_bytes)
        out.append(L.gap_bytes)
        if L.bias is None:
            out.append(b"\x00")
        else:
            out.append(b"\x01")
            out.append(np.asarray(L.bias, dtype="<f4").tobytes())
    return b"".join(out)


class _Reader:
    def __init__(self, buf: bytes):
        self.buf = buf
        self.pos = 0

    def take(self, n: int) -> bytes:
        if self.pos + n > len(self.buf):
            raise CDNIError("truncated", f"need {n} bytes at {self.pos}")
        b = self.buf[self.pos:self.pos + n]
        self.pos += n
        return b

    def unpack(self, fmt: str):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt)))


def _read_table(rd: _Reader) -> Dict[int, int]:
    (n,) = rd.unpack("<H")
    out = {}
    for _ in range(n):
        s, L = rd.unpack("<HB")
        out[s] = L
    return out


def deserialize(buf: bytes) -> List[Layer]:
    rd = _Reader(buf)
    if rd.take(4) != MAGIC:
        raise CDNIError("magic")
    ver, nl = rd.unpack("<HI")
    if ver != VERSION:
        raise CDNIError("version", str(ver))
    layers = []
    for _ in range(nl):
        rows, cols, bh, bw = rd.unpack("<IIII")
        k, r = rd.unpack("<BB")
        (ncb,) = rd.unpack("<H")
        cb = np.frombuffer(rd.take(4 * ncb), dtype="<f4").astype(np.float32)
        vl = _read_table(rd)
        gl = _read_table(rd)
        if bh == 0 or bw == 0 or rows % bh or cols % bw:
            raise CDNIError("malformed", f"block {bh}x{bw} does not tile {rows}x{cols}")
        nst = rows if (bh == 1 and bw == cols) else (rows // bh) * (cols // bw)
        rp = np.frombuffer(rd.take(16 * (nst + 1)), dtype="<u8").reshape(nst + 1, 2).astype(np.int64)
        vb = rd.take((int(rp[-1, 0]) + 7) // 8)
        gb = rd.take((int(rp[-1, 1]) + 7) // 8)
        (hb,) = rd.unpack("<B")
        bias = np.frombuffer(rd.take(4 * rows), dtype="<f4").astype(np.float32) if hb else None
        layers.append(Layer(rows, cols, k, r, cb, vl, gl, rp, vb, gb, bias, bh, bw))
    if rd.pos != len(buf):
        raise CDNIError("malformed", "trailing bytes")
    return layers
