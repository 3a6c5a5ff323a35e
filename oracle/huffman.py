"""Huffman coding of the val and col_ind streams ("Huffman
encoding is employed on both the weight clusters and the index differences to
ensure that more common cluster centres and index differences are represented
with fewer bits"; Fig. 1e).

Readings:
  C-14 one code per (layer, stream), built from that layer's token counts;
       zero-frequency symbols get no code.
  C-15 merge rule: repeatedly merge the two lowest nodes ordered by
       (count, smallest symbol id in the subtree); code length = leaf depth.
       One symbol -> length 1; no symbols -> empty table.
  C-16 lengths are not limited (the product rejects > 32 bits).
  C-17 canonical codes in (length, symbol) order, MSB-first bit order,
       absolute bit offsets, streams byte-padded with zeros only at the end.
"""
from __future__ import annotations

import heapq
from typing import Dict, List, Sequence, Tuple

import numpy as np


def code_lengths(freqs: Dict[int, int]) -> Dict[int, int]:
    """Huffman code length per symbol with the C-15 tie rule."""
    syms = sorted(s for s, f in freqs.items() if f > 0)
    if not syms:
        return {}
    if len(syms) == 1:
        return {syms[0]: 1}
    # heap items: (count, min symbol in subtree, node id); node id is unique
    heap = []
    children: List[Tuple[int, int]] = []
    leaf_of: Dict[int, int] = {}
    for s in syms:
        nid = len(children)
        children.append((-1, s))         # leaf: (-1, symbol)
        leaf_of[nid] = s
        heap.append((int(freqs[s]), s, nid))
    heapq.heapify(heap)
    while len(heap) > 1:
        c1, m1, n1 = heapq.heappop(heap)
        c2, m2, n2 = heapq.heappop(heap)
        nid = len(children)
        children.append((n1, n2))
        heapq.heappush(heap, (c1 + c2, min(m1, m2), nid))
    root = heap[0][2]
    lengths: Dict[int, int] = {}
    stack = [(root, 0)]
    while stack:
        nid, depth = stack.pop()
        a, b = children[nid]
        if a == -1:
            lengths[b] = depth
        else:
            stack.append((a, depth + 1))
            stack.append((b, depth + 1))
    return lengths


def canonical_codes(lengths: Dict[int, int]) -> Dict[int, Tuple[int, int]]:
    """symbol -> (code, length); codes assigned in (length, symbol) order:
    code_0 = 0, code_i = (code_{i-1} + 1) << (len_i - len_{i-1})."""
    order = sorted(lengths.items(), key=lambda kv: (kv[1], kv[0]))
    out: Dict[int, Tuple[int, int]] = {}
    code = 0
    prev_len = None
    for s, L in order:
        if prev_len is None:
            code = 0
        else:
            code = (code + 1) << (L - prev_len)
        out[s] = (code, L)
        prev_len = L
    return out


def encode(tokens: np.ndarray, codes: Dict[int, Tuple[int, int]]) -> Tuple[bytes, int, np.ndarray]:
    """Concatenate the codes of `tokens` MSB-first.  Returns (bytes padded with
    zero bits at the end, total bit count, bit offset of every token)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    if tokens.size == 0:
        return b"", 0, np.zeros(0, dtype=np.int64)
    maxsym = int(tokens.max())
    code_of = np.zeros(maxsym + 1, dtype=np.int64)
    len_of = np.zeros(maxsym + 1, dtype=np.int64)
    for s, (c, L) in codes.items():
        if s <= maxsym:
            code_of[s] = c
            len_of[s] = L
    lens = len_of[tokens]
    if np.any(lens == 0):
        raise ValueError("token without a code")
    cds = code_of[tokens]
    offs = np.zeros(tokens.size, dtype=np.int64)
    np.cumsum(lens[:-1], out=offs[1:])
    total = int(offs[-1] + lens[-1])
    # expand every code into its bits, MSB first (in chunks of tokens)
    bits = np.empty(total, dtype=np.uint8)
    step = 1 << 20
    for s in range(0, tokens.size, step):
        e = min(tokens.size, s + step)
        ln = lens[s:e]
        tok_of_bit = np.repeat(np.arange(s, e), ln)
        b0 = int(offs[s])
        b1 = int(offs[e - 1] + lens[e - 1])
        bit_in_tok = np.arange(b0, b1) - offs[tok_of_bit]
        shift = lens[tok_of_bit] - 1 - bit_in_tok
        bits[b0:b1] = ((cds[tok_of_bit] >> shift) & 1).astype(np.uint8)
    return np.packbits(bits).tobytes(), total, offs


class CanonicalDecoder:
    """Plain bit-by-bit canonical decoder (first code / count per length)."""

    def __init__(self, lengths: Dict[int, int]):
        self.lengths = dict(lengths)
        self.max_len = max(lengths.values()) if lengths else 0
        order = sorted(lengths.items(), key=lambda kv: (kv[1], kv[0]))
        self.sorted_syms = [s for s, _ in order]
        self.count = [0] * (self.max_len + 2)
        for _, L in order:
            self.count[L] += 1
        self.first_code = [0] * (self.max_len + 2)
        self.first_index = [0] * (self.max_len + 2)
        code = 0
        idx = 0
        for L in range(1, self.max_len + 1):
            self.first_code[L] = code
            self.first_index[L] = idx
            code = (code + self.count[L]) << 1
            idx += self.count[L]

    def decode_range(self, data: bytes, bit_begin: int, bit_end: int) -> List[int]:
        """Decode every code that starts in [bit_begin, bit_end); a code that
        runs past bit_end is a malformed stream."""
        out: List[int] = []
        pos = bit_begin
        while pos < bit_end:
            code = 0
            L = 0
            while True:
                if pos >= bit_end or L >= self.max_len:
                    raise ValueError("malformed stream: code crosses range end")
                byte = data[pos >> 3]
                bit = (byte >> (7 - (pos & 7))) & 1
                pos += 1
                code = (code << 1) | bit
                L += 1
                off = code - self.first_code[L]
                if 0 <= off < self.count[L]:
                    out.append(self.sorted_syms[self.first_index[L] + off])
                    break
        return out


def kraft_sum(lengths: Dict[int, int]) -> float:
    from fractions import Fraction
    return float(sum(Fraction(1, 1 << L) for L in lengths.values()))


def cost(freqs: Dict[int, int], lengths: Dict[int, int]) -> int:
    return sum(int(freqs[s]) * lengths[s] for s in lengths)
