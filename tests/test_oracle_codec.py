"""Pins of the oracle's codec (prune, quantize, relative index, Huffman, CDNI,
whole pipeline) against what the paper and mathematics fix -- not against the
oracle itself.  CPU only."""
import itertools
import random

import numpy as np
import pytest

from oracle import cdni, compress, decode, huffman, prune, quantize, relindex
import synth


# ---------------------------------------------------------------- prune

def test_prune_spec_example():
    # S:L86 2x2 example: keep the two largest magnitudes.
    W = np.array([[0.5, 0.01], [-0.4, 0.0]], dtype=np.float32)
    m = prune.prune_mask(W, 0.5)
    assert m.tolist() == [[True, False], [True, False]]


@pytest.mark.parametrize("seed", range(20))
def test_prune_fast_equals_stable_sort_with_ties(seed):
    rng = np.random.default_rng(seed)
    # few distinct magnitudes -> many ties at the threshold
    W = rng.integers(-4, 5, size=(13, 17)).astype(np.float32)
    d = float(rng.uniform(0, 1))
    a = prune.prune_mask(W, d)
    b = prune.prune_mask_sorted(W, d)
    assert (a == b).all()
    assert a.sum() == prune.n_keep_for(d, W.size)


def test_prune_magnitude_order_and_count():
    W = synth.random_matrix(64, 96, seed=3)
    m = prune.prune_mask(W, 0.1)
    assert m.sum() == int(np.floor(0.1 * W.size + 0.5))
    assert np.abs(W[m]).min() >= np.abs(W[~m]).max()


def test_prune_extremes():
    W = synth.random_matrix(5, 7, seed=1)
    assert prune.prune_mask(W, 0.0).sum() == 0
    assert prune.prune_mask(W, 1.0).all()


def test_prune_config_counts():
    # C5 fc6: floor(0.04 * 4096 * 25088 + 0.5) = 4,110,418
    assert prune.n_keep_for(0.04, 4096 * 25088) == 4110418
    assert prune.n_keep_for(0.09, 4096 * 9216) == 3397386


# ---------------------------------------------------------- quantize

def test_codebook_closed_form():
    kept = np.array([-0.3, 0.7, 0.1, -0.05], dtype=np.float32)
    cb = quantize.linear_codebook(kept, 3)
    assert cb.size == 8 and cb[0] == 0.0
    # endpoints are exactly the extreme kept weights; interior uniformly spaced
    assert cb[1] == np.float32(-0.3) and cb[7] == np.float32(0.7)
    steps = np.diff(cb[1:].astype(np.float64))
    assert np.allclose(steps, 1.0 / 6.0, rtol=1e-6)


@pytest.mark.parametrize("r", [1, 2, 5, 8])
def test_assignment_is_nearest_and_monotone(r):
    v = synth.random_matrix(1, 3000, seed=r).ravel()
    v = v[np.abs(v) > 0.5]
    cb = quantize.linear_codebook(v, r)
    q = quantize.assign(v, cb).astype(np.int64)
    assert q.min() >= 1 and q.max() <= (1 << r) - 1          # index 0 only for pads
    d_best = np.abs(v.astype(np.float64) - cb[q].astype(np.float64))
    # nearest centre: no centre strictly closer (checked against every centre)
    for j in range(1, 1 << r):
        assert (d_best <= np.abs(v.astype(np.float64) - np.float64(cb[j])) + 0).all()
    order = np.argsort(v, kind="stable")
    assert (np.diff(q[order]) >= 0).all()                      # monotone in w


def test_assignment_ties_to_smaller_index():
    cb = np.array([0.0, -1.0, 1.0, 3.0], dtype=np.float32)
    q = quantize.assign(np.array([0.0, 2.0], dtype=np.float32), cb)
    assert q.tolist() == [1, 2]


def test_degenerate_codebook():
    cb = quantize.linear_codebook(np.array([0.25, 0.25], dtype=np.float32), 5)
    assert (cb[1:] == np.float32(0.25)).all()
    assert quantize.assign(np.array([0.25], dtype=np.float32), cb).tolist() == [1]
    assert (quantize.linear_codebook(np.zeros(0, np.float32), 5) == 0).all()


# ---------------------------------------------------- relative index

# ------------------------------------------------ Lloyd k-means variant (C-33)

def test_lloyd_spec_example():
    """{0.9, 1.1, 2.9, 3.1}, r = 2 -> the used centres are 1.0 and
    3.0 (the grid's middle centre gets no weight and stays unused)."""
    v = np.array([0.9, 1.1, 2.9, 3.1], np.float32)
    cb = quantize.lloyd_codebook(v, 2)
    q = quantize.assign(v, cb)
    assert cb[0] == 0.0
    assert np.allclose(sorted(set(cb[q].tolist())), [1.0, 3.0], atol=1e-6)
    assert q[0] == q[1] and q[2] == q[3] and q[0] != q[2]


def _sse(v, cb):
    return float(np.sum((v.astype(np.float64) - cb[quantize.assign(v, cb)].astype(np.float64)) ** 2))


@pytest.mark.parametrize("seed", range(6))
def test_lloyd_fixed_point_and_no_worse_than_grid(seed):
    """At convergence every used centre is the mean of the weights nearest to
    it (1-D k-means stationarity, up to fp32 storage), and Lloyd steps never
    increase the squared error of the linear grid they start from."""
    rng = np.random.default_rng(seed)
    v = np.concatenate([rng.normal(-0.05, 0.01, 300), rng.normal(0.04, 0.02, 500)]).astype(np.float32)
    r = 3 + seed % 3
    cb = quantize.lloyd_codebook(v, r)
    q = quantize.assign(v, cb)
    for j in np.unique(q):
        m = float(np.mean(v[q == j].astype(np.float64)))
        assert abs(m - float(cb[j])) <= 1e-5 * max(abs(float(v.min())), abs(float(v.max())))
    assert _sse(v, cb) <= _sse(v, quantize.linear_codebook(v, r)) * (1 + 1e-9)
    assert np.all(np.diff(cb[1:].astype(np.float64)) >= 0)          # 1-D clusters stay ordered


def test_lloyd_degenerate_inputs():
    assert np.all(quantize.lloyd_codebook(np.zeros(0, np.float32), 4) == 0)
    cb = quantize.lloyd_codebook(np.full(50, 0.25, np.float32), 3)
    q = quantize.assign(np.full(50, 0.25, np.float32), cb)
    assert np.all(cb[q] == np.float32(0.25))


@pytest.mark.parametrize("seed,d,r,k", [(0, 0.1, 5, 4), (1, 0.3, 3, 2), (2, 0.04, 5, 5)])
def test_kmeans_decode_of_compress_is_prune_quantize(seed, d, r, k):
    W = synth.random_matrix(40, 257, seed=seed, scale=0.05)
    c = compress.compress_layer(W, d, r, k, quantizer="kmeans")
    assert np.array_equal(decode.decode_dense(c.layer), c.dense_q())


# ------------------------------------ block-contiguous container (Alg. 2, C-34)

def test_blocked_layout_paper_example():
    """an 8x8 matrix in 4x4 blocks becomes 4x16, each row one block
    stored contiguously; Alg. 2 l.11-12 map stored row i back to
    (row_id, col_id) = ((i / (cols/bw)) * bh, (i % (cols/bw)) * bw)."""
    A = np.arange(64).reshape(8, 8)
    M = compress.to_blocked(A, 4, 4)
    assert M.shape == (4, 16)
    assert M[0].tolist() == [0, 1, 2, 3, 8, 9, 10, 11, 16, 17, 18, 19, 24, 25, 26, 27]
    assert M[1].tolist() == [4, 5, 6, 7, 12, 13, 14, 15, 20, 21, 22, 23, 28, 29, 30, 31]
    assert M[2, 0] == 32 and M[3, 15] == 63
    L = cdni.Layer(8, 8, 4, 5, np.zeros(32, np.float32), {}, {}, np.zeros((5, 2), np.int64), b"", b"", None, 4, 4)
    for i in range(4):
        for p in range(16):
            r, c = L.unflatten(i, p)
            assert A[r, c] == M[i, p]


@pytest.mark.parametrize("rows,cols,bh,bw,d,k", [(256, 512, 128, 128, 0.1, 4), (64, 256, 64, 256, 0.3, 2),
                                                 (32, 128, 4, 64, 0.05, 4), (128, 192, 32, 64, 0.2, 8)])
def test_blocked_decode_of_compress_is_prune_quantize(rows, cols, bh, bw, d, k):
    W = synth.random_matrix(rows, cols, seed=rows + bh, scale=0.05)
    c = compress.compress_layer(W, d, 5, k, bh=bh, bw=bw)
    L = cdni.deserialize(cdni.serialize([c.layer]))[0]
    assert (L.bh, L.bw, L.stored_rows) == (bh, bw, (rows // bh) * (cols // bw))
    assert np.array_equal(decode.decode_dense(L), c.dense_q())
    # the same prune/quantize as the unblocked container: only the storage order differs
    u = compress.compress_layer(W, d, 5, k)
    assert np.array_equal(u.dense_q(), c.dense_q())


def test_blocked_unit_block_is_the_plain_container():
    W = synth.random_matrix(20, 64, seed=3, scale=0.05)
    a = compress.compress_layer(W, 0.3, 4, 3)
    b = compress.compress_layer(W, 0.3, 4, 3, bh=1, bw=64)
    assert cdni.serialize([a.layer]) == cdni.serialize([b.layer])


def test_blocked_rejects_non_tiling_blocks():
    W = synth.random_matrix(20, 64, seed=3, scale=0.05)
    with pytest.raises(ValueError):
        compress.compress_layer(W, 0.3, 4, 3, bh=3, bw=64)
    c = compress.compress_layer(W, 0.3, 4, 3, bh=4, bw=32)
    buf = bytearray(cdni.serialize([c.layer]))
    buf[18:22] = (5).to_bytes(4, "little")           # bh = 5 does not divide 20 rows
    with pytest.raises(cdni.CDNIError):
        cdni.deserialize(bytes(buf))


def test_relindex_spec_k2_example():
    # k=2, columns {0,5,11} -> gaps [0,3,0,3,1], vals [x,0,y,0,z]
    v, g = relindex.encode_row([0, 5, 11], [7, 8, 9], k=2)
    assert g == [0, 3, 0, 3, 1]
    assert v == [7, 0, 8, 0, 9]
    dec = relindex.decode_row(v, g)
    assert [(c, q) for c, q in dec if q != 0] == [(0, 7), (5, 8), (11, 9)]


def test_relindex_paper_padding_rule():
    # k=2, first non-zero of a row at column >= 4 -> a pad first
    v, g = relindex.encode_row([4], [1], k=2)
    assert v == [0, 1] and g == [3, 0]
    v, g = relindex.encode_row([3], [1], k=2)       # fits in 2 bits: no pad
    assert v == [1] and g == [3]
    # k=4, first column 40 -> (0,15),(0,15),(x,8)
    v, g = relindex.encode_row([40], [5], k=4)
    assert list(zip(v, g)) == [(0, 15), (0, 15), (5, 8)]


@pytest.mark.parametrize("seed", range(10))
def test_relindex_roundtrip_and_vectorised(seed):
    rng = np.random.default_rng(seed)
    rows, cols, k = 9, 200, int(rng.integers(1, 6))
    mask = rng.random((rows, cols)) < rng.uniform(0.0, 0.3)
    q = rng.integers(1, 32, size=(rows, cols))
    vt, gt, rt = relindex.encode_matrix(mask, q, k)
    pos = 0
    for i in range(rows):
        cs = list(np.flatnonzero(mask[i]))
        ev, eg = relindex.encode_row(cs, list(q[i, cs]), k)
        n = int(rt[i])
        assert list(vt[pos:pos + n]) == ev and list(gt[pos:pos + n]) == eg
        assert max(eg, default=0) < (1 << k)
        dec = relindex.decode_row(ev, eg)
        assert [c for c, s in dec if s != 0] == cs
        # pads carry value index 0 and gap 2^k - 1 (C-06)
        assert all(gg == (1 << k) - 1 for vv, gg in zip(ev, eg) if vv == 0)
        pos += n
    assert pos == vt.size


# ------------------------------------------------ Huffman

def _brute_force_min_cost(freqs):
    syms = list(freqs)
    n = len(syms)
    best = None
    for L in itertools.product(range(1, n), repeat=n):
        if sum(2.0 ** -l for l in L) <= 1.0 + 1e-12:
            c = sum(freqs[s] * l for s, l in zip(syms, L))
            best = c if best is None else min(best, c)
    return best


@pytest.mark.parametrize("seed", range(40))
def test_huffman_optimal_vs_brute_force(seed):
    rng = random.Random(seed)
    n = rng.randint(2, 6)
    freqs = {s: rng.randint(1, 20) for s in rng.sample(range(40), n)}
    L = huffman.code_lengths(freqs)
    assert huffman.cost(freqs, L) == _brute_force_min_cost(freqs)
    assert huffman.kraft_sum(L) == 1.0


def test_huffman_spec_examples():
    assert huffman.code_lengths({0: 3, 1: 1, 2: 1}) == {0: 1, 1: 2, 2: 2}
    assert set(huffman.code_lengths({0: 1, 1: 1, 2: 1, 3: 1}).values()) == {2}
    assert huffman.code_lengths({5: 9}) == {5: 1}
    assert huffman.kraft_sum({5: 1}) == 0.5
    assert huffman.code_lengths({}) == {}


def test_canonical_codes_and_bits():
    codes = huffman.canonical_codes({0: 1, 1: 2, 2: 2})       # a=0, b=10, c=11
    assert codes == {0: (0, 1), 1: (2, 2), 2: (3, 2)}
    data, nbits, _ = huffman.encode(np.array([0, 0, 1]), codes)   # 0,0,1,0
    assert nbits == 4 and data == bytes([0b00100000])


def test_canonical_prefix_free_and_deterministic():
    rng = np.random.default_rng(1)
    toks = rng.zipf(1.5, 5000) % 40
    f = {int(s): int(c) for s, c in enumerate(np.bincount(toks)) if c}
    L1, L2 = huffman.code_lengths(f), huffman.code_lengths(dict(reversed(list(f.items()))))
    assert L1 == L2
    codes = huffman.canonical_codes(L1)
    words = [format(c, f"0{l}b") for c, l in codes.values()]
    for a in words:
        for b in words:
            assert a == b or not b.startswith(a)


def test_huffman_roundtrip_10k():
    rng = random.Random(7)
    for t in range(10000):
        n = rng.randint(0, 12)
        alpha = rng.randint(1, 9)
        toks = [rng.randrange(alpha) for _ in range(n)]
        f = {}
        for s in toks:
            f[s] = f.get(s, 0) + 1
        L = huffman.code_lengths(f)
        data, nbits, _ = huffman.encode(np.array(toks, dtype=np.int64), huffman.canonical_codes(L))
        dec = huffman.CanonicalDecoder(L).decode_range(data, 0, nbits) if n else []
        assert dec == toks
        assert nbits == huffman.cost(f, L)


def test_decode_rejects_code_crossing_end():
    L = {0: 1, 1: 2, 2: 2}
    data, nbits, _ = huffman.encode(np.array([1, 2]), huffman.canonical_codes(L))
    with pytest.raises(ValueError):
        huffman.CanonicalDecoder(L).decode_range(data, 0, nbits - 1)


# --------------------------------------------------------------- CDNI + pipeline

def _small(seed, rows=23, cols=71, d=0.2, r=5, k=4, bias=True):
    W = synth.random_matrix(rows, cols, seed=seed, scale=0.05)
    v = synth.random_matrix(1, rows, seed=seed + 1).ravel() if bias else None
    return W, compress.compress_layer(W, d, r, k, v)


@pytest.mark.parametrize("seed,d,r,k", [(0, 0.2, 5, 4), (1, 0.05, 5, 2), (2, 0.6, 8, 8),
                                        (3, 0.01, 2, 1), (4, 1.0, 4, 3), (5, 0.0, 5, 4)])
def test_decode_of_compress_is_prune_quantize(seed, d, r, k):
    W, c = _small(seed, d=d, r=r, k=k)
    L = cdni.deserialize(cdni.serialize([c.layer]))[0]
    Wd = decode.decode_dense(L)
    # S:L153/L170 roundtrip, bit-exact: kept entries equal their centre
    mask = prune.prune_mask(W, d)
    expect = np.zeros_like(W)
    if mask.any():
        cb = quantize.linear_codebook(W[mask], r)
        expect[mask] = cb[quantize.assign(W[mask], cb)]
    assert np.array_equal(Wd.view(np.uint32), expect.view(np.uint32))
    # token streams decode back exactly, pads included
    R, C, S, V = decode.decode_layer(L)
    assert np.array_equal(S, c.val_tokens)
    assert int(c.row_tokens.sum()) == S.size


def test_cdni_roundtrip_and_errors():
    _, c = _small(9)
    buf = cdni.serialize([c.layer, c.layer])
    again = cdni.serialize(cdni.deserialize(buf))
    assert again == buf
    assert cdni.serialize([]) == b"CDNI" + bytes([1, 0, 0, 0, 0, 0])
    with pytest.raises(cdni.CDNIError) as e:
        cdni.deserialize(buf[:-1])
    assert e.value.kind == "truncated"
    with pytest.raises(cdni.CDNIError) as e:
        cdni.deserialize(b"XDNI" + buf[4:])
    assert e.value.kind == "magic"
    with pytest.raises(cdni.CDNIError) as e:
        cdni.deserialize(buf[:4] + bytes([2, 0]) + buf[6:])
    assert e.value.kind == "version"


def test_all_pruned_layer():
    W, c = _small(11, d=0.0)
    assert c.layer.row_ptr.max() == 0 and c.layer.val_bytes == b""
    L = cdni.deserialize(cdni.serialize([c.layer]))[0]
    assert decode.decode_dense(L).sum() == 0


def test_c1_full_roundtrip():
    spec = synth.CONFIGS["C1"].fc[0]
    W, v = synth.fc_weights(spec, 0)
    c = compress.compress_layer(W, spec.density, spec.r, spec.k, v)
    L = cdni.deserialize(cdni.serialize([c.layer]))[0]
    assert np.array_equal(decode.decode_dense(L), c.dense_q())
    nnz = int(c.mask.sum())
    assert nnz == 104858
    # compressed size well under the dense fp32 size (S acceptance 4)
    assert len(c.layer.val_bytes) + len(c.layer.gap_bytes) < 0.05 * W.nbytes
    # Kraft equality of both codes (BASELINE north_star oracle check)
    assert huffman.kraft_sum(L.val_lengths) == 1.0 and huffman.kraft_sum(L.gap_lengths) == 1.0
