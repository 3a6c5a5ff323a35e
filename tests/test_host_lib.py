"""CPU tests of the C-ABI library's host side (no GPU): the library loads and
exports every symbol in include/cdn.h; the product compressor is byte-identical
to the oracle's; the load-time host walk re-derives the oracle's tokens; the
CDNI validator rejects malformed containers; the C++ DP equals the oracle DP."""
import math
import os
import random
import re
import struct

import numpy as np
import pytest

import paper_1711_00244_b200 as cdn
from oracle import cdni as ocdni, compress as ocompress, decode as odecode, planner as oplanner
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "cdn.h")).read()
    names = set(re.findall(r"\b(cdn_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 18
    lib = cdn.load_library()
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert cdn.abi_version() == 2


def _oracle_bytes(W, d, r, k, bias):
    c = ocompress.compress_layer(W, d, r, k, bias)
    return ocdni.serialize([c.layer]), c


@pytest.mark.parametrize("seed,rows,cols,d,r,k,bias", [
    (0, 23, 71, 0.2, 5, 4, True), (1, 40, 300, 0.03, 5, 4, True), (2, 17, 33, 0.7, 8, 8, False),
    (3, 9, 500, 0.01, 2, 1, True), (4, 12, 12, 1.0, 4, 3, True), (5, 8, 8, 0.0, 5, 4, True),
    (6, 64, 64, 0.25, 1, 2, False), (7, 5, 1000, 0.5, 8, 2, True)])
def test_compressor_byte_identical_to_oracle(seed, rows, cols, d, r, k, bias):
    W = synth.random_matrix(rows, cols, seed=seed, scale=0.05)
    v = synth.random_matrix(1, rows, seed=seed + 99).ravel() if bias else None
    ob, _ = _oracle_bytes(W, d, r, k, v)
    pb = cdn.compress_dense(W, d, r, k, v)
    assert pb == ob


@pytest.mark.parametrize("seed,rows,cols,d,r,k", [
    (0, 23, 71, 0.2, 5, 4), (1, 40, 300, 0.03, 5, 4), (2, 17, 33, 0.7, 8, 8), (3, 9, 500, 0.01, 2, 1),
    (6, 64, 64, 0.25, 1, 2), (7, 5, 1000, 0.5, 3, 2)])
def test_kmeans_compressor_byte_identical_to_oracle(seed, rows, cols, d, r, k):
    """The Lloyd quantizer (C-33) in the product compressor reproduces the
    oracle's arithmetic exactly (binary64 means in row-major order)."""
    W = synth.random_matrix(rows, cols, seed=seed, scale=0.05)
    v = synth.random_matrix(1, rows, seed=seed + 99).ravel()
    c = ocompress.compress_layer(W, d, r, k, v, quantizer="kmeans")
    assert cdn.compress_dense(W, d, r, k, v, quantizer="kmeans") == ocdni.serialize([c.layer])


@pytest.mark.parametrize("rows,cols,bh,bw,q", [(256, 512, 128, 128, "linear"), (64, 256, 4, 64, "kmeans"),
                                               (30, 90, 10, 45, "linear"), (64, 64, 64, 64, "linear")])
def test_blocked_compressor_byte_identical_to_oracle(rows, cols, bh, bw, q):
    W = synth.random_matrix(rows, cols, seed=bh + bw, scale=0.05)
    v = synth.random_matrix(1, rows, seed=3).ravel()
    c = ocompress.compress_layer(W, 0.1, 5, 4, v, quantizer=q, bh=bh, bw=bw)
    assert cdn.compress_dense(W, 0.1, 5, 4, v, quantizer=q, bh=bh, bw=bw) == ocdni.serialize([c.layer])


def test_compressor_ties_and_duplicates():
    # many equal magnitudes: exact-count tie rule (C-10) and quantizer ties (C-07)
    rng = np.random.default_rng(3)
    W = (rng.integers(-3, 4, size=(20, 30)) * 0.125).astype(np.float32)
    for d in (0.1, 0.33, 0.5):
        assert cdn.compress_dense(W, d, 3, 2, None) == _oracle_bytes(W, d, 3, 2, None)[0]


def test_compressor_c1_identical():
    spec = synth.CONFIGS["C1"].fc[0]
    W, v = synth.fc_weights(spec, 0)
    assert cdn.compress_dense(W, spec.density, spec.r, spec.k, v) == _oracle_bytes(W, spec.density, spec.r, spec.k, v)[0]


def test_host_walk_equals_oracle_decode():
    spec = synth.CONFIGS["C1"].fc[0]
    W, v = synth.fc_weights(spec, 0)
    buf, c = _oracle_bytes(W, spec.density, spec.r, spec.k, v)
    row, col, sym = cdn.debug_host_walk(buf)
    L = ocdni.deserialize(buf)[0]
    R, Cc, S, _ = odecode.decode_layer(L)
    assert np.array_equal(row, R) and np.array_equal(col, Cc) and np.array_equal(sym, S)


@pytest.mark.parametrize("bh,bw", [(128, 128), (4, 64), (64, 256)])
def test_host_walk_blocked_equals_oracle_decode(bh, bw):
    """A block-contiguous container (Alg. 2, C-34): the load-time walk runs over
    the stored rows of M' (blocks) and reproduces the oracle's tokens."""
    W = synth.random_matrix(256, 512, seed=bh, scale=0.05)
    v = synth.random_matrix(1, 256, seed=1).ravel()
    c = ocompress.compress_layer(W, 0.08, 5, 4, v, bh=bh, bw=bw)
    buf = ocdni.serialize([c.layer])
    row, col, sym = cdn.debug_host_walk(buf)
    R, Cc, S, _ = odecode.decode_layer(c.layer)
    assert np.array_equal(row, R) and np.array_equal(col, Cc) and np.array_equal(sym, S)


def _layer_bytes(seed=0, rows=6, cols=40, d=0.3, r=3, k=2):
    W = synth.random_matrix(rows, cols, seed=seed)
    c = ocompress.compress_layer(W, d, r, k, None)
    return c.layer


def _expect_error(buf, name):
    with pytest.raises(cdn.CDNError) as e:
        cdn.debug_host_walk(buf)
    assert e.value.name == name, str(e.value)


def test_cdni_validation_errors():
    L = _layer_bytes()
    good = ocdni.serialize([L])
    cdn.debug_host_walk(good)
    _expect_error(good[:-3], "CDN_E_TRUNCATED")
    _expect_error(b"XDNI" + good[4:], "CDN_E_MAGIC")
    _expect_error(good[:4] + struct.pack("<H", 7) + good[6:], "CDN_E_VERSION")
    _expect_error(good + b"\0", "CDN_E_MALFORMED")
    # Kraft violation: lengthen one val code
    L2 = _layer_bytes()
    s = max(L2.val_lengths)
    L2.val_lengths[s] += 1
    _expect_error(ocdni.serialize([L2]), "CDN_E_MALFORMED")
    # code length > 32
    L3 = _layer_bytes()
    L3.val_lengths = {0: 1, 1: 33}
    _expect_error(ocdni.serialize([L3]), "CDN_E_UNSUPPORTED")
    # a block that does not tile the matrix (C-34)
    bad = bytearray(good)
    rows = struct.unpack_from("<I", bad, 10)[0]
    bad[18:22] = struct.pack("<I", rows + 1)
    _expect_error(bytes(bad), "CDN_E_MALFORMED")
    # row_ptr moved by one code: token counts of the two streams differ
    L5 = _layer_bytes()
    rp = L5.row_ptr.copy()
    # shift row 1's val start to row 2's: row 0 gets extra val tokens
    rp[1, 0] = rp[2, 0]
    L5.row_ptr = rp
    _expect_error(ocdni.serialize([L5]), "CDN_E_MALFORMED")
    # k > 8 unsupported
    L6 = _layer_bytes()
    L6.k = 9
    _expect_error(ocdni.serialize([L6]), "CDN_E_UNSUPPORTED")


def test_column_out_of_range_rejected():
    # declare fewer columns than the streams address
    L = _layer_bytes(cols=40)
    L.cols = 20
    L.bw = 20
    _expect_error(ocdni.serialize([L]), "CDN_E_MALFORMED")


def test_pad_invariant_rejected():
    # hand-built single-row layer: tokens (val 0, gap 0) violate C-06
    from oracle import huffman
    vt = np.array([0, 1]); gt = np.array([0, 0])
    vl = {0: 1, 1: 1}; gl = {0: 1}
    vb, vn, _ = huffman.encode(vt, huffman.canonical_codes(vl))
    gb, gn, _ = huffman.encode(gt, huffman.canonical_codes(gl))
    L = ocdni.Layer(1, 8, 2, 1, np.array([0.0, 0.5], np.float32), vl, gl,
                    np.array([[0, 0], [vn, gn]]), vb, gb)
    _expect_error(ocdni.serialize([L]), "CDN_E_MALFORMED")


def _rand_problem(rng, f, Bmax, latency):
    time = np.zeros((f, Bmax))
    for i in range(f):
        base, slope, ex = rng.uniform(0.5, 5), rng.uniform(0.05, 2), rng.uniform(0.6, 1.1)
        time[i] = [base + slope * B ** ex for B in range(1, Bmax + 1)]
    inb = [rng.randint(1, 20) for _ in range(f)]
    outb = [rng.randint(1, 20) for _ in range(f)]
    ws = [rng.randint(0, 10) for _ in range(f)]
    tot = rng.randint(20, 40 * Bmax)
    lat = rng.uniform(5, 60) if latency else None
    p = oplanner.Problem([{B: time[i][B - 1] for B in range(1, Bmax + 1)} for i in range(f)],
                         inb, outb, ws, tot, lat)
    return p, time


@pytest.mark.parametrize("seed", range(300))
def test_cpp_dp_equals_oracle_dp(seed):
    rng = random.Random(1000 + seed)
    f, Bmax = rng.randint(1, 4), rng.randint(1, 12)
    p, time = _rand_problem(rng, f, Bmax, latency=(seed % 3 == 0))
    ref = oplanner.dp_plan(p, Bmax)
    try:
        bs, opt = cdn.plan_dp(time, p.in_bytes, p.out_bytes, p.ws, p.tot, p.latency or 0.0, step=1)
    except cdn.CDNError as e:
        assert e.name == "CDN_E_INFEASIBLE" and ref is None
        return
    assert ref is not None
    assert bs == ref.batches and opt == ref.time
    # coarser memory grid (C-25): never better than exact, and exactly feasible
    for step in (4, 16):
        try:
            bs2, opt2 = cdn.plan_dp(time, p.in_bytes, p.out_bytes, p.ws, p.tot, p.latency or 0.0, step=step)
        except cdn.CDNError:
            continue
        assert opt2 / bs2[-1] >= ref.per_image * (1 - 1e-12)
        assert oplanner.chain_cost(p, bs2) < math.inf
