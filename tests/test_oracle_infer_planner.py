"""Pins of the oracle's inference and planner.  CPU only."""
import itertools
import math
import random

import os

import numpy as np
import pytest

from oracle import compress, decode, cdni, infer, planner
import synth


# ------------------------------------------------------------- FC (Eq. 1-2)

def test_fc_identity_weight():
    # identity weights (compressed) x any a -> a (+ zero bias)
    n = 16
    W = np.eye(n, dtype=np.float32)
    c = compress.compress_layer(W, 1.0 / n, 5, 4)
    L = cdni.deserialize(cdni.serialize([c.layer]))[0]
    Wq = decode.decode_dense(L)
    a = synth.random_activations(n, 3, seed=2)
    assert np.array_equal(infer.fc_forward(Wq, a), a.astype(np.float64))


def test_fc_all_pruned_is_bias():
    W = synth.random_matrix(7, 9, seed=4)
    v = synth.random_matrix(1, 7, seed=5).ravel()
    c = compress.compress_layer(W, 0.0, 5, 4, v)
    y = infer.fc_forward(c.dense_q(), synth.random_activations(9, 4, 1), v)
    assert np.array_equal(y, np.broadcast_to(v.astype(np.float64), (4, 7)))


def test_fc_linearity_and_sparse_equals_dense():
    import scipy.sparse as sp
    W = synth.random_matrix(30, 40, seed=8) * (synth.random_matrix(30, 40, seed=9) > 1.0)
    v = synth.random_matrix(1, 30, seed=10).ravel()
    a1, a2 = synth.random_activations(40, 5, 1), synth.random_activations(40, 5, 2)
    alpha = 1.75
    y = lambda a: infer.fc_forward(W, a, v)
    lhs = y(alpha * a1.astype(np.float64) + a2)
    rhs = alpha * (y(a1) - v) + y(a2)
    assert np.allclose(lhs, rhs, rtol=1e-12, atol=1e-12)
    assert np.allclose(infer.fc_forward(sp.csr_matrix(W), a1, v), y(a1), rtol=1e-14, atol=1e-14)


# ---------------------------------------------------------- CONV

@pytest.mark.parametrize("geom", [(3, 3, 1, 0, 1), (3, 3, 2, 1, 1), (5, 5, 1, 2, 2), (1, 1, 1, 0, 1),
                                  (11, 11, 4, 0, 1)])
def test_im2col_gemm_equals_direct(geom):
    kh, kw, s, p, g = geom
    rng = np.random.default_rng(0)
    H = 13 if kh < 11 else 27
    x = rng.random((2, H, H, 4 * g)).astype(np.float32)
    M = 6 * g
    W = rng.standard_normal((M, kh * kw * 4)).astype(np.float32)
    y1 = infer.conv_forward(x, W, None, kh, kw, s, p, g, apply_relu=False, bf16=False)
    y2 = infer.conv_direct(x.astype(np.float64), W, kh, kw, s, p, g)
    assert np.allclose(y1, y2, rtol=1e-12, atol=1e-11)


def test_conv_1x1_identity():
    x = np.random.default_rng(1).random((2, 5, 5, 4)).astype(np.float32)
    W = np.eye(4, dtype=np.float32)
    y = infer.conv_forward(x, W, None, 1, 1, 1, 0, 1, apply_relu=False, bf16=False)
    assert np.array_equal(y, x.astype(np.float64))


def test_bf16_round_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 1.0 + 2 ** -9, -2.5], dtype=np.float32)
    # 1+2^-8 is a tie -> even (1.0); 1+3*2^-8 tie -> 1+2^-6 ... check by definition of bf16 spacing
    got = infer.bf16_round(x)
    assert got[0] == 1.0 and got[1] == 1.0 and got[2] == np.float32(1.0 + 2 ** -6)
    assert got[3] == 1.0 and got[4] == -2.5


def test_pool_and_lrn_special_cases():
    x = np.full((1, 7, 7, 3), 2.5)
    assert (infer.maxpool(x) == 2.5).all() and infer.maxpool(x).shape == (1, 3, 3, 3)
    assert (infer.lrn(np.zeros((1, 2, 2, 8))) == 0).all()


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden(name):
    rows = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].strip()
        if line:
            k, *v = line.split()
            rows[k] = [float(t) for t in v]
    return rows


def test_lrn_hand_computed_cases():
    """tests/golden/lrn_maxpool_hand.txt: closed-form LRN values that pin the
    window (+-2 channels, clipped at the channel edges, no wrap-around), the
    alpha/n scaling, beta and k of reading C-20."""
    g = _golden("lrn_maxpool_hand.txt")
    for case in ("lrnA", "lrnB"):
        a = np.array(g[case + "_in"]).reshape(1, 1, 1, -1)
        got = infer.lrn(a).ravel()
        assert np.allclose(got, g[case + "_out"], rtol=1e-12, atol=0), (case, got)
    # the same pixel repeated over a 2x3 image and a batch of 2: LRN is per pixel
    a = np.tile(np.array(g["lrnA_in"]), (2, 2, 3, 1))
    assert np.allclose(infer.lrn(a), np.tile(np.array(g["lrnA_out"]), (2, 2, 3, 1)), rtol=1e-12)


def test_maxpool_hand_computed_case():
    """3x3 / stride 2 max-pool of a non-constant 5x5x2 image (golden file):
    window size, stride and the no-padding output size 2x2."""
    g = _golden("lrn_maxpool_hand.txt")
    h, w = np.meshgrid(np.arange(5), np.arange(5), indexing="ij")
    x = np.stack([5 * h + w, -(5 * h + w)], axis=-1).astype(np.float64)[None]
    y = infer.maxpool(x, 3, 2)
    assert y.shape == (1, 2, 2, 2)
    assert np.array_equal(y[0, :, :, 0].ravel(), g["pool_c0"])
    assert np.array_equal(y[0, :, :, 1].ravel(), g["pool_c1"])
    # batch of two distinct images: each pooled on its own
    x2 = np.concatenate([x, x + 100.0])
    y2 = infer.maxpool(x2, 3, 2)
    assert np.array_equal(y2[1], y[0] + 100.0)


def test_fc_abs_scale_hand_computed():
    """sum_j |W_ij a_j| + |v_i| on a 2x2 example worked by hand:
    row 0: |1*1| + |-2*-1| + |0.5| = 3.5; row 1: |0| + |3*-1| + |-0.25| = 3.25."""
    W = np.array([[1.0, -2.0], [0.0, 3.0]])
    a = np.array([[1.0, -1.0]])
    v = np.array([0.5, -0.25])
    assert np.array_equal(infer.fc_abs_scale(W, a, v), [[3.5, 3.25]])
    import scipy.sparse as sp
    assert np.array_equal(infer.fc_abs_scale(sp.csr_matrix(W), a, v), [[3.5, 3.25]])


def test_table4_memory_column():
    """P:L584-596 Table 4 'Memory (MB)' = OUT(i,B) = 4 B x elements x B, in MiB,
    reproduced to the printed 2 decimals for all 13 layers at B=16 and B=256
    (tests/golden/table4_memory_mib.txt).  Pins the C-19 conv/pool geometry."""
    table4 = _golden("table4_memory_mib.txt")
    rows = infer.alexnet_layer_shapes()
    assert [n for n, _ in rows] == list(table4)
    for name, elems in rows:
        for B, printed in zip((16, 256), table4[name]):
            mib = 4 * elems * B / 2 ** 20
            assert abs(mib - printed) <= 0.005 + 1e-9, (name, B, mib, printed)


# ---------------------------------------------------------- planner

def _random_problem(rng, f, Bmax, latency=False):
    time = []
    for i in range(f):
        base = rng.uniform(0.5, 5)
        slope = rng.uniform(0.05, 2)
        time.append({B: base + slope * B ** rng.uniform(0.6, 1.1) for B in range(1, Bmax + 1)})
    inb = [rng.randint(1, 20) for _ in range(f)]
    outb = [rng.randint(1, 20) for _ in range(f)]
    ws = [rng.randint(0, 10) for _ in range(f)]
    tot = rng.randint(20, 40 * Bmax)
    lat = rng.uniform(5, 60) if latency else None
    return planner.Problem(time, inb, outb, ws, tot, lat)


@pytest.mark.parametrize("seed", range(600))
def test_dp_equals_brute_force(seed):
    rng = random.Random(seed)
    f = rng.randint(1, 4)
    Bmax = rng.randint(1, 8)
    p = _random_problem(rng, f, Bmax, latency=(seed % 3 == 0))
    a = planner.dp_plan(p, Bmax)
    b = planner.brute_force(p, Bmax)
    assert (a is None) == (b is None)
    if a is not None:
        assert math.isclose(a.per_image, b.per_image, rel_tol=1e-12)
        # the DP's plan is itself a feasible chain with the claimed cost
        assert math.isclose(planner.chain_cost(p, a.batches), a.time, rel_tol=1e-12)
        for x, y in zip(a.batches, a.batches[1:]):
            assert x <= y and y % x == 0
        fx = planner.fixed_batch(p, Bmax)
        if fx is not None:                                    # dominance
            assert a.per_image <= fx.per_image * (1 + 1e-12)


def test_single_layer_is_argmin_time_per_image():
    rng = random.Random(5)
    p = _random_problem(rng, 1, 16)
    p.tot = 10 ** 9
    pl = planner.dp_plan(p, 16)
    assert pl.per_image == min(p.time[0][B] / B for B in range(1, 17))


def test_remainder_replan():
    """K=64, B*=60 -> one round of 60, then plan again for 4."""
    f = 2
    Bmax = 64
    time = [{B: 1.0 + 0.01 * B for B in range(1, Bmax + 1)} for _ in range(f)]
    # memory: 1 byte per image in and out; TOT admits B <= 60 at the last layer
    p = planner.Problem(time, [0, 1], [1, 1], [0, 0], tot=120)
    segs, total = planner.plan_requests(p, 64)
    assert [(r, pl.batches[-1]) for r, pl in segs] == [(1, 60), (1, 4)]


def test_table_size_estimate():
    """14 layers x 64 batch sizes x (14 MB / 100 KB = 140) steps,
    4-byte cells -> 501,760 B = 490 KiB, 'around 500KB'."""
    nb = planner.table_bytes(14, 64, 14_000_000, 100_000)
    assert nb == 501_760 and abs(nb / 1024 - 500) < 15


def test_table5_columns_vs_rule():
    """P:L779-800 Table 5 vs the recurrence's monotone/divisibility rule
    (P:L675-679): the 1.5x and 2x columns satisfy it, the 2.5x column does not
    (reading C-28)."""
    col15 = [2, 4, 4, 4, 4, 4, 4, 4, 4, 4, 64, 64, 64]
    col2 = [4] * 10 + [64] * 3
    col25 = [6] * 9 + [32, 60, 60, 60]
    ok = lambda c: all(b <= B and B % b == 0 for b, B in zip(c, c[1:]))
    assert ok(col15) and ok(col2) and not ok(col25)


def test_unconstrained_memory_gives_per_layer_optimum_shape():
    # Time superlinear per image -> larger batches never help: all-ones plan
    time = [{B: B * 1.0 + 0.1 * B * B for B in range(1, 9)} for _ in range(3)]
    p = planner.Problem(time, [1, 1, 1], [1, 1, 1], [0, 0, 0], tot=10 ** 9)
    assert planner.dp_plan(p, 8).batches == [1, 1, 1]
    # strongly sublinear time -> the largest batch everywhere
    time = [{B: 10.0 + 0.01 * B for B in range(1, 9)} for _ in range(3)]
    p = planner.Problem(time, [1, 1, 1], [1, 1, 1], [0, 0, 0], tot=10 ** 9)
    assert planner.dp_plan(p, 8).batches == [8, 8, 8]


@pytest.mark.parametrize("bh,bw", [(4, 64), (16, 32), (32, 128)])
def test_algorithm2_blocked_inference_equals_dense_product(bh, bw):
    """Alg. 2 step by step (decode a stored row, arrange bh x bw, multiply the
    input slice, accumulate the output slice) = the plain product W_q a."""
    from oracle import compress, infer
    W = synth.random_matrix(64, 256, seed=bh + bw, scale=0.05)
    v = synth.random_matrix(1, 64, seed=2).ravel()
    c = compress.compress_layer(W, 0.15, 5, 4, v, bh=bh, bw=bw)
    a = synth.random_activations(256, 5, seed=4)
    y = infer.fc_forward_blocked(c.layer, a, v, apply_relu=True)
    ref = infer.fc_forward(c.dense_q(), a, v, apply_relu=True)
    assert np.allclose(y, ref, rtol=1e-12, atol=1e-12)
