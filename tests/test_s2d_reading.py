"""Reading C-37: a strided CONV with no padding equals a
stride-1 CONV over the space-to-depth regrouped input with the regrouped
kernel -- the same products, reordered.  The product's conv1 path (conv.cu
k_s2d_bf16 + the implicit GEMM, api.cpp's K map) relies on this; here it is
checked on the CPU against the oracle's direct convolution loop (no GPU, no
product code): regrouping + stride-1 convolution reproduce the strided one
exactly in fp64, and the K map (r, s, c) -> ((r//s_)*Ks + s//s_)*Cp +
((r%s_)*s_ + s%s_)*C + c places every filter tap where the regrouped kernel
reads it."""
import numpy as np
import pytest

from oracle import infer


def s2d_input(x, st, cp):
    """[B][H][W][C] -> [B][ceil(H/st)][ceil(W/st)][cp]: channel (dy*st + dx)*C + c of
    super-pixel (Y, X) = x[st*Y + dy][st*X + dx][c] (zero outside, zero past st*st*C)."""
    B, H, W, C = x.shape
    Hs, Ws = -(-H // st), -(-W // st)
    out = np.zeros((B, Hs, Ws, cp))
    for Y in range(Hs):
        for X in range(Ws):
            for dy in range(st):
                for dx in range(st):
                    yy, xx = st * Y + dy, st * X + dx
                    if yy < H and xx < W:
                        c0 = (dy * st + dx) * C
                        out[:, Y, X, c0:c0 + C] = x[:, yy, xx, :]
    return out


def kmap(kh, kw, C, st, cp):
    ks = -(-kh // st)
    m = np.empty(kh * kw * C, dtype=np.int64)
    for r in range(kh):
        for s in range(kw):
            for c in range(C):
                k = (r * kw + s) * C + c                       # the decoded K index (C-18)
                m[k] = ((r // st) * ks + s // st) * cp + ((r % st) * st + s % st) * C + c
    return m, ks


@pytest.mark.parametrize("H,kh,st,C,M", [(23, 11, 4, 3, 5), (27, 11, 4, 3, 2), (13, 5, 2, 3, 3), (16, 4, 4, 4, 2),
                                        (19, 7, 2, 4, 3)])
def test_space_to_depth_equals_strided_conv(H, kh, st, C, M):
    rng = np.random.default_rng(H * 100 + kh)
    x = rng.standard_normal((2, H, H, C))
    Wq = rng.standard_normal((M, kh * kh * C))
    ref = infer.conv_direct(x, Wq, kh, kh, st, 0, 1)           # the paper's convolution (stride st)
    cp = ((st * st * C + 7) // 8) * 8
    m, ks = kmap(kh, kh, C, st, cp)
    assert len(set(m.tolist())) == m.size                      # the map is injective
    Ws = np.zeros((M, ks * ks * cp))
    Ws[:, m] = Wq                                              # regrouped kernel (taps past kh stay 0)
    xs = s2d_input(x, st, cp)
    got = infer.conv_direct(xs, Ws, ks, ks, 1, 0, 1)           # stride-1 over super-pixels
    Ho = infer.conv_out_hw(H, kh, st, 0)
    assert got.shape[1] >= Ho and got.shape[2] >= Ho
    # the product's rule: the super-pixel output grid equals the strided one
    if -(-H // st) - ks + 1 == Ho:
        assert got.shape[1:3] == (Ho, Ho)
    np.testing.assert_allclose(got[:, :Ho, :Ho], ref, rtol=1e-12, atol=1e-12)


def test_alexnet_conv1_geometry():
    """AlexNet conv1 (227 x 227 x 3, 11 x 11, stride 4, no padding, Table 4's 55 x 55 output):
    57 x 57 super-pixels of 48 channels (padded to 64) and a 3 x 3 super-kernel give exactly
    the 55 x 55 grid, the K map fills 363 of the 576 padded K positions."""
    H, kh, st, C = 227, 11, 4, 3
    Hs, ks = -(-H // st), -(-kh // st)
    assert (Hs, ks) == (57, 3)
    assert Hs - ks + 1 == infer.conv_out_hw(H, kh, st, 0) == 55
    m, _ = kmap(kh, kh, C, st, 64)
    assert m.size == 363 and m.max() < ks * ks * 64 and len(set(m.tolist())) == 363
