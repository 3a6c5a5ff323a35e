"""GPU parity of the CONV path: Huffman decode of the filter
matrix -> dense bf16 -> im2col -> tcgen05 GEMM (fp32 accumulate) -> bias ->
ReLU -> LRN -> max-pool, against the oracle's bf16-emulating fp64 convolution
(O9, readings C-18..C-21) on the SAME fp32 input (per-layer isolation, C-21).
Gate: ||y_gpu - y_ref||_inf / ||y_ref||_inf <= 1e-4 (north_star)."""
import numpy as np
import pytest

import synth
from oracle import cdni, compress, infer

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    return torch, torch.device("cuda:0")


def bf16_bits(x):
    """fp32 -> bf16 bit patterns (RNE), via the oracle's rounding."""
    return (infer.bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)


def rel_err(y, ref):
    return np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-30)


@pytest.mark.parametrize("M,N,K,relu", [(128, 96, 64, False), (300, 128, 384, True), (257, 192, 1216, False),
                                        (640, 384, 2304, True), (77, 40, 128, False), (1, 16, 64, False)])
def test_tcgen05_gemm_hook(torch_dev, M, N, K, relu):
    """The tensor-core GEMM alone: bf16 operands, fp32 accumulate, vs fp64."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    rng = np.random.default_rng(M * 7 + N)
    a = rng.standard_normal((M, K), dtype=np.float32)
    w = rng.standard_normal((N, K), dtype=np.float32)
    bias = rng.standard_normal(N, dtype=np.float32)
    ta = torch.from_numpy(bf16_bits(a).view(np.int16)).to(dev)
    tw = torch.from_numpy(bf16_bits(w).view(np.int16)).to(dev)
    tb = torch.from_numpy(bias).to(dev)
    out = torch.full((M, N), float("nan"), dtype=torch.float32, device=dev)
    cdn.debug_gemm_bf16(ta, M, tw, N, K, tb, relu, out, N)
    torch.cuda.synchronize()
    ref = infer.bf16_round(a).astype(np.float64) @ infer.bf16_round(w).astype(np.float64).T + bias
    if relu:
        ref = np.maximum(ref, 0)
    y = out.cpu().numpy()
    assert np.isfinite(y).all()
    assert rel_err(y, ref) <= 1e-5
    scale = np.abs(infer.bf16_round(a)).astype(np.float64) @ np.abs(infer.bf16_round(w)).astype(np.float64).T
    assert (np.abs(y - ref) <= 2 * K * 2.0 ** -24 * scale + 1e-6).all()


_CACHE = {}


def conv_case(i, density=None, quantizer="linear"):
    spec = synth.ALEXNET_CONV[i]
    d = spec.density if density is None else density
    key = (i, d, quantizer)
    if key not in _CACHE:
        W, v = synth.fc_weights(spec, 0)
        c = compress.compress_layer(W, d, spec.r, spec.k, v, quantizer=quantizer)
        _CACHE[key] = (spec, c, cdni.serialize([c.layer]), v)
    return _CACHE[key]


IN_HW = [227, 27, 13, 13, 13]


def conv_input(i, B):
    spec = synth.ALEXNET_CONV[i]
    if i == 0:
        return synth.conv_inputs(B, 227, 3, seed=0)
    rng = np.random.default_rng(100 + i)
    x = rng.standard_normal((B, IN_HW[i], IN_HW[i], spec.in_ch), dtype=np.float32)
    return np.maximum(x, np.float32(0))


def oracle_conv(spec, c, v, x):
    y = infer.conv_forward(x, c.dense_q(), v, spec.kh, spec.kw, spec.stride, spec.pad, spec.groups,
                           apply_relu=True, bf16=True)
    if spec.lrn:
        y = infer.lrn(y)
    if spec.pool:
        y = infer.maxpool(y, 3, 2)
    return y


@pytest.mark.parametrize("i,B,density,quantizer", [(0, 2, None, "linear"), (1, 2, None, "linear"),
                                                   (2, 3, None, "linear"), (3, 2, None, "linear"),
                                                   (4, 2, None, "linear"),
                                                   # the paper's 63% conv5, k-means
                                                   (4, 2, 0.63, "kmeans")])
@pytest.mark.parametrize("s2d", ["1", "0"])
def test_alexnet_conv_layer_vs_oracle(torch_dev, monkeypatch, i, B, density, quantizer, s2d):
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    if s2d == "0" and i != 0:
        pytest.skip("the space-to-depth switch concerns conv1 only")
    spec, c, buf, v = conv_case(i, density, quantizer)
    x = conv_input(i, B)
    monkeypatch.setenv("CDN_CONV_S2D", s2d)
    m = cdn.Model(0)
    m.load_layer(buf, cdn.LayerDesc.conv(spec.in_ch, IN_HW[i], IN_HW[i], spec.kh, spec.kw, spec.stride, spec.pad,
                                         spec.groups, relu=True, lrn=spec.lrn, pool_k=3 if spec.pool else 0,
                                         pool_s=2 if spec.pool else 0))
    monkeypatch.delenv("CDN_CONV_S2D")
    oh, ow, oc = m.out_shape(0)
    # stride-1 layers with channel groups of >= 8 channels (conv2-5) run the
    # implicit GEMM (TMA im2col, no patch matrix); conv1 (3 channels, stride 4)
    # the same after a space-to-depth regrouping (4 x 4 x 3 = 48 channels, a 3 x 3
    # kernel), or the explicit im2col when that is switched off
    want = ("k_gemm_bf16 (conv, space-to-depth, implicit im2col)" if s2d == "1" else "k_gemm_bf16 (conv)") \
        if i == 0 else "k_gemm_bf16 (conv, implicit im2col)"
    assert m.kernel_name(0, B) == want
    xd = torch.from_numpy(x).to(dev)
    yd = torch.full((B, oh, ow, oc), float("nan"), dtype=torch.float32, device=dev)
    m.conv_forward(0, xd, B, yd)
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    ref = oracle_conv(spec, c, v, x)
    assert y.shape == ref.shape
    assert np.isfinite(y).all()
    e = rel_err(y, ref)
    assert e <= TOL, e
    m.close()


def test_conv_rejects_fc_entry_and_bad_geometry(torch_dev):
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    spec, c, buf, v = conv_case(2)
    m = cdn.Model(0)
    with pytest.raises(cdn.CDNError) as e:
        m.load_layer(buf, cdn.LayerDesc.conv(spec.in_ch, 13, 13, 5, 5, 1, 1))   # kh*kw*C != cols
    assert e.value.name == "CDN_E_SHAPE"
    m.load_layer(buf, cdn.LayerDesc.conv(spec.in_ch, 13, 13, 3, 3, 1, 1))
    x = torch.zeros((spec.in_ch, 1), device=dev)
    with pytest.raises(cdn.CDNError):
        m.layer_forward(0, x, 1, 1, x, 1)
    m.close()


def test_c4_alexnet_end_to_end(torch_dev):
    """Config C4: conv1-conv5 (84/38/35/37/37 %, r = k = 8) + fc6/fc7/fc8, batch
    64 of 227x227x3 U(0,1) images through cdn_model_infer.  Every layer is
    gated at 1e-4 against the oracle on the GPU's own input for that layer
    (per-layer isolation, C-21); infer's scores equal the layer-by-layer GPU
    chain; the chained bf16 error against the all-oracle chain is reported and
    loosely bounded (SURVEY [EST-5])."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    B = 64
    cfg = synth.CONFIGS["C4"]
    m = cdn.Model(0)
    comps = []
    hw = 227
    for i, spec in enumerate(cfg.conv):
        _, c, buf, v = conv_case(i)
        m.load_layer(buf, cdn.LayerDesc.conv(spec.in_ch, hw, hw, spec.kh, spec.kw, spec.stride, spec.pad,
                                             spec.groups, relu=True, lrn=spec.lrn, pool_k=3 if spec.pool else 0,
                                             pool_s=2 if spec.pool else 0))
        hw = m.out_shape(i)[0]
        comps.append(("conv", spec, c, v))
    for spec in cfg.fc:
        W, v = synth.fc_weights(spec, cfg.seed)
        c = compress.compress_layer(W, spec.density, spec.r, spec.k, v)
        m.load_layer(cdni.serialize([c.layer]), cdn.LayerDesc.fc(spec.relu))
        comps.append(("fc", spec, c, v))
    x = synth.conv_inputs(B, 227, 3, seed=cfg.seed)
    m.set_plan([B] * len(comps))
    scores = np.zeros((B, cfg.fc[-1].rows), np.float32)
    m.infer(x, B, scores, on_device=False)

    # layer by layer on the GPU, each gated against the oracle on the same input
    cur = torch.from_numpy(x).to(dev)
    chain = x
    for li, (kind, spec, c, v) in enumerate(comps):
        if kind == "conv":
            oh, ow, oc = m.out_shape(li)
            y = torch.empty((B, oh, ow, oc), dtype=torch.float32, device=dev)
            m.conv_forward(li, cur, B, y)
            torch.cuda.synchronize()
            ref = oracle_conv(spec, c, v, cur.cpu().numpy())
            chain = oracle_conv(spec, c, v, chain).astype(np.float32)
            yn = y.cpu().numpy()
        else:
            a = cur.reshape(B, -1)
            xf = a.T.contiguous()
            ld = (B + 3) // 4 * 4
            xp = torch.zeros((xf.shape[0], ld), dtype=torch.float32, device=dev)
            xp[:, :B] = xf
            yf = torch.zeros((spec.rows, ld), dtype=torch.float32, device=dev)
            m.layer_forward(li, xp, ld, B, yf, ld)
            torch.cuda.synchronize()
            y = yf[:, :B].T.contiguous()
            ref = infer.fc_forward(sparse_q(c), a.cpu().numpy(), v, apply_relu=spec.relu)
            chain = infer.fc_forward(sparse_q(c), chain.reshape(B, -1), v, apply_relu=spec.relu).astype(np.float32)
            yn = y.cpu().numpy()
        e = rel_err(yn, ref)
        assert e <= TOL, (li, e)
        cur = y
    assert np.array_equal(scores, cur.cpu().numpy())
    e2e = rel_err(scores, chain)
    print(f"C4 end-to-end chained error vs oracle chain: {e2e:.2e}")
    assert e2e <= 2e-2
    m.close()


def sparse_q(c):
    import scipy.sparse as sp
    r, col = np.nonzero(c.mask)
    vals = c.layer.codebook[c.q[r, col]].astype(np.float32)
    return sp.csr_matrix((vals, (r, col)), shape=c.mask.shape)


def test_c4_variable_batch_plan_under_budget(torch_dev):
    """SURVEY NEXT #1 on the device: AlexNet conv1-5 + fc6-8 under TOT = 48 MiB
    for K = 32 images: the planner's divisor chain (the DP of P:L694-720, or the
    best fixed batch when that runs faster within the executor's memory).  Infer
    with it: the
    library's inference scratch stays within TOT (reading C-36), the scores
    match the oracle chain (bf16 CONV emulation, C-21) within the bound of the
    fixed-batch end-to-end test, and equal the fixed-batch GPU scores up to
    rounding."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    cfg = synth.CONFIGS["C4"]
    m = cdn.Model(0)
    comps = []
    hw = 227
    for i, spec in enumerate(cfg.conv):
        _, c, buf, v = conv_case(i)
        m.load_layer(buf, cdn.LayerDesc.conv(spec.in_ch, hw, hw, spec.kh, spec.kw, spec.stride, spec.pad,
                                             spec.groups, relu=True, lrn=spec.lrn, pool_k=3 if spec.pool else 0,
                                             pool_s=2 if spec.pool else 0))
        hw = m.out_shape(i)[0]
        comps.append(("conv", spec, c, v))
    for spec in cfg.fc:
        W, v = synth.fc_weights(spec, cfg.seed)
        c = compress.compress_layer(W, spec.density, spec.r, spec.k, v)
        m.load_layer(cdni.serialize([c.layer]), cdn.LayerDesc.fc(spec.relu))
        comps.append(("fc", spec, c, v))
    K = 32
    tot = 48 << 20  # (tight enough that conv1's per-image footprint caps the conv batch)
    m.set_memory_budget(tot)
    batches, predicted = m.plan(K)
    print("C4 plan under 48 MiB:", batches, f"{predicted:.3f} ms for {K} images")
    assert all(batches[i + 1] % batches[i] == 0 for i in range(len(batches) - 1))
    x = synth.conv_inputs(K, 227, 3, seed=1)
    s_plan = np.zeros((K, 1000), np.float32)
    m.release_scratch()
    m.scratch_bytes(reset_peak=True)
    m.infer(x, K, s_plan, on_device=False)
    _, peak = m.scratch_bytes()
    print(f"C4 scratch peak {peak / 2**20:.2f} MiB of {tot / 2**20:.0f} MiB")
    assert peak <= tot
    # the oracle chain (fp64 layers; CONV on bf16-rounded inputs and weights, C-21)
    chain = x
    for kind, spec, c, v in comps:
        if kind == "conv":
            chain = oracle_conv(spec, c, v, chain).astype(np.float32)
        else:
            chain = infer.fc_forward(sparse_q(c), chain.reshape(K, -1), v, apply_relu=spec.relu).astype(np.float32)
    e = rel_err(s_plan, chain)
    print(f"C4 planned scores vs oracle chain: {e:.2e}")
    assert e <= 2e-3
    m.set_plan([K] * len(batches))
    s_fix = np.zeros((K, 1000), np.float32)
    m.infer(x, K, s_fix, on_device=False)
    assert rel_err(s_plan, s_fix) <= 1e-4
    m.close()


@pytest.mark.parametrize("i", [0, 1, 2, 3, 4])
def test_conv_layer_decode_bit_exact(torch_dev, i):
    """SURVEY §4 T3 on the CONV layers of C4 (r = k = 8, 256-entry codebooks,
    8-bit gaps, densities 84/38/35/37/37 %): cdn_layer_decode's tokens (row,
    column, symbol, codebook value) equal the oracle's pre-encoding streams
    bit for bit, and the real tokens are exactly the kept weights."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    spec, c, buf, v = conv_case(i)
    m = cdn.Model(0)
    m.load_layer(buf, cdn.LayerDesc.conv(spec.in_ch, IN_HW[i], IN_HW[i], spec.kh, spec.kw, spec.stride, spec.pad,
                                         spec.groups, relu=True, lrn=spec.lrn, pool_k=3 if spec.pool else 0,
                                         pool_s=2 if spec.pool else 0))
    n = m.decode_count(0)
    assert n == c.val_tokens.size
    row = torch.empty(n, dtype=torch.int32, device=dev)
    col = torch.empty(n, dtype=torch.int32, device=dev)
    sym = torch.empty(n, dtype=torch.uint8, device=dev)
    val = torch.empty(n, dtype=torch.float32, device=dev)
    m.decode(0, row, col, sym, val)
    torch.cuda.synchronize()
    R, Cc, S, V = (t.cpu().numpy() for t in (row, col, sym, val))
    er = np.repeat(np.arange(c.row_tokens.size), c.row_tokens)
    # columns by the C-01 prefix sum within each row
    ec = np.empty(n, np.int64)
    o = 0
    for t in c.row_tokens:
        ec[o:o + t] = np.cumsum(c.gap_tokens[o:o + t] + 1) - 1
        o += t
    assert np.array_equal(R, er)
    assert np.array_equal(Cc, ec)
    assert np.array_equal(S, c.val_tokens.astype(np.uint8))
    assert np.array_equal(V.view(np.uint32), c.layer.codebook[c.val_tokens].astype(np.float32).view(np.uint32))
    real = S != 0
    assert real.sum() == c.mask.sum() and c.mask[R[real], Cc[real]].all()
    m.close()


def test_c4_planner_goes_variable_with_room(torch_dev):
    """With room for the FC layers' batch but not for the CONV trunk at it (K = 64,
    some TOT between 64 and 192 MiB) the DP's variable-batch chain -- CONV layers at a smaller batch than the FC layers,
    the shape of the paper's Table 5 -- beats every fixed batch the executor
    can run within TOT (profiles/r02_variable_batch_c4.jsonl: 0.56 vs 0.67 ms)."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    cfg = synth.CONFIGS["C4"]
    m = cdn.Model(0)
    hw = 227
    for i, spec in enumerate(cfg.conv):
        _, c, buf, v = conv_case(i)
        m.load_layer(buf, cdn.LayerDesc.conv(spec.in_ch, hw, hw, spec.kh, spec.kw, spec.stride, spec.pad,
                                             spec.groups, relu=True, lrn=spec.lrn, pool_k=3 if spec.pool else 0,
                                             pool_s=2 if spec.pool else 0))
        hw = m.out_shape(i)[0]
    for spec in cfg.fc:
        W, v = synth.fc_weights(spec, cfg.seed)
        c = compress.compress_layer(W, spec.density, spec.r, spec.k, v)
        m.load_layer(cdni.serialize([c.layer]), cdn.LayerDesc.fc(spec.relu))
    # the budget where that happens moves with the executor's footprint (bf16
    # levels between CONV layers shrank it: at 192 MiB a fixed 64 now fits), so
    # the budgets between "nothing but small batches" and "64 everywhere" are scanned
    variable = []
    for mib in (64, 80, 96, 112, 128, 144, 160, 176, 192):
        m.set_memory_budget(mib << 20)
        batches, predicted = m.plan(64)
        print(f"C4 plan under {mib} MiB:", batches, f"{predicted:.3f} ms for 64 images")
        assert all(batches[i + 1] % batches[i] == 0 for i in range(len(batches) - 1))
        if batches[0] < batches[-1]:
            variable.append(mib)
    assert variable, "no budget at which the planner runs the CONV layers at a smaller batch than the FC layers"
    m.close()


def test_small_conv_net_bf16_chain_vs_layers(torch_dev):
    """A CONV trunk off AlexNet's shapes, through cdn_model_infer and layer by
    layer: (a) 8 -> 16 channels, LRN + pool, feeding a layer whose 16-channel
    groups are padded to 64 (k_lrn_pool_rows writes the padding zeros of the
    bf16 level); (b) 16 -> 64, no LRN / pool, feeding a 64-channel layer (the
    halo GEMM's epilogue writes the bf16 level); (c) 64 -> 24 in two groups,
    pool only, feeding (d) 24 -> 40 (12-channel groups: not a multiple of 8, so
    the level stays fp32 and the layer converts its own input); then an FC
    layer.  Each layer is gated against the oracle on the GPU's own input, and
    infer's scores equal the layer-by-layer chain bit for bit (rounding to bf16
    in the producer is the consumer's own first step, C-21)."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    specs = [synth.ConvSpec("a", 16, 8, 3, 3, 1, 1, 1, 0.6, lrn=True, pool=True, seed_offset=301),
             synth.ConvSpec("b", 64, 16, 3, 3, 1, 1, 1, 0.5, seed_offset=302),
             synth.ConvSpec("c", 24, 64, 5, 5, 1, 2, 2, 0.5, pool=True, seed_offset=303),
             synth.ConvSpec("d", 40, 24, 3, 3, 1, 1, 2, 0.7, seed_offset=304)]
    B, hw0 = 5, 21
    m = cdn.Model(0)
    comps = []
    hw = hw0
    for i, spec in enumerate(specs):
        W, v = synth.fc_weights(spec, 0)
        c = compress.compress_layer(W, spec.density, spec.r, spec.k, v)
        m.load_layer(cdni.serialize([c.layer]),
                     cdn.LayerDesc.conv(spec.in_ch, hw, hw, spec.kh, spec.kw, spec.stride, spec.pad, spec.groups,
                                        relu=True, lrn=spec.lrn, pool_k=3 if spec.pool else 0,
                                        pool_s=2 if spec.pool else 0))
        hw = m.out_shape(i)[0]
        comps.append((spec, c, v))
    feat = int(np.prod(m.out_shape(len(specs) - 1)))
    fspec = synth.FCSpec("fc", 37, feat, 0.2, 0.05, relu=False, seed_offset=305)
    Wf, vf = synth.fc_weights(fspec, 0)
    cf = compress.compress_layer(Wf, fspec.density, fspec.r, fspec.k, vf)
    m.load_layer(cdni.serialize([cf.layer]), cdn.LayerDesc.fc(False))
    rng = np.random.default_rng(77)
    x = rng.random((B, hw0, hw0, 8), dtype=np.float32)
    m.set_plan([B] * (len(specs) + 1))
    scores = np.zeros((B, 37), np.float32)
    for _ in range(3):  # eager, captured, replayed
        m.infer(x, B, scores, on_device=False)
    cur = torch.from_numpy(x).to(dev)
    for li, (spec, c, v) in enumerate(comps):
        oh, ow, oc = m.out_shape(li)
        y = torch.empty((B, oh, ow, oc), dtype=torch.float32, device=dev)
        m.conv_forward(li, cur, B, y)
        torch.cuda.synchronize()
        ref = oracle_conv(spec, c, v, cur.cpu().numpy())
        e = rel_err(y.cpu().numpy(), ref)
        assert e <= TOL, (li, e)
        cur = y
    a = cur.reshape(B, -1)
    ld = (B + 3) // 4 * 4
    xp = torch.zeros((feat, ld), dtype=torch.float32, device=dev)
    xp[:, :B] = a.T
    yf = torch.zeros((37, ld), dtype=torch.float32, device=dev)
    m.layer_forward(len(specs), xp, ld, B, yf, ld)
    torch.cuda.synchronize()
    ref = infer.fc_forward(sparse_q(cf), a.cpu().numpy(), vf, apply_relu=False)
    yn = yf[:, :B].T.contiguous().cpu().numpy()
    assert rel_err(yn, ref) <= TOL
    assert np.array_equal(scores, yn)
    # the same request in two phases of the trunk (variable batch: 2 + 2 + 1 is not a chain; 1 then 5)
    m.set_plan([1] * len(specs) + [B])
    s2 = np.zeros_like(scores)
    m.infer(x, B, s2, on_device=False)
    assert rel_err(s2, scores) <= 1e-5
    m.close()
