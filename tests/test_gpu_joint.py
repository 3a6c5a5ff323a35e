"""GPU parity of the merged-stream kernels (joint.cu) against the fp64 oracle:
the small-batch k_fc_j (B <= 4) on every FC config layer at B = 1..4, the edge
fixtures with narrow joint LUTs (many slow-path tokens) and column groups
Q = 1, 2, 4 (the lane split and the cross-CTA partial sums); the medium-batch
k_fc_jm (B = 5..128, groups of <= 32 images) on the same layers and fixtures;
bit-identical repeated launches (fixed reduction orders).  Tolerance: ||dy||_inf / ||y||_inf <= 1e-4
(north_star) and the elementwise fp32 accumulation bound."""
import zlib

import numpy as np
import pytest

import synth
from oracle import cdni, compress, infer

pytestmark = pytest.mark.gpu

_CACHE = {}


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    return torch, torch.device("cuda:0")


def layer(key, W, d, r, k, v):
    if key not in _CACHE:
        c = compress.compress_layer(W, d, r, k, v)
        _CACHE[key] = (c, cdni.serialize([c.layer]))
    return _CACHE[key]


def config_layer(cfg, i):
    spec = synth.CONFIGS[cfg].fc[i]
    W, v = synth.fc_weights(spec, synth.CONFIGS[cfg].seed)
    c, buf = layer((cfg, i), W, spec.density, spec.r, spec.k, v)
    return spec, c, buf, v


def load(buf, relu, monkeypatch=None, jl=None, jq=None):
    import paper_1711_00244_b200 as cdn
    if monkeypatch is not None:
        if jl is not None:
            monkeypatch.setenv("CDN_JL", str(jl))
        if jq is not None:
            monkeypatch.setenv("CDN_JQ", str(jq))
    m = cdn.Model(0)
    m.load_layer(buf, cdn.LayerDesc.fc(relu))
    if monkeypatch is not None:
        monkeypatch.delenv("CDN_JL", raising=False)
        monkeypatch.delenv("CDN_JQ", raising=False)
    return m


def forward(torch, dev, m, a, N, stream=0):
    B = a.shape[0]
    x = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)
    y = torch.full((N, B), float("nan"), dtype=torch.float32, device=dev)
    m.layer_forward(0, x, B, B, y, B, stream=stream)
    torch.cuda.synchronize()
    return y.cpu().numpy().T


def check(torch, dev, m, c, v, a, relu, kernel="k_fc_j"):
    assert m.kernel_name(0, a.shape[0]) == kernel
    y = forward(torch, dev, m, a, c.layer.rows)
    ref = infer.fc_forward(c.dense_q(), a, v, apply_relu=relu)
    assert np.isfinite(y).all()
    e = np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-30)
    assert e <= 1e-4, e
    scale = infer.fc_abs_scale(c.dense_q(), a, v)
    kmax = max(1, int(c.row_tokens.max()))
    elem = (np.abs(y - ref) / np.maximum(scale, 1e-30)).max()
    assert elem <= 2 * kmax * 2.0 ** -24 + 1e-12, elem
    return y


CONFIG_LAYERS = [("C1", 0), ("C2", 0), ("C3", 1), ("C3", 2), ("C5", 0), ("C5", 1), ("C5", 2)]


@pytest.mark.parametrize("cfg,i", CONFIG_LAYERS)
def test_config_layers_b1_to_b4(torch_dev, cfg, i):
    torch, dev = torch_dev
    spec, c, buf, v = config_layer(cfg, i)
    m = load(buf, spec.relu)
    for B in (1, 2, 3, 4):
        if m.kernel_name(0, B) != "k_fc_j":  # x slice of B > 1 larger than shared memory
            assert B > 1
            continue
        check(torch, dev, m, c, v, synth.fc_inputs(spec.cols, B, 0), spec.relu)
    m.close()


EDGE = [
    # name, rows, cols, density, r, k, scale
    ("all_pruned", 16, 50, 0.0, 5, 4, 1.0),
    ("single_nnz", 16, 50, 1.0 / 800, 5, 4, 1.0),
    ("k2_long_pads", 33, 700, 0.01, 5, 2, 1.0),
    ("k1_pads", 9, 300, 0.05, 3, 1, 1.0),
    ("r1_single_symbol", 20, 64, 0.3, 1, 4, 1.0),
    ("k8_r5", 40, 363, 0.5, 5, 8, 1.0),
    ("ragged_tiny", 1, 5, 0.6, 2, 2, 1.0),
    ("wide_rows", 3, 25088, 0.04, 5, 4, 1.0),
    ("tall", 2000, 17, 0.3, 5, 4, 1.0),
    ("ragged_groups", 333, 1001, 0.07, 5, 4, 0.3),
]


@pytest.mark.parametrize("name,rows,cols,d,r,k,scale", EDGE)
@pytest.mark.parametrize("jl,jq", [(None, None), (8, 1), (11, 2), (14, 4)])
def test_edge_fixtures(torch_dev, monkeypatch, name, rows, cols, d, r, k, scale, jl, jq):
    """Narrow windows (jL = 8) send most tokens through the code-by-code slow
    path; Q = 2 / 4 split every row's lanes into column groups whose partial
    sums the last-arriving CTA adds (rows with few or no tokens per group)."""
    torch, dev = torch_dev
    W = synth.random_matrix(rows, cols, seed=zlib.crc32(name.encode()) % 1000, scale=scale)
    v = synth.random_matrix(1, rows, seed=7).ravel()
    c, buf = layer(name, W, d, r, k, v)
    m = load(buf, False, monkeypatch, jl, jq)
    for B in (1, 2, 4):
        a = synth.random_activations(cols, B, seed=B)
        if m.kernel_name(0, B) == "k_fc_j":
            check(torch, dev, m, c, v, a, False)
    m.close()


@pytest.mark.parametrize("jq", [1, 2, 4])
def test_column_groups_c5_fc6(torch_dev, monkeypatch, jq):
    """C5 fc6 at B = 1 with each column-group split: the same oracle bound,
    and repeated launches bit-identical (partial sums added in group order)."""
    torch, dev = torch_dev
    spec, c, buf, v = config_layer("C5", 0)
    m = load(buf, True, monkeypatch, None, jq)
    a = synth.fc_inputs(spec.cols, 1, 3)
    y0 = check(torch, dev, m, c, v, a, True)
    for _ in range(3):
        assert np.array_equal(forward(torch, dev, m, a, spec.rows), y0)
    m.close()


def test_small_batch_infer_stack_c3(torch_dev):
    """The C3 stack through cdn_model_infer at K = 3 (every layer on k_fc_j):
    per-layer isolation against the oracle chain is covered by the layer tests;
    here the chained scores stay within the north_star bound of the fp64 chain
    rounded to fp32 between layers."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    cfg = synth.CONFIGS["C3"]
    m = cdn.Model(0)
    cs = []
    for i, spec in enumerate(cfg.fc):
        _, c, buf, v = config_layer("C3", i)
        m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
        cs.append((c, v, spec.relu))
        assert m.kernel_name(i, 3) == "k_fc_j"
    K = 3
    a = synth.fc_inputs(cfg.fc[0].cols, K, 5)
    xi = torch.from_numpy(a).to(dev)
    so = torch.zeros((K, cfg.fc[-1].rows), dtype=torch.float32, device=dev)
    m.infer(xi, K, so, on_device=True)
    torch.cuda.synchronize()
    h = a.astype(np.float64)
    for c, v, relu in cs:
        h = infer.fc_forward(c.dense_q(), h.astype(np.float32), v, apply_relu=relu)
    y = so.cpu().numpy()
    assert np.abs(y - h).max() / np.abs(h).max() <= 1e-4
    m.close()


@pytest.mark.parametrize("cfg,i", [("C5", 0), ("C5", 2), ("C2", 0), ("C1", 0)])
def test_cold_back_to_back_replicas(torch_dev, cfg, i):
    """The b1_cold protocol as a correctness check: R resident replicas of a
    layer, L2 flushed, launches back to back on one stream (programmatic
    dependent launches; every CTA's stream pieces still in flight when its
    warps start) -- every replica's output equal to the first one's and within
    the oracle bound.  Catches staging races that a single warm launch hides."""
    torch, dev = torch_dev
    spec, c, buf, v = config_layer(cfg, i)
    R = 6
    ms = [load(buf, False) for _ in range(R)]
    a = synth.fc_inputs(spec.cols, 1, 9)
    x = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)
    ys = [torch.full((spec.rows, 1), float("nan"), dtype=torch.float32, device=dev) for _ in range(R)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)
    ref = infer.fc_forward(c.dense_q(), a, v, apply_relu=False)[0]
    for rep in range(3):
        flush.zero_()
        torch.cuda.synchronize()
        for m, y in zip(ms, ys):
            m.layer_forward(0, x, 1, 1, y, 1, stream=s.cuda_stream)
        torch.cuda.synchronize()
        out = [y.cpu().numpy()[:, 0] for y in ys]
        for o in out:
            assert np.array_equal(o, out[0])
            assert np.abs(o - ref).max() / np.abs(ref).max() <= 1e-4
    for m in ms:
        m.close()


# ---- the medium-batch kernel k_fc_jm (plan_fc_jm): one lane per (row, column
# group), launches of <= 32 images, partial sums added by k_j_reduce


def load_medium(buf, relu, monkeypatch=None, jmq=None):
    import paper_1711_00244_b200 as cdn
    if monkeypatch is not None and jmq is not None:
        monkeypatch.setenv("CDN_JMQ", str(jmq))
    m = cdn.Model(0)
    m.load_layer(buf, cdn.LayerDesc.fc(relu))
    if monkeypatch is not None:
        monkeypatch.delenv("CDN_JMQ", raising=False)
    m.set_kernel_policy(1 << 20, 1 << 20)  # no large-batch kernels: B > 4 takes the medium split
    return m


@pytest.mark.parametrize("cfg,i", CONFIG_LAYERS)
def test_medium_config_layers(torch_dev, cfg, i):
    torch, dev = torch_dev
    spec, c, buf, v = config_layer(cfg, i)
    m = load_medium(buf, spec.relu)
    for B in (5, 8, 13, 32, 45, 128):
        a = synth.fc_inputs(spec.cols, B, B)
        y0 = check(torch, dev, m, c, v, a, spec.relu, "k_fc_jm")
        assert np.array_equal(forward(torch, dev, m, a, spec.rows), y0)  # fixed reduction order
    m.close()


@pytest.mark.parametrize("name,rows,cols,d,r,k,scale", EDGE)
@pytest.mark.parametrize("jmq", [None, 1, 3])
def test_medium_edge_fixtures(torch_dev, monkeypatch, name, rows, cols, d, r, k, scale, jmq):
    """Q = 1 (direct outputs), 3 (ragged groups, rows with empty groups) and
    the load-time choice; batches that leave image groups partly empty."""
    torch, dev = torch_dev
    W = synth.random_matrix(rows, cols, seed=zlib.crc32(name.encode()) % 1000, scale=scale)
    v = synth.random_matrix(1, rows, seed=7).ravel()
    c, buf = layer(name, W, d, r, k, v)
    m = load_medium(buf, False, monkeypatch, jmq)
    for B in (5, 16, 33):
        if m.kernel_name(0, B) != "k_fc_jm":  # x slice of a single group larger than shared memory
            assert cols > 4000
            continue
        a = synth.random_activations(cols, B, seed=B)
        check(torch, dev, m, c, v, a, False, "k_fc_jm")
    m.close()


def test_medium_strided_input(torch_dev):
    """ldx > B (a slice of a wider activation buffer) and an unaligned ldx:
    the staging loads fall back from 16-byte vectors to scalars."""
    torch, dev = torch_dev
    spec, c, buf, v = config_layer("C2", 0)
    m = load_medium(buf, spec.relu)
    for B, ldx in ((7, 9), (20, 24), (32, 35)):
        a = synth.fc_inputs(spec.cols, B, 11)
        xb = np.full((spec.cols, ldx), np.nan, dtype=np.float32)
        xb[:, :B] = a.T
        x = torch.from_numpy(xb).to(dev)
        y = torch.full((spec.rows, B), float("nan"), dtype=torch.float32, device=dev)
        m.layer_forward(0, x, ldx, B, y, B)
        torch.cuda.synchronize()
        yy = y.cpu().numpy().T
        ref = infer.fc_forward(c.dense_q(), a, v, apply_relu=spec.relu)
        assert np.abs(yy - ref).max() / np.abs(ref).max() <= 1e-4
    m.close()
