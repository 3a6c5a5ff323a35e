"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Decode: bit-exact (row, column, symbol, codebook value),
pads included.  Layer outputs: ||y_gpu - y_ref||_inf / ||y_ref||_inf <= 1e-4
against the fp64 oracle on the same fp32 input (north_star tolerance); the
elementwise error relative to sum_j |w_ij a_j| + |v_i| is also checked against
a bound derived from fp32 accumulation."""
import os
import zlib

import numpy as np
import pytest

import synth
from oracle import cdni, compress, decode, infer

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    return torch, torch.device("cuda:0")


_CACHE = {}


def oracle_layer(key, W, d, r, k, bias):
    if key not in _CACHE:
        c = compress.compress_layer(W, d, r, k, bias)
        _CACHE[key] = (c, cdni.serialize([c.layer]))
    return _CACHE[key]


def config_layer(cfg, i):
    spec = synth.CONFIGS[cfg].fc[i]
    W, v = synth.fc_weights(spec, synth.CONFIGS[cfg].seed)
    c, buf = oracle_layer((cfg, i), W, spec.density, spec.r, spec.k, v)
    return spec, c, buf


def make_model(torch, buf, relu=False, rank=0, world=1):
    import paper_1711_00244_b200 as cdn
    m = cdn.Model(0, rank=rank, world=world)
    m.load_layer(buf, cdn.LayerDesc.fc(relu))
    return m


def gpu_decode(torch, dev, m, layer=0):
    n = m.decode_count(layer)
    row = torch.empty(n, dtype=torch.int32, device=dev)
    col = torch.empty(n, dtype=torch.int32, device=dev)
    sym = torch.empty(n, dtype=torch.uint8, device=dev)
    val = torch.empty(n, dtype=torch.float32, device=dev)
    m.decode(layer, row, col, sym, val)
    torch.cuda.synchronize()
    return row.cpu().numpy(), col.cpu().numpy(), sym.cpu().numpy(), val.cpu().numpy()


def expected_tokens(c):
    """(row, col, sym, val) of every token from the oracle's own pre-encoding
    streams: columns by the C-01 prefix sum, values from the codebook."""
    rows = np.repeat(np.arange(c.row_tokens.size), c.row_tokens)
    g = c.gap_tokens + 1
    cs = np.cumsum(g)
    starts = np.zeros(c.row_tokens.size + 1, dtype=np.int64)
    np.cumsum(c.row_tokens, out=starts[1:])
    base = np.zeros_like(cs)
    nonempty = c.row_tokens > 0
    first = starts[:-1][nonempty]
    offs = np.where(first > 0, cs[first - 1], 0)
    base_idx = np.repeat(offs, c.row_tokens[nonempty])
    col = cs - base_idx - 1
    sym = c.val_tokens
    val = c.layer.codebook[sym]
    return rows, col, sym, val


def check_decode(torch, dev, c, buf):
    m = make_model(torch, buf)
    R, Cc, S, V = gpu_decode(torch, dev, m)
    er, ec, es, ev = expected_tokens(c)
    assert np.array_equal(R, er)
    assert np.array_equal(Cc, ec)
    assert np.array_equal(S, es.astype(np.uint8))
    assert np.array_equal(V.view(np.uint32), ev.astype(np.float32).view(np.uint32))
    # real tokens are exactly the kept entries with their centres
    real = S != 0
    assert np.array_equal(c.mask[R[real], Cc[real]], np.ones(real.sum(), bool))
    assert real.sum() == c.mask.sum()
    return m, (R, Cc, S, V)


def rel_err(y, ref):
    return np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-30)


def gpu_forward(torch, dev, m, a, N, layer=0):
    """a: image-major [B][K] fp32 -> y image-major [B][N] via feature-major device buffers."""
    B = a.shape[0]
    x = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)
    y = torch.full((N, B), float("nan"), dtype=torch.float32, device=dev)
    m.layer_forward(layer, x, B, B, y, B)
    torch.cuda.synchronize()
    return y.cpu().numpy().T


def check_forward(torch, dev, m, c, bias, a, relu):
    y = gpu_forward(torch, dev, m, a, c.layer.rows)
    ref = infer.fc_forward(c.dense_q(), a, bias, apply_relu=relu)
    assert np.isfinite(y).all()
    e = rel_err(y, ref)
    assert e <= TOL, e
    scale = infer.fc_abs_scale(c.dense_q(), a, bias)
    kmax = max(1, int(c.row_tokens.max()))
    elem = (np.abs(y - ref) / np.maximum(scale, 1e-30)).max()
    # fp32 summation bound gamma_n; at B >= 16 the default policy may pick the
    # fp16-split tensor-core kernel (each product within ~2^-21 relative,
    # DESIGN.md §9)
    split = 2.0 ** -20 if a.shape[0] >= 16 else 0.0
    assert elem <= 2 * kmax * 2.0 ** -24 + split + 1e-12, elem
    return e


# --------------------------------------------------------------------- decode

def test_decode_c1_bit_exact_vs_plain_decode(torch_dev):
    torch, dev = torch_dev
    spec, c, buf = config_layer("C1", 0)
    m, (R, Cc, S, V) = check_decode(torch, dev, c, buf)
    # and against the plain bit-by-bit Alg. 1 decode of the container
    L = cdni.deserialize(buf)[0]
    r2, c2, s2, v2 = decode.decode_layer(L)
    assert np.array_equal(R, r2) and np.array_equal(Cc, c2) and np.array_equal(S, s2)


@pytest.mark.parametrize("cfg,i", [("C2", 0), ("C3", 1), ("C3", 2), ("C5", 0), ("C5", 1), ("C5", 2)])
def test_decode_config_layers_bit_exact(torch_dev, cfg, i):
    torch, dev = torch_dev
    spec, c, buf = config_layer(cfg, i)
    m, (R, Cc, S, V) = check_decode(torch, dev, c, buf)
    # sampled rows against the plain decode (long codes of up to 20 bits included)
    L = cdni.deserialize(buf)[0]
    rows = [0, 1, L.rows // 2, L.rows - 1]
    r2, c2, s2, _ = decode.decode_layer(L, rows)
    sel = np.isin(R, rows)
    assert np.array_equal(R[sel], r2) and np.array_equal(Cc[sel], c2) and np.array_equal(S[sel], s2)


@pytest.mark.parametrize("G", ["1", "2", "8", "32"])
def test_decode_every_lane_split(torch_dev, G, monkeypatch):
    torch, dev = torch_dev
    monkeypatch.setenv("CDN_LANES_PER_ROW", G)
    spec, c, buf = config_layer("C2", 0)
    m, _ = check_decode(torch, dev, c, buf)
    st = m.stats(0)
    assert st["lanes_per_row"] == int(G)


EDGE = [
    # name, rows, cols, density, r, k, scale
    ("all_pruned", 16, 50, 0.0, 5, 4, 1.0),
    ("single_nnz", 16, 50, 1.0 / 800, 5, 4, 1.0),
    ("k2_long_pads", 33, 700, 0.01, 5, 2, 1.0),
    ("k1_pads", 9, 300, 0.05, 3, 1, 1.0),
    ("r1_single_symbol", 20, 64, 0.3, 1, 4, 1.0),
    ("dense_k8_r8", 40, 363, 0.84, 8, 8, 1.0),
    ("ragged_tiny", 1, 5, 0.6, 2, 2, 1.0),
    ("wide_rows", 3, 25088, 0.04, 5, 4, 1.0),
    ("tall", 2000, 17, 0.3, 5, 4, 1.0),
]


@pytest.mark.parametrize("name,rows,cols,d,r,k,scale", EDGE)
def test_edge_fixtures_decode_and_forward(torch_dev, name, rows, cols, d, r, k, scale):
    torch, dev = torch_dev
    W = synth.random_matrix(rows, cols, seed=zlib.crc32(name.encode()) % 1000, scale=scale)
    v = synth.random_matrix(1, rows, seed=7).ravel()
    c, buf = oracle_layer(name, W, d, r, k, v)
    m, _ = check_decode(torch, dev, c, buf)
    for B in (1, 3, 8, 13):
        a = synth.random_activations(cols, B, seed=B)
        check_forward(torch, dev, m, c, v, a, relu=False)


def test_long_codes_take_the_slow_path(torch_dev):
    """Skewed symbol counts give val codes longer than the 10-bit primary LUT."""
    torch, dev = torch_dev
    spec, c, buf = config_layer("C5", 0)
    assert max(c.layer.val_lengths.values()) > 10
    # tokens with long codes exist and decoded exactly (covered by the full check)
    long_syms = [s for s, L in c.layer.val_lengths.items() if L > 10]
    assert np.isin(c.val_tokens, long_syms).any()


# --------------------------------------------------------------------- forward

@pytest.mark.parametrize("B", [1, 2, 3, 8, 31, 32, 33, 128])
def test_forward_c2(torch_dev, B):
    torch, dev = torch_dev
    spec, c, buf = config_layer("C2", 0)
    m = make_model(torch, buf, relu=False)
    W, v = synth.fc_weights(spec, 0)
    a = synth.fc_inputs(spec.cols, B, 0)
    check_forward(torch, dev, m, c, v, a, relu=False)


def test_forward_c1_b1(torch_dev):
    torch, dev = torch_dev
    spec, c, buf = config_layer("C1", 0)
    m = make_model(torch, buf)
    _, v = synth.fc_weights(spec, 0)
    check_forward(torch, dev, m, c, v, synth.fc_inputs(spec.cols, 1, 0), relu=False)


@pytest.mark.parametrize("i", [0, 1, 2])
@pytest.mark.parametrize("B", [1, 8, 64])
def test_forward_c5_layers(torch_dev, i, B):
    torch, dev = torch_dev
    spec, c, buf = config_layer("C5", i)
    m = make_model(torch, buf, relu=spec.relu)
    _, v = synth.fc_weights(spec, 0)
    a = synth.fc_inputs(spec.cols, B, 0)
    check_forward(torch, dev, m, c, v, a, relu=spec.relu)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_shards_concatenate_to_full(torch_dev, world):
    """Row-block sharding: each rank's slice of the same streams
    gives exactly the rows of the 1-GPU result."""
    torch, dev = torch_dev
    spec, c, buf = config_layer("C3", 2)   # fc8 1000 rows: ragged last shard at 3 and 8
    _, v = synth.fc_weights(spec, 0)
    a = synth.fc_inputs(spec.cols, 4, 0)     # B = 4: small-batch kernel, shard-invariant order
    full = gpu_forward(torch, dev, make_model(torch, buf), a, spec.rows)
    parts = []
    for r in range(world):
        m = make_model(torch, buf, rank=r, world=world)
        st = m.stats(0)
        y = gpu_forward(torch, dev, m, a, st["row_end"] - st["row_begin"])
        parts.append(y)
        R, Cc, S, V = gpu_decode(torch, dev, m)
        assert (R >= st["row_begin"]).all() and (R < st["row_end"]).all()
    got = np.concatenate(parts, axis=1)
    assert np.array_equal(got, full)


VARIANTS = [("kmeans", 4, 0.04), ("linear", 5, 0.04), ("kmeans", 5, 0.09), ("linear", 8, 0.2)]


@pytest.mark.parametrize("quantizer,k,d", VARIANTS)
@pytest.mark.parametrize("B,policy", [(1, (1000, 1 << 30)), (8, (1000, 1 << 30)), (64, (1, 1 << 30)),
                                       (256, (1, 1))])
def test_paper_variants_all_kernels(torch_dev, quantizer, k, d, B, policy):
    """SURVEY §8(f) row 4 variants through every FC kernel: the Lloyd k-means
    codebook (C-33) and 5-/8-bit relative indices (VGG's 5-bit gaps, P:L453;
    k > 4 leaves the multi-symbol LUT kernels for the pad-folding ones)."""
    torch, dev = torch_dev
    key = f"variant-{quantizer}-{k}-{d}"
    W = synth.random_matrix(700, 3000, seed=zlib.crc32(key.encode()) % 1000, scale=0.02)
    v = synth.random_matrix(1, 700, seed=5).ravel()
    if key not in _CACHE:
        c = compress.compress_layer(W, d, 5, k, v, quantizer=quantizer)
        _CACHE[key] = (c, cdni.serialize([c.layer]))
    c, buf = _CACHE[key]
    m = make_model(torch, buf, relu=True)
    m.set_kernel_policy(*policy)
    a = synth.fc_inputs(3000, B, 3)
    check_forward_sparse(torch, dev, m, c, v, a, relu=True, split_tc=policy[1] == 1)
    m.close()


# ------------------------------- block-contiguous container (Alg. 2)

BLOCKED = [(512, 1024, 128, 128), (384, 768, 64, 256), (256, 640, 256, 64), (1024, 2048, 1024, 1024),
           (300, 512, 100, 128)]


def blocked_case(rows, cols, bh, bw, d=0.06):
    key = ("blocked", rows, cols, bh, bw, d)
    if key not in _CACHE:
        W = synth.random_matrix(rows, cols, seed=(rows * 7 + bh) % 1000, scale=0.02)
        v = synth.random_matrix(1, rows, seed=11).ravel()
        c = compress.compress_layer(W, d, 5, 4, v, bh=bh, bw=bw)
        _CACHE[key] = (c, cdni.serialize([c.layer]), v)
    return _CACHE[key]


@pytest.mark.parametrize("rows,cols,bh,bw", BLOCKED)
@pytest.mark.parametrize("B", [1, 37, 300])
def test_blocked_container_forward(torch_dev, rows, cols, bh, bw, B):
    """Alg. 2's block-contiguous storage consumed natively: the list decoder
    walks the stored rows of M' (blocks) and routes every entry to its weight
    row / K tile; the tensor-core contraction is the same."""
    torch, dev = torch_dev
    c, buf, v = blocked_case(rows, cols, bh, bw)
    m = make_model(torch, buf, relu=True)
    assert m.kernel_name(0, B) == "k_fc_tc"
    a = synth.fc_inputs(cols, B, 5)
    check_forward_sparse(torch, dev, m, c, v, a, relu=True, split_tc=True)
    if rows * cols <= 512 * 1024 and B == 37:   # and the paper's Alg. 2 itself, step by step
        y = gpu_forward(torch, dev, m, a, rows)
        ref = infer.fc_forward_blocked(c.layer, a, v, apply_relu=True)
        assert rel_err(y, ref) <= TOL
    m.close()


def test_blocked_decode_hook_stored_coordinates(torch_dev):
    """cdn_layer_decode on a blocked layer returns the stored matrix's tokens
    (block index, position in the flattened block), bit-exact."""
    torch, dev = torch_dev
    c, buf, v = blocked_case(*BLOCKED[0])
    m = make_model(torch, buf)
    R, Cc, S, V = gpu_decode(torch, dev, m)
    er, ec, es, ev = decode.decode_layer(c.layer)
    assert np.array_equal(R, er) and np.array_equal(Cc, ec) and np.array_equal(S, es.astype(np.uint8))
    assert np.array_equal(V.view(np.uint32), ev.astype(np.float32).view(np.uint32))
    m.close()


def test_blocked_layer_in_infer_stack(torch_dev):
    """A blocked layer between plain ones inside infer (C3-sized)."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    W1 = synth.random_matrix(512, 1024, seed=21, scale=0.02)
    v1 = synth.random_matrix(1, 512, seed=22).ravel()
    c1 = compress.compress_layer(W1, 0.09, 5, 4, v1)
    v2 = synth.random_matrix(1, 384, seed=26).ravel()
    W3 = synth.random_matrix(100, 384, seed=23, scale=0.02)
    v3 = synth.random_matrix(1, 100, seed=24).ravel()
    c3 = compress.compress_layer(W3, 0.25, 5, 4, v3)
    c2b = compress.compress_layer(synth.random_matrix(384, 512, seed=25, scale=0.02), 0.06, 5, 4, v2,
                                  bh=128, bw=128)
    m = cdn.Model(0)
    m.load_layer(cdni.serialize([c1.layer]), cdn.LayerDesc.fc(True))
    m.load_layer(cdni.serialize([c2b.layer]), cdn.LayerDesc.fc(True))
    m.load_layer(cdni.serialize([c3.layer]), cdn.LayerDesc.fc(False))
    K = 64
    a = synth.fc_inputs(1024, K, 9)
    scores = np.zeros((K, 100), np.float32)
    m.set_plan([K, K, K])
    m.infer(a, K, scores, on_device=False)
    x = a
    for c, v, relu in ((c1, v1, True), (c2b, v2, True), (c3, v3, False)):
        x = infer.fc_forward(sparse_q(c), x, v, apply_relu=relu).astype(np.float32)
    assert rel_err(scores, x) <= TOL
    m.close()


def test_tc_infer_stack_image_major_and_phases(torch_dev):
    """The tensor-core path inside infer: lists decoded ahead on the side stream
    and reused by later phases of the call, the first layer splitting the
    image-major input directly (no transpose), host and device buffers."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    cfg = synth.CONFIGS["C3"]
    m = cdn.Model(0)
    comps = []
    for i, spec in enumerate(cfg.fc):
        _, c, buf = config_layer("C3", i)
        m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
        comps.append((c, synth.fc_weights(spec, 0)[1], spec.relu))
    m.set_kernel_policy(1, 1)            # tensor-core kernel at every batch
    K = 300
    a = synth.fc_inputs(cfg.fc[0].cols, K, 0)
    x = a
    for c, v, relu in comps:
        x = infer.fc_forward(sparse_q(c), x, v, apply_relu=relu).astype(np.float32)
    for plan in ([100, 300, 300], [150, 150, 300], [K, K, K]):
        m.set_plan(plan)
        scores = np.zeros((K, cfg.fc[-1].rows), np.float32)
        m.infer(a, K, scores, on_device=False)
        assert rel_err(scores, x) <= TOL, plan
    xi = torch.from_numpy(a).to(dev)
    so = torch.zeros((K, cfg.fc[-1].rows), dtype=torch.float32, device=dev)
    m.infer(xi, K, so, on_device=True)
    torch.cuda.synchronize()
    assert rel_err(so.cpu().numpy(), x) <= TOL
    m.close()


def test_host_input_prefetch_many_rounds(torch_dev):
    """Host-buffer infer: each round's input goes up in pieces on the copy
    streams into alternating staging buffers while earlier phases compute.
    Many rounds (and a ragged remainder) must give the same bits as the
    device-resident call, and a second call with other inputs must not see
    the first call's staged data."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    cfg = synth.CONFIGS["C3"]
    m = cdn.Model(0)
    for i, spec in enumerate(cfg.fc):
        _, _, buf = config_layer("C3", i)
        m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
    n_out = cfg.fc[-1].rows
    for K, plan in ((200, [8, 16, 32]), (300, [50, 100, 100]), (77, [1, 4, 12])):
        m.set_plan(plan)
        for seed in (1, 2):
            a = synth.fc_inputs(cfg.fc[0].cols, K, seed)
            host = np.zeros((K, n_out), np.float32)
            m.infer(a, K, host, on_device=False)
            xi = torch.from_numpy(a).to(dev)
            so = torch.zeros((K, n_out), dtype=torch.float32, device=dev)
            m.infer(xi, K, so, on_device=True)
            torch.cuda.synchronize()
            assert np.array_equal(host, so.cpu().numpy()), (K, plan, seed)
    m.close()


def test_repeated_infer_graph_replay(torch_dev):
    """Identical infer calls on device buffers: the first runs eagerly, the
    second is captured into a CUDA graph, later ones replay it; every call's
    output is the same bits and counts the same kernel launches, and changing
    the input buffer or the plan leaves the graph."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    cfg = synth.CONFIGS["C3"]
    m = cdn.Model(0)
    for i, spec in enumerate(cfg.fc):
        _, c, buf = config_layer("C3", i)
        m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
    m.set_kernel_policy(1, 128)
    K = 256
    a = synth.fc_inputs(cfg.fc[0].cols, K, 0)
    xi = torch.from_numpy(a).to(dev)
    so = torch.zeros((K, cfg.fc[-1].rows), dtype=torch.float32, device=dev)
    outs, counts = [], []
    for it in range(5):
        if it == 3:
            xi.mul_(1.0)                     # same buffer, same values: the graph reads the live input
        n0 = cdn.kernel_launches()
        m.infer(xi, K, so, on_device=True)
        torch.cuda.synchronize()
        counts.append(cdn.kernel_launches() - n0)
        outs.append(so.cpu().numpy().copy())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    assert len(set(counts)) == 1 and counts[0] > 0
    # a new input buffer with other values: no stale graph
    a2 = synth.fc_inputs(cfg.fc[0].cols, K, 1)
    xi2 = torch.from_numpy(a2).to(dev)
    for _ in range(3):
        m.infer(xi2, K, so, on_device=True)
    torch.cuda.synchronize()
    x = a2
    for i, spec in enumerate(cfg.fc):
        _, c, _ = config_layer("C3", i)
        x = infer.fc_forward(sparse_q(c), x, synth.fc_weights(spec, 0)[1], apply_relu=spec.relu).astype(np.float32)
    assert rel_err(so.cpu().numpy(), x) <= TOL
    m.close()


def test_tc_fold_list_decoder_subprocess():
    """The pad-folding list decoder (layers outside the multi-symbol LUT
    limits; forced here with CDN_TC_LIST=fold) through the same parity check."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_parity as t, torch; "
            "t.test_tc_forward_configs((torch, torch.device('cuda:0')), 'C5', 2, 300); "
            "t.test_tc_forward_configs((torch, torch.device('cuda:0')), 'C3', 0, 200); print('ok')")
    env = dict(os.environ, CDN_TC_LIST="fold")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


# ----------------------------------------------------------------- end to end

def test_infer_c3_stack_matches_oracle_chain(torch_dev):
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    cfg = synth.CONFIGS["C3"]
    m = cdn.Model(0)
    comps = []
    for i, spec in enumerate(cfg.fc):
        _, c, buf = config_layer("C3", i)
        m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
        comps.append((c, synth.fc_weights(spec, 0)[1], spec.relu))
    K = 24
    a = synth.fc_inputs(cfg.fc[0].cols, K, 0)
    scores = np.zeros((K, cfg.fc[-1].rows), np.float32)
    m.set_plan([2, 6, 12])              # variable batch: 12/6 phases of 6, 6/2 phases of 2
    m.infer(a, K, scores, on_device=False)
    x = a
    for c, v, relu in comps:
        x = infer.fc_forward(c.dense_q(), x, v, apply_relu=relu).astype(np.float32)
    assert rel_err(scores, x) <= TOL
    # device-resident input/output, plan = whole batch
    m.set_plan([K, K, K])
    xi = torch.from_numpy(a).to(dev)
    so = torch.zeros((K, cfg.fc[-1].rows), dtype=torch.float32, device=dev)
    m.infer(xi, K, so, on_device=True)
    torch.cuda.synchronize()
    assert rel_err(so.cpu().numpy(), x) <= TOL


# ------------------------------------------------- large-batch band kernel (K3b)

def sparse_q(c):
    """prune∘quantize(W) as a scipy CSR matrix (same values as dense_q)."""
    import scipy.sparse as sp
    r, col = np.nonzero(c.mask)
    vals = c.layer.codebook[c.q[r, col]].astype(np.float32)
    return sp.csr_matrix((vals, (r, col)), shape=c.mask.shape)


def check_forward_sparse(torch, dev, m, c, bias, a, relu, split_tc=False):
    y = gpu_forward(torch, dev, m, a, c.layer.rows)
    Wq = sparse_q(c)
    ref = infer.fc_forward(Wq, a, bias, apply_relu=relu)
    assert np.isfinite(y).all()
    e = rel_err(y, ref)
    assert e <= TOL, e
    scale = infer.fc_abs_scale(Wq, a, bias)
    kmax = max(1, int(c.row_tokens.max()))
    elem = (np.abs(y - ref) / np.maximum(scale, 1e-30)).max()
    # fp32 accumulation bound; the tensor-core kernel adds the fp16-split
    # error (each product within ~2^-21 relative)
    bound = 2 * kmax * 2.0 ** -24 + (2.0 ** -20 if split_tc else 0.0) + 1e-12
    assert elem <= bound, elem
    return e


BAND_CASES = [("C1", 0, B) for B in (16, 32, 48, 100, 200)] + \
             [("C2", 0, B) for B in (16, 40, 64, 96, 128, 256)] + \
             [("C5", 0, 128), ("C5", 0, 512), ("C5", 1, 64), ("C5", 1, 512), ("C5", 2, 64), ("C5", 2, 512),
              ("C3", 2, 160)]


@pytest.mark.parametrize("cfg,i,B", BAND_CASES)
def test_band_forward_configs(torch_dev, cfg, i, B):
    """Warp-specialised band kernel (every VEC width, K-split reduction S > 1,
    ragged row blocks: fc8 has 1000 rows, ragged batch tiles) vs the oracle."""
    torch, dev = torch_dev
    spec, c, buf = config_layer(cfg, i)
    m = make_model(torch, buf, relu=spec.relu)
    m.set_kernel_policy(1, 1 << 30)   # band kernel (tensor-core path off)
    _, v = synth.fc_weights(spec, synth.CONFIGS[cfg].seed)
    a = synth.fc_inputs(spec.cols, B, synth.CONFIGS[cfg].seed)
    check_forward_sparse(torch, dev, m, c, v, a, relu=spec.relu)


@pytest.mark.parametrize("name,rows,cols,d,r,k,scale", EDGE)
@pytest.mark.parametrize("B", [1, 5, 36])
def test_band_edge_fixtures(torch_dev, name, rows, cols, d, r, k, scale, B):
    """Edge fixtures (all pruned, single nonzero, long pad runs, k=1, one
    symbol, dense r=8/k=8, 1x5, very wide, very tall) through the band kernel,
    including batches smaller than one tile."""
    torch, dev = torch_dev
    W = synth.random_matrix(rows, cols, seed=zlib.crc32(name.encode()) % 1000, scale=scale)
    v = synth.random_matrix(1, rows, seed=7).ravel()
    c, buf = oracle_layer(name, W, d, r, k, v)
    m = make_model(torch, buf)
    m.set_kernel_policy(1, 1 << 30)   # band kernel (tensor-core path off)
    a = synth.random_activations(cols, B, seed=B + 100)
    check_forward(torch, dev, m, c, v, a, relu=False)


def test_band_list_overflow_repeats_band(torch_dev):
    """A few rows carry all the large weights (dense rows in a 5%-dense layer):
    their per-band lists overflow the 32-entry stage capacity, so the decode
    warps repeat the band; the result must not change."""
    torch, dev = torch_dev
    rows, cols = 300, 4000
    W = synth.random_matrix(rows, cols, seed=5, scale=0.01)
    W[::37] *= 1000.0                  # 9 rows hold the largest magnitudes
    v = synth.random_matrix(1, rows, seed=6).ravel()
    c, buf = oracle_layer("skewed_rows", W, 0.05, 5, 4, v)
    assert c.mask[::37].mean() > 0.9    # those rows survive pruning almost whole
    m = make_model(torch, buf, relu=True)
    m.set_kernel_policy(1, 1 << 30)   # band kernel (tensor-core path off)
    for B in (8, 64, 128):
        a = synth.random_activations(cols, B, seed=B)
        check_forward(torch, dev, m, c, v, a, relu=True)


def test_band_and_small_kernels_agree(torch_dev):
    """The two FC kernels compute the same layer (different summation order)."""
    torch, dev = torch_dev
    spec, c, buf = config_layer("C2", 0)
    a = synth.fc_inputs(spec.cols, 24, 0)
    m1 = make_model(torch, buf)
    m1.set_kernel_policy(1000, 1 << 30)  # small-batch kernel
    m2 = make_model(torch, buf)
    m2.set_kernel_policy(1, 1 << 30)     # band kernel
    y1 = gpu_forward(torch, dev, m1, a, spec.rows)
    y2 = gpu_forward(torch, dev, m2, a, spec.rows)
    assert rel_err(y2, y1) <= 2e-6


def test_band_repeated_launches_are_deterministic(torch_dev):
    """Split partials are reduced in a fixed order and the arrival counters
    reset themselves: repeated launches are bit-identical."""
    torch, dev = torch_dev
    spec, c, buf = config_layer("C5", 2)
    m = make_model(torch, buf, relu=False)
    a = synth.fc_inputs(spec.cols, 512, 0)
    ys = [gpu_forward(torch, dev, m, a, spec.rows) for _ in range(3)]
    assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[1], ys[2])


# ----------------------------------------------------------------- planner (C3)

def test_c3_planner_under_64mib_budget(torch_dev):
    """Config C3: AlexNet FC stack, TOT = 64 MiB, batch chosen by the planner
    from 1..K.  On the device-profiled Time table and the
    library's memory model (IN / OUT / WS with every workspace, reading C-24),
    the library's plan is a divisor chain, feasible under the EXACT memory
    model, never better than the exact oracle DP (C-25); infer with it
    (remainder re-plan) matches the oracle chain, the library's
    inference scratch never exceeds TOT (reading C-36), and the DP's predicted
    time matches the measured one."""
    torch, dev = torch_dev
    import time
    import paper_1711_00244_b200 as cdn
    from oracle import planner as oplanner
    cfg = synth.CONFIGS["C3"]
    m = cdn.Model(0)
    comps = []
    for i, spec in enumerate(cfg.fc):
        _, c, buf = config_layer("C3", i)
        m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
        comps.append((c, synth.fc_weights(spec, 0)[1], spec.relu))
    K = 100
    m.set_memory_budget(cfg.tot_bytes)
    T = m.profile(K, 5)
    batches, predicted = m.plan(K)
    inb, outb, ws = m.memory_model(K)
    p = oplanner.Problem([{B: float(T[i][B - 1]) for B in range(1, K + 1)} for i in range(3)], list(inb), list(outb),
                         list(ws), cfg.tot_bytes)
    assert all(batches[i + 1] % batches[i] == 0 for i in range(2))
    cost = oplanner.chain_cost(p, batches)
    assert np.isfinite(cost)
    exact = oplanner.dp_plan(p, K)
    assert cost / batches[-1] >= exact.per_image * (1 - 1e-9)
    assert predicted > 0
    # the whole request through the planned executor, host buffers: scratch <= TOT
    a = synth.fc_inputs(cfg.fc[0].cols, K, 0)
    scores = np.zeros((K, cfg.fc[-1].rows), np.float32)
    m.release_scratch()
    m.scratch_bytes(reset_peak=True)
    m.infer(a, K, scores, on_device=False)
    cur, peak = m.scratch_bytes()
    print(f"C3 plan {batches}: scratch peak {peak / 2**20:.2f} MiB of {cfg.tot_bytes / 2**20:.0f} MiB")
    assert peak <= cfg.tot_bytes
    x = a
    for c, v, relu in comps:
        x = infer.fc_forward(sparse_q(c), x, v, apply_relu=relu).astype(np.float32)
    assert rel_err(scores, x) <= TOL
    # device buffers: the same bound, and the DP's predicted time against the
    # measured one (graph replay of the planned call, median of 20)
    _, predicted_dev = m.plan(K)
    xi = torch.from_numpy(a).to(dev)
    so = torch.zeros((K, cfg.fc[-1].rows), dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(dev)
    m.scratch_bytes(reset_peak=True)
    for _ in range(3):
        m.infer(xi, K, so, on_device=True, stream=s.cuda_stream)
    torch.cuda.synchronize()
    ms = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        m.infer(xi, K, so, on_device=True, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    meas = float(np.median(ms))
    _, peak = m.scratch_bytes()
    assert peak <= cfg.tot_bytes
    print(f"C3 predicted {predicted_dev:.4f} ms, measured {meas:.4f} ms")
    assert abs(predicted_dev - meas) <= 0.10 * meas
    assert rel_err(so.cpu().numpy(), x) <= TOL
    m.close()


# ------------------------------------------- tensor-core FC kernel (NEXT #2)

TC_CASES = [("C5", 0, 512), ("C5", 0, 300), ("C5", 1, 256), ("C5", 2, 512), ("C5", 2, 130), ("C2", 0, 128),
            ("C3", 2, 384), ("C1", 0, 256), ("C1", 0, 17)]


@pytest.mark.parametrize("cfg,i,B", TC_CASES)
def test_tc_forward_configs(torch_dev, cfg, i, B):
    """W tiles decoded into shared memory + 3-pass bf16-split tcgen05
    contraction (K-split partials, ragged row / batch / K tiles) vs the oracle."""
    torch, dev = torch_dev
    spec, c, buf = config_layer(cfg, i)
    m = make_model(torch, buf, relu=spec.relu)
    m.set_kernel_policy(1, 1)
    _, v = synth.fc_weights(spec, synth.CONFIGS[cfg].seed)
    a = synth.fc_inputs(spec.cols, B, synth.CONFIGS[cfg].seed)
    check_forward_sparse(torch, dev, m, c, v, a, relu=spec.relu, split_tc=True)


@pytest.mark.parametrize("name,rows,cols,d,r,k,scale", EDGE)
def test_tc_edge_fixtures(torch_dev, name, rows, cols, d, r, k, scale):
    torch, dev = torch_dev
    W = synth.random_matrix(rows, cols, seed=zlib.crc32(name.encode()) % 1000, scale=scale)
    v = synth.random_matrix(1, rows, seed=7).ravel()
    c, buf = oracle_layer(name, W, d, r, k, v)
    m = make_model(torch, buf)
    m.set_kernel_policy(1, 1)
    a = synth.random_activations(cols, 36, seed=99)
    check_forward_sparse(torch, dev, m, c, v, a, relu=False, split_tc=True)


# ------------------------------------- column-sharded layers

@pytest.mark.parametrize("cfg,i", [("C5", 0), ("C5", 1), ("C5", 2), ("C3", 2)])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_column_sharded_layer_partials(torch_dev, cfg, i, world):
    """Megatron-style column blocks through shard-only handles (rank r of
    `world`, CDN_SHARD_COLS, no communicator): each rank's cdn_layer_forward on
    its column block of x gives the partial sums of every row (no bias / ReLU);
    their sum + bias (+ ReLU) matches the oracle within the north_star bound and
    the fp16-split elementwise bound."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    spec, c, buf = config_layer(cfg, i)
    _, v = synth.fc_weights(spec, synth.CONFIGS[cfg].seed)
    B = 96
    a = synth.fc_inputs(spec.cols, B, 2)
    total = np.zeros((spec.rows, B), np.float64)
    cover = 0
    for r in range(world):
        m = cdn.Model(0, rank=r, world=world)
        m.set_sharding(cdn.CDN_SHARD_COLS)
        m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
        st = m.stats(0)
        k0, k1 = st["col_begin"], st["col_end"]
        assert (k0, k1) == cdn.col_block(spec.cols, r, world) and st["row_begin"] == 0 and st["row_end"] == spec.rows
        assert m.kernel_name(0, B) == "k_fc_tc"
        cover += k1 - k0
        x = torch.from_numpy(np.ascontiguousarray(a[:, k0:k1].T)).to(dev)
        if k1 == k0:
            x = torch.zeros((1, B), dtype=torch.float32, device=dev)
        y = torch.full((spec.rows, B), float("nan"), dtype=torch.float32, device=dev)
        m.layer_forward(0, x, B, B, y, B)
        torch.cuda.synchronize()
        total += y.cpu().numpy().astype(np.float64)
        m.close()
    assert cover == spec.cols
    out = (total + v[:, None]).T
    if spec.relu:
        out = np.maximum(out, 0.0)
    ref = infer.fc_forward(sparse_q(c), a, v, apply_relu=spec.relu)
    assert rel_err(out, ref) <= TOL
    scale = infer.fc_abs_scale(sparse_q(c), a, v)
    kmax = int(c.row_tokens.max())
    assert (np.abs(out - ref) / np.maximum(scale, 1e-30)).max() <= 2 * kmax * 2.0 ** -24 + world * 2.0 ** -20


@pytest.mark.gpu
def test_fused_split_scales_bit_identical(torch_dev, monkeypatch):
    """A tensor-core layer's reduce / epilogue leaves the max |y| of every
    (32-row group, image) for the next tensor-core layer's fp16 split, which
    then skips its own pass over x.  The scale is the same
    power of two either way, so the scores must be bit-identical to the
    separate max pass -- for device and host input, the first call (whose
    autotune runs must not clobber the producer's maxima) and graph replays,
    whole-batch and variable-batch plans."""
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    cfg = synth.CONFIGS["C3"]
    outs = {}
    for fuse in ("1", "0"):
        monkeypatch.setenv("CDN_TC_FUSE_SCALES", fuse)
        m = cdn.Model(0)
        monkeypatch.delenv("CDN_TC_FUSE_SCALES")
        for i, spec in enumerate(cfg.fc):
            _, _, buf = config_layer("C3", i)
            m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
        for K, plan in ((256, [256, 256, 256]), (300, [50, 100, 100])):
            m.set_plan(plan)
            a = synth.fc_inputs(cfg.fc[0].cols, K, 1)
            host = np.zeros((K, 1000), np.float32)
            m.infer(a, K, host, on_device=False)
            xi = torch.from_numpy(a).to(dev)
            for rep in range(3):  # eager, captured, replayed
                so = torch.zeros((K, 1000), dtype=torch.float32, device=dev)
                m.infer(xi, K, so, on_device=True)
                torch.cuda.synchronize()
                assert np.array_equal(so.cpu().numpy(), host), (fuse, K, rep)
            outs[(fuse, K)] = host
        m.close()
    for K in (256, 300):
        assert np.array_equal(outs[("1", K)], outs[("0", K)]), K
