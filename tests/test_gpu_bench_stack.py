"""The benchmark's exact call checked against the oracle: config C5 (VGG-16 FC
stack) at B = 512 through cdn_model_infer with bench.py's plan and kernel
policy (tensor-core path on every layer), run eagerly, captured and replayed
as a CUDA graph; every run's scores within the north_star bound of the fp64
oracle chain, replays bit-identical to the eager run, and each layer isolated
(the same policy, the oracle chain's fp32 input of that layer) against the
oracle layer.  The conv+FC AlexNet stack under a variable-batch plan is
checked the same way in tests/test_gpu_conv.py."""
import numpy as np
import pytest

import synth
from oracle import cdni, compress, infer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    import __graft_entry__
    __graft_entry__.build()
    return torch, torch.device("cuda:0")


def test_bench_c5_b512_infer_matches_oracle(torch_dev):
    torch, dev = torch_dev
    import paper_1711_00244_b200 as cdn
    cfg = synth.CONFIGS["C5"]
    B = 512
    m = cdn.Model(0)
    layers = []
    for spec in cfg.fc:
        W, v = synth.fc_weights(spec, cfg.seed)
        c = compress.compress_layer(W, spec.density, spec.r, spec.k, v)
        del W
        m.load_layer(cdni.serialize([c.layer]), cdn.LayerDesc.fc(spec.relu))
        layers.append((spec, c, v))
    m.set_plan([B] * 3)
    m.set_kernel_policy(0, 16)  # bench.py's policy
    assert [m.kernel_name(i, B) for i in range(3)] == ["k_fc_tc"] * 3
    a = synth.fc_inputs(cfg.fc[0].cols, B, cfg.seed)
    # oracle chain: fp64 layers, fp32 between them (the GPU's layer inputs are fp32)
    hs = [a.astype(np.float32)]
    for spec, c, v in layers:
        hs.append(infer.fc_forward(c.dense_q(), hs[-1], v, apply_relu=spec.relu).astype(np.float32))
    ref = infer.fc_forward(layers[-1][1].dense_q(), hs[-2], layers[-1][2], apply_relu=False)

    s = torch.cuda.Stream(dev)
    xi = torch.from_numpy(a).to(dev)
    outs = []
    for _ in range(4):  # eager, captured, replayed, replayed
        so = torch.zeros((B, cfg.fc[-1].rows), dtype=torch.float32, device=dev)
        m.infer(xi, B, so, on_device=True, stream=s.cuda_stream)
        torch.cuda.synchronize()
        outs.append(so.cpu().numpy())
    # the graph path keys on the output buffer: rerun on one buffer for replays
    so = torch.zeros((B, cfg.fc[-1].rows), dtype=torch.float32, device=dev)
    for _ in range(4):
        m.infer(xi, B, so, on_device=True, stream=s.cuda_stream)
        torch.cuda.synchronize()
        outs.append(so.cpu().numpy())
    for y in outs:
        assert np.isfinite(y).all()
        assert np.abs(y - ref).max() / np.abs(ref).max() <= 1e-4
        assert np.array_equal(y, outs[0])
    # per-layer isolation with the same policy
    for i, (spec, c, v) in enumerate(layers):
        x = torch.from_numpy(np.ascontiguousarray(hs[i].T)).to(dev)
        y = torch.zeros((spec.rows, B), dtype=torch.float32, device=dev)
        m.layer_forward(i, x, B, B, y, B)
        torch.cuda.synchronize()
        yl = y.cpu().numpy().T
        r = infer.fc_forward(c.dense_q(), hs[i], v, apply_relu=spec.relu)
        assert np.abs(yl - r).max() / np.abs(r).max() <= 1e-4
        scale = infer.fc_abs_scale(c.dense_q(), hs[i], v)
        kmax = int(c.row_tokens.max())
        assert (np.abs(yl - r) / np.maximum(scale, 1e-30)).max() <= 2 * kmax * 2.0 ** -24 + 2.0 ** -20
    m.close()
