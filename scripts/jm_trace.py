"""k_fc_j medium-batch launch traced (CDN_J_TRACE) for one config layer and
batch: python scripts/jm_trace.py CFG LAYER B OUT.bin"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def main():
    cfg, li, B, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    if os.path.exists(out):
        os.remove(out)
    os.environ["CDN_J_TRACE"] = out  # every launch traced (read at the library's first launch)
    import torch
    import paper_1711_00244_b200 as cdn
    spec = synth.CONFIGS[cfg].fc[li]
    W, v = synth.fc_weights(spec, synth.CONFIGS[cfg].seed)
    buf = cdn.compress_dense(W, spec.density, spec.r, spec.k, v)
    m = cdn.Model(0)
    m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
    m.set_kernel_policy(1 << 20, 1 << 20)
    dev = torch.device("cuda:0")
    x = torch.from_numpy(np.ascontiguousarray(synth.fc_inputs(spec.cols, B, 0).T)).to(dev)
    y = torch.zeros((spec.rows, B), dtype=torch.float32, device=dev)
    for _ in range(3):
        m.layer_forward(0, x, B, B, y, B)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
