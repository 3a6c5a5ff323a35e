"""Run one config layer at batch B through cdn_layer_forward over R resident
replicas, N rounds (for ncu captures of the small-batch kernel).
Usage: python scripts/j_one.py CFG LAYER [B] [R] [N]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def main():
    import torch
    import paper_1711_00244_b200 as cdn
    from paper_1711_00244_b200 import build
    build.build()
    cfg, li = sys.argv[1], int(sys.argv[2])
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    R = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    N = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    spec = synth.CONFIGS[cfg].fc[li]
    W, v = synth.fc_weights(spec, synth.CONFIGS[cfg].seed)
    buf = cdn.compress_dense(W, spec.density, spec.r, spec.k, v)
    ms = [cdn.Model(0) for _ in range(R)]
    for m in ms:
        m.load_layer(buf, cdn.LayerDesc.fc(False))
    dev = torch.device("cuda:0")
    s = torch.cuda.Stream(dev)
    torch.cuda.set_stream(s)
    a = synth.fc_inputs(spec.cols, B, 0)
    x = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)
    y = torch.zeros((spec.rows, B), dtype=torch.float32, device=dev)
    for _ in range(N):
        for m in ms:
            m.layer_forward(0, x, B, B, y, B, stream=s.cuda_stream)
    torch.cuda.synchronize()
    print("ok", ms[0].kernel_name(0, B))


if __name__ == "__main__":
    main()
