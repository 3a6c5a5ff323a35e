"""Small invocations of every kernel family for compute-sanitizer memcheck:
decode, small-batch, band, tensor-core FC, CONV (decode-dense, im2col, tcgen05
GEMM, LRN, pool), on small seeded layers with ragged shapes."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    import torch
    import paper_1711_00244_b200 as cdn
    dev = torch.device("cuda:0")
    for (rows, cols, d, r, k) in [(300, 700, 0.1, 5, 4), (16, 50, 1.0 / 800, 5, 4), (33, 700, 0.01, 5, 2),
                                  (40, 363, 0.84, 8, 8), (1, 5, 0.6, 2, 2), (130, 4100, 0.23, 5, 4)]:
        W = synth.random_matrix(rows, cols, seed=rows + cols, scale=0.05)
        v = synth.random_matrix(1, rows, seed=3).ravel()
        buf = cdn.compress_dense(W, d, r, k, v)
        for pol in [(1000, 1 << 30), (1, 1 << 30), (1, 1)]:
            m = cdn.Model(0)
            m.load_layer(buf, cdn.LayerDesc.fc(True))
            m.set_kernel_policy(*pol)
            n = m.decode_count(0)
            if n:
                t = [torch.empty(n, dtype=dt, device=dev) for dt in (torch.int32, torch.int32, torch.uint8,
                                                                    torch.float32)]
                m.decode(0, *t)
            for B in (1, 3, 8, 36, 130, 257):
                ld = (B + 3) // 4 * 4
                x = torch.rand((cols, ld), device=dev)
                y = torch.zeros((rows, ld), device=dev)
                m.layer_forward(0, x, ld, B, y, ld)
            torch.cuda.synchronize()
            m.close()
    spec = synth.ALEXNET_CONV[1]
    W, v = synth.fc_weights(spec, 0)
    buf = cdn.compress_dense(W, spec.density, spec.r, spec.k, v)
    m = cdn.Model(0)
    m.load_layer(buf, cdn.LayerDesc.conv(spec.in_ch, 27, 27, spec.kh, spec.kw, spec.stride, spec.pad, spec.groups,
                                         relu=True, lrn=True, pool_k=3, pool_s=2))
    x = torch.rand((2, 27, 27, spec.in_ch), device=dev)
    oh, ow, oc = m.out_shape(0)
    y = torch.zeros((2, oh, ow, oc), device=dev)
    m.conv_forward(0, x, 2, y)
    torch.cuda.synchronize()
    m.close()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
