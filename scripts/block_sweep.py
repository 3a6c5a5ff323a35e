"""GPU analogue of the paper's block-size sweep (Fig. 3): C2
AlexNet fc6 (9216 -> 4096, 9%) stored row-major and block-contiguous (Alg. 2,
bh x bw from 128x128 to 1024x1024), batch 16 and 256 (the paper's).  Per
configuration: the decode kernel (k_tc_list: Huffman + gap prefix sum into the
list), the contraction (k_split_x + k_fc_tc + k_tc_reduce) and the whole layer
call, CUDA-event timed, median of reps after an L2 flush.  JSON lines.
Usage: python scripts/block_sweep.py [--reps 10]"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--batches", default="16,256")
    args = ap.parse_args()
    import torch
    import paper_1711_00244_b200 as cdn
    from paper_1711_00244_b200 import build
    build.build()
    dev = torch.device("cuda:0")
    spec = synth.CONFIGS["C2"].fc[0]
    W, v = synth.fc_weights(spec, synth.CONFIGS["C2"].seed)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.Stream(dev)
    for bh, bw in [(1, 0), (128, 128), (256, 256), (512, 512), (1024, 1024), (128, 1024), (1024, 128)]:
        buf = cdn.compress_dense(W, spec.density, spec.r, spec.k, v, bh=bh, bw=bw)
        m = cdn.Model(0)
        m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
        m.set_kernel_policy(1, 1)   # the tensor-core path for every layout (blocked layers only run there)
        for B in [int(b) for b in args.batches.split(",")]:
            x = torch.rand((spec.cols, B), device=dev)
            y = torch.zeros((spec.rows, B), device=dev)
            with torch.cuda.stream(st):
                for _ in range(3):
                    m.layer_forward(0, x, B, B, y, B, stream=st.cuda_stream)
            torch.cuda.synchronize()
            tot, dec, mul = [], [], []
            for _ in range(args.reps):
                flush.zero_()
                torch.cuda.synchronize()
                cdn.kernel_timer(True)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(st):
                    e0.record(st)
                    m.layer_forward(0, x, B, B, y, B, stream=st.cuda_stream)
                    e1.record(st)
                torch.cuda.synchronize()
                tot.append(e0.elapsed_time(e1) * 1e3)
                dec.append(cdn.kernel_time("k_tc_list")[0] * 1e3)
                mul.append((cdn.kernel_time("k_fc_tc")[0] + cdn.kernel_time("k_split_x")[0]) * 1e3)
                cdn.kernel_timer(False)
            print(json.dumps({"layer": "C2 fc6 9216x4096 9%", "block": "row-major" if bh == 1 else f"{bh}x{bw}",
                              "B": B, "compressed_bytes": len(buf), "decode_us": float(np.median(dec)),
                              "multiply_us": float(np.median(mul)), "layer_us": float(np.median(tot))}),
                  flush=True)
        m.close()


if __name__ == "__main__":
    main()
