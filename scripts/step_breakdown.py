"""Per-kernel time inside one infer step (library kernel timer: CUDA events on
the launching stream around every launch of each kernel family), for config
C4 (AlexNet conv1-5 + fc, B = 64) or C5 (VGG-16 fc stack, B = 512).  Kernels
on the side stream overlap the main stream, so the shares can sum past 100%.
JSON: step time (timer off), per-kernel ms per step, launches per step.
Usage: python scripts/step_breakdown.py [--cfg C4] [--steps 10]"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

KERNELS = ("k_gemm_bf16", "k_conv_halo", "k_s2d_bf16", "k_to_bf16_pad", "k_decode_conv", "k_im2col", "k_lrn", "k_lrn_pool", "k_maxpool", "k_fc_jm", "k_fc_j", "k_j_reduce", "k_decode_dense", "k_transpose", "k_fc_tc",
           "k_tc_list", "k_split_x", "k_tc_reduce", "k_fc_band", "k_fc_ms", "k_fc_fold")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C4", choices=["C4", "C5"])
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import paper_1711_00244_b200 as cdn
    from paper_1711_00244_b200 import build
    build.build()
    dev = torch.device("cuda:0")
    cfg = synth.CONFIGS[args.cfg]
    m = cdn.Model(0)
    if args.cfg == "C4":
        hw = cfg.image_hw
        for i, spec in enumerate(cfg.conv):
            W, v = synth.fc_weights(spec, cfg.seed)
            m.load_layer(cdn.compress_dense(W, spec.density, spec.r, spec.k, v),
                         cdn.LayerDesc.conv(spec.in_ch, hw, hw, spec.kh, spec.kw, spec.stride, spec.pad, spec.groups,
                                            relu=True, lrn=spec.lrn, pool_k=3 if spec.pool else 0,
                                            pool_s=2 if spec.pool else 0))
            hw = m.out_shape(i)[0]
        B = cfg.batches[0]
        x = torch.from_numpy(synth.conv_inputs(B, cfg.image_hw, cfg.image_c, cfg.seed)).to(dev)
    else:
        B = 512
        x = torch.from_numpy(synth.fc_inputs(cfg.fc[0].cols, B, cfg.seed)).to(dev)
    for spec in cfg.fc:
        W, v = synth.fc_weights(spec, cfg.seed)
        m.load_layer(cdn.compress_dense(W, spec.density, spec.r, spec.k, v), cdn.LayerDesc.fc(spec.relu))
    nl = m.num_layers()
    m.set_plan([B] * nl)
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    sp = st.cuda_stream
    out = torch.zeros((B, cfg.fc[-1].rows), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def run(n):
        ts = []
        for _ in range(n):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            m.infer(x, B, out, on_device=True, stream=sp)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    run(3)
    step_ms = run(args.steps)
    cdn.kernel_timer(True)
    timed_ms = run(args.steps)
    rows = {}
    for k in KERNELS:
        tot, n = cdn.kernel_time(k)
        if n:
            rows[k] = {"ms_per_step": tot / args.steps, "launches_per_step": n / args.steps,
                       "share": tot / args.steps / step_ms}
    cdn.kernel_timer(False)
    print(json.dumps({"cfg": args.cfg, "B": B, "step_ms": step_ms, "images_per_s": B / step_ms * 1e3,
                      "step_ms_timer_on": timed_ms, "kernels": rows,
                      "layers": [m.kernel_name(i, B) for i in range(nl)]}, indent=1), flush=True)
    m.close()


if __name__ == "__main__":
    main()
