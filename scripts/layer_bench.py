"""Per-layer kernel timing with CUDA graphs (no host launch latency inside the
measurement).  Usage: python scripts/layer_bench.py [--cfg C5] [--batches 1,8,64,512]
[--replicas 8] [--reps 20].  Prints one JSON object per (layer, B).  Also the
target for ncu: `-k regex:k_fc_forward`."""
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
    ap.add_argument("--cfg", default="C5")
    ap.add_argument("--layers", default="")
    ap.add_argument("--batches", default="1,8,64,512")
    ap.add_argument("--replicas", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--single", action="store_true", help="one launch, no timing (ncu target)")
    ap.add_argument("--policy", default="auto", choices=["auto", "tc", "band"],
                    help="large-batch kernel: autotuned (default), tensor-core or band")
    args = ap.parse_args()
    import torch
    import paper_1711_00244_b200 as cdn
    from paper_1711_00244_b200 import build
    build.build()
    dev = torch.device("cuda:0")
    cfg = synth.CONFIGS[args.cfg]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    sel = [int(s) for s in args.layers.split(",")] if args.layers else range(len(cfg.fc))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for li in sel:
        spec = cfg.fc[li]
        W, v = synth.fc_weights(spec, cfg.seed)
        buf = cdn.compress_dense(W, spec.density, spec.r, spec.k, v)
        del W
        models = []
        for _ in range(args.replicas):
            m = cdn.Model(0)
            m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
            if args.policy == "tc":
                m.set_kernel_policy(1, 1)
            elif args.policy == "band":
                m.set_kernel_policy(1, 1 << 30)
            models.append(m)
        st = models[0].stats(0)
        for B in [int(b) for b in args.batches.split(",")]:
            x = torch.rand((spec.cols, B), device=dev)
            y = torch.zeros((spec.rows, B), device=dev)
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                for m in models:
                    m.layer_forward(0, x, B, B, y, B, stream=s.cuda_stream)
            torch.cuda.synchronize()
            times = []
            if args.single:
                models[0].layer_forward(0, x, B, B, y, B, stream=s.cuda_stream)
                torch.cuda.synchronize()
                continue
            for _ in range(args.reps):
                if not args.no_flush:
                    flush.zero_()
                torch.cuda.synchronize()
                with torch.cuda.stream(s):
                    # keep the GPU busy while the host enqueues, so host launch
                    # latency never sits between the events
                    torch.cuda._sleep(3_000_000)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    for m in models:
                        m.layer_forward(0, x, B, B, y, B, stream=s.cuda_stream)
                    e1.record(s)
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) / len(models))
            if not times:
                continue
            ms = float(np.median(times))
            algo = st["algo_bytes_fixed"] + 4 * spec.cols * B + 4 * spec.rows * B
            flops = 2.0 * st["nnz"] * B + spec.rows * B
            print(json.dumps({"cfg": args.cfg, "layer": spec.name, "B": B, "us": ms * 1e3,
                              "kernel": models[0].kernel_name(0, B),
                              "gbs": algo / ms / 1e6, "hbm_frac": algo / ms / 1e6 / peaks["hbm_gbs"],
                              "tflops": flops / ms / 1e9, "tokens": st["tokens"], "nnz": st["nnz"],
                              "G": st["lanes_per_row"], "index_bytes": st["index_bytes"],
                              "stream_bytes": st["stream_bytes"]}), flush=True)
        for m in models:
            m.close()


if __name__ == "__main__":
    main()
