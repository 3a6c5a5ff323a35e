"""SURVEY §8(d) grid of reports on one GPU: every FC config at its batches,
through the public infer call (device-resident input, fixed plan = the batch
for every layer, L2 flushed before every timed call, graph replay as in
bench.py), plus the planner's choice for C3 under its 64 MiB budget.  Per line:
images/s, compressed GB/s, the HBM fraction of the algorithmic bytes
(compressed streams + tables + activations in/out), and the
kernel each layer ran.  JSON lines.
Usage: python scripts/grid_report.py [--reps 20]"""
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
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    import paper_1711_00244_b200 as cdn
    from paper_1711_00244_b200 import build
    build.build()
    dev = torch.device("cuda:0")
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    sp = st.cuda_stream
    for name in ("C1", "C2", "C3", "C5"):
        cfg = synth.CONFIGS[name]
        m = cdn.Model(0)
        for spec in cfg.fc:
            W, v = synth.fc_weights(spec, cfg.seed)
            m.load_layer(cdn.compress_dense(W, spec.density, spec.r, spec.k, v), cdn.LayerDesc.fc(spec.relu))
        stats = [m.stats(i) for i in range(len(cfg.fc))]
        comp = sum(s["stream_bytes"] for s in stats)
        batches = list(cfg.batches) if name != "C3" else [1, 8, 32, 128, 256]
        plans = [(B, [B] * len(cfg.fc)) for B in batches]
        if name == "C3":
            plans.append((256, None))  # the planner under the config's budget
        for K, plan in plans:
            if plan is None:
                m.set_memory_budget(cfg.tot_bytes)
                bs, _ = m.plan(K)
            else:
                m.set_plan(plan)
                bs = plan
            a = synth.fc_inputs(cfg.fc[0].cols, K, cfg.seed)
            x = torch.from_numpy(a).to(dev)
            out = torch.zeros((K, cfg.fc[-1].rows), dtype=torch.float32, device=dev)
            for _ in range(3):
                m.infer(x, K, out, on_device=True, stream=sp)
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                m.infer(x, K, out, on_device=True, stream=sp)
                e1.record(st)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = float(np.median(ts)) / 1e3
            algo = 0.0
            for i, s in enumerate(stats):
                rounds = K // bs[i] if bs[i] else 1
                algo += rounds * (s["algo_bytes_fixed"] + 4.0 * s["cols"] * bs[i] + 4.0 * s["rows"] * bs[i])
            print(json.dumps({
                "config": name, "K": K, "plan": bs, "images_per_s": K / t, "ms": t * 1e3,
                "compressed_gbs": comp * (K / max(bs[0], 1)) / t / 1e9,
                "hbm_frac": algo / t / 1e9 / pk["hbm_gbs"],
                "kernels": [m.kernel_name(i, bs[i]) for i in range(len(cfg.fc))]}), flush=True)
        m.close()


if __name__ == "__main__":
    main()
