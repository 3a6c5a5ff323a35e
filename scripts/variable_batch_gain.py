"""Variable-batch vs fixed-batch execution under a memory budget on the device
(the synthetic analogue of the paper's Figs. 5/6 and
Table 5).  AlexNet conv1-5 + fc6-8 (config C4 weights), K images:
for each budget TOT, the library profiles Time(i, B) on the GPU, plans with the
DP of P:L694-720 (cdn_model_plan), and infer runs that plan; the baseline is the
best single batch size that fits TOT, run the same way.
Usage: python scripts/variable_batch_gain.py [--K 64] [--budgets 64,96,128,192]"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def build(cdn):
    cfg = synth.CONFIGS["C4"]
    m = cdn.Model(0)
    hw = cfg.image_hw
    for i, spec in enumerate(cfg.conv):
        W, v = synth.fc_weights(spec, cfg.seed)
        m.load_layer(cdn.compress_dense(W, spec.density, spec.r, spec.k, v),
                     cdn.LayerDesc.conv(spec.in_ch, hw, hw, spec.kh, spec.kw, spec.stride, spec.pad, spec.groups,
                                        relu=True, lrn=spec.lrn, pool_k=3 if spec.pool else 0,
                                        pool_s=2 if spec.pool else 0))
        hw = m.out_shape(i)[0]
    for spec in cfg.fc:
        W, v = synth.fc_weights(spec, cfg.seed)
        m.load_layer(cdn.compress_dense(W, spec.density, spec.r, spec.k, v), cdn.LayerDesc.fc(spec.relu))
    return m


def fixed_candidates(T, inb, outb, ws, tot, K):
    """Single batches B (all layers) by predicted time per image, those the
    recurrence's model admits (IN + WS + OUT <= TOT per layer, no ancestor
    reserve when every phase count is 1); remainder rounds at the same B are
    charged pro rata.  The caller runs them best first and keeps the first
    whose metered executor scratch stays within TOT -- the bar the planned
    run meets too (reading C-36)."""
    c = []
    for B in range(1, K + 1):
        if all(inb[i] * B + ws[i] + outb[i] * B <= tot for i in range(len(T))):
            c.append((sum(T[i][B - 1] for i in range(len(T))) / B, B))
    return [(B, per) for per, B in sorted(c)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", type=int, default=64)
    ap.add_argument("--budgets", default="48,64,96,128,144,160,192")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_1711_00244_b200 as cdn
    dev = torch.device("cuda:0")
    m = build(cdn)
    K = args.K
    f = m.num_layers()
    st = [m.stats(i) for i in range(f)]
    x = torch.from_numpy(synth.conv_inputs(K, 227, 3, seed=7)).to(dev)
    out = torch.zeros((K, 1000), dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(dev)
    m.set_memory_budget(1 << 40)
    T = m.profile(K, args.reps)
    rows = []
    for mb in [int(b) for b in args.budgets.split(",")]:
        tot = mb << 20
        m.set_memory_budget(tot)
        m.set_plan([])
        try:
            plan, pred = m.plan(K)
        except cdn.CDNError as e:
            rows.append({"tot_mib": mb, "dp": None, "error": e.name})
            continue
        res = {"tot_mib": mb, "dp_plan": plan, "dp_pred_ms": pred}
        inb, outb, ws = m.memory_model(K)

        def run(p_list):
            m.set_plan(p_list)
            with torch.cuda.stream(s):
                m.infer(x, K, out, on_device=True, stream=s.cuda_stream)
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    e0.record(s)
                    m.infer(x, K, out, on_device=True, stream=s.cuda_stream)
                    e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            return float(np.median(ts))

        m.release_scratch()
        m.scratch_bytes(reset_peak=True)
        res["dp_ms"] = run([])  # [] = no fixed plan: the executor plans with the DP
        res["dp_scratch_peak_mib"] = m.scratch_bytes()[1] / 2**20
        # fixed-batch baseline: every layer at one B, the best
        # predicted B whose run keeps the executor's scratch within TOT
        best = None
        for B, per in fixed_candidates(T, inb, outb, ws, tot, K):
            m.release_scratch()
            m.scratch_bytes(reset_peak=True)
            ms = run([B] * f)
            peak = m.scratch_bytes()[1]
            if peak <= tot:
                best = {"B": B, "pred_ms_per_image": per, "ms": ms, "scratch_peak_mib": peak / 2**20}
                break
        res["fixed_best"] = best
        if best:
            res["dp_gain"] = best["ms"] / res["dp_ms"] - 1.0
        rows.append(res)
        print(json.dumps(res), flush=True)
    m.close()


if __name__ == "__main__":
    main()
