"""End-to-end (pinned host input -> host scores) images/s of the C5 stack under
several batch plans: the executor's H2D prefetch overlaps a first-layer
phase's copy with the previous phase's compute, so a finer first level trades
tensor-core efficiency for overlap.  Also checks each plan's scores against
the device-resident call.  JSON lines.
Usage: python scripts/e2e_plans.py [--reps 20]"""
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
    ap.add_argument("--numa", type=int, default=1, help="pin to the GPU's local CPUs before pinning memory")
    args = ap.parse_args()
    import torch
    import paper_1711_00244_b200 as cdn
    from paper_1711_00244_b200 import build
    build.build()
    dev = torch.device("cuda:0")
    pr = torch.cuda.get_device_properties(dev)
    sysd = "/sys/bus/pci/devices/%04x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
    info = {"pci": sysd, "cpus_before": len(os.sched_getaffinity(0))}
    try:
        info["numa_node"] = open(sysd + "/numa_node").read().strip()
        cl = open(sysd + "/local_cpulist").read().strip()
        info["local_cpulist"] = cl
        if args.numa:
            cpus = set()
            for part in cl.split(","):
                a, _, b = part.partition("-")
                cpus.update(range(int(a), int(b or a) + 1))
            os.sched_setaffinity(0, cpus)
    except OSError as e:
        info["err"] = str(e)
    info["cpus_after"] = len(os.sched_getaffinity(0))
    print(json.dumps(info), flush=True)
    cfg = synth.CONFIGS["C5"]
    m = cdn.Model(0)
    for spec in cfg.fc:
        W, v = synth.fc_weights(spec, cfg.seed)
        m.load_layer(cdn.compress_dense(W, spec.density, spec.r, spec.k, v), cdn.LayerDesc.fc(spec.relu))
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    sp = st.cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for K in (512, 1024):  # the copy alone: the floor of any plan
        h = torch.empty((K, cfg.fc[0].cols), dtype=torch.float32).pin_memory()
        d = torch.empty((K, cfg.fc[0].cols), dtype=torch.float32, device=dev)
        d.copy_(h, non_blocking=True)
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            d.copy_(h, non_blocking=True)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        print(json.dumps({"K": K, "h2d_only_ms": t, "h2d_gbs": h.numel() * 4 / t / 1e6,
                          "images_per_s_ceiling": K / t * 1e3}), flush=True)
    for K, plan in ((512, [512, 512, 512]), (512, [256, 512, 512]), (512, [128, 512, 512]),
                    (512, [128, 256, 512]), (512, [64, 512, 512]), (1024, [512, 512, 512]),
                    (1024, [256, 512, 512])):
        a = synth.fc_inputs(cfg.fc[0].cols, K, cfg.seed)
        a_pin = torch.from_numpy(a).pin_memory()
        s_pin = torch.zeros((K, cfg.fc[-1].rows), dtype=torch.float32).pin_memory()
        m.set_plan(plan)
        x = torch.from_numpy(a).to(dev)
        ref = torch.zeros((K, cfg.fc[-1].rows), dtype=torch.float32, device=dev)
        m.infer(x, K, ref, on_device=True, stream=sp)
        for _ in range(3):
            m.infer(a_pin, K, s_pin, on_device=False, stream=sp)
        torch.cuda.synchronize()
        err = float((s_pin - ref.cpu()).abs().max())
        ts = []
        for _ in range(args.reps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            m.infer(a_pin, K, s_pin, on_device=False, stream=sp)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        print(json.dumps({"K": K, "plan": plan, "e2e_images_per_s": K / t * 1e3, "ms": t,
                          "h2d_gbs": K * cfg.fc[0].cols * 4 / t / 1e6, "max_abs_vs_device": err}), flush=True)
    m.close()


if __name__ == "__main__":
    main()
