"""Medium-batch probe: per FC config layer and batch, the warm per-call time of
the merged-stream medium split (k_fc_j + k_j_reduce, forced by a kernel
policy with no large-batch kernels) beside the tensor-core and band kernels,
and the kernel the default autotune keeps.  Prints one JSON line per
(layer, B).  Usage: python scripts/jm_probe.py [B ...]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def timed(torch, m, x, B, y, sp, reps=20):
    m.layer_forward(0, x, B, B, y, B, stream=sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        m.layer_forward(0, x, B, B, y, B, stream=sp)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    import torch
    import paper_1711_00244_b200 as cdn
    from paper_1711_00244_b200 import build
    build.build()
    Bs = [int(a) for a in sys.argv[1:]] or [5, 8, 16, 32, 64, 128]
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    layers = [("C5", 0), ("C5", 1), ("C5", 2), ("C2", 0), ("C3", 0), ("C3", 1), ("C3", 2), ("C1", 0)]
    if os.environ.get("JM_LAYERS"):  # e.g. "C5:0,C2:0"
        layers = [(t.split(":")[0], int(t.split(":")[1])) for t in os.environ["JM_LAYERS"].split(",")]
    for cfg, li in layers:
        spec = synth.CONFIGS[cfg].fc[li]
        W, v = synth.fc_weights(spec, synth.CONFIGS[cfg].seed)
        buf = cdn.compress_dense(W, spec.density, spec.r, spec.k, v)
        del W
        m = cdn.Model(0)
        m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
        for B in Bs:
            a = synth.fc_inputs(spec.cols, B, 0)
            x = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)
            y = torch.zeros((spec.rows, B), dtype=torch.float32, device=dev)
            r = {"layer": f"{cfg} fc{li}", "rows": spec.rows, "cols": spec.cols, "B": B}
            m.set_kernel_policy(1 << 20, 1 << 20)
            r["jm_kernel"] = m.kernel_name(0, B)
            r["jm_us"] = timed(torch, m, x, B, y, sp)
            cdn.kernel_timer(True)
            timed(torch, m, x, B, y, sp)
            for k in ("k_fc_jm", "k_j_reduce"):
                t, n = cdn.kernel_time(k)
                r[k + "_us"] = t / max(n, 1) * 1e3
            cdn.kernel_timer(False)
            yj = y.cpu().numpy()
            if os.environ.get("JM_ONLY"):
                print(json.dumps(r), flush=True)
                continue
            m.set_kernel_policy(1, 1 << 20)
            r["band_us"] = timed(torch, m, x, B, y, sp) if B >= 8 else None
            m.set_kernel_policy(0, 1)
            r["tc_us"] = timed(torch, m, x, B, y, sp)
            yt = y.cpu().numpy()
            r["jm_vs_tc_rel"] = float(np.abs(yj - yt).max() / max(np.abs(yt).max(), 1e-30))
            m.set_kernel_policy(0, 0)
            r["auto_us"] = timed(torch, m, x, B, y, sp)
            r["auto_kernel"] = m.kernel_name(0, B)
            print(json.dumps(r), flush=True)
        m.close()


if __name__ == "__main__":
    main()
