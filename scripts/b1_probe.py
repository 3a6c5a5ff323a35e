"""B = 1 probe of the small-batch FC kernels: correctness against a dense fp64
product of the host-walk tokens, and cold-L2 per-launch time over R resident
replicas (the bench's b1_cold protocol).  Usage: python scripts/b1_probe.py [R]"""
import json
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
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6542.4
    out = {}
    todo = [("C5", 0), ("C5", 1), ("C5", 2), ("C2", 0), ("C1", 0)]
    if os.environ.get("B1_LAYERS"):  # e.g. "C5:0,C2:0"
        todo = [(c.split(":")[0], int(c.split(":")[1])) for c in os.environ["B1_LAYERS"].split(",")]
    for cfg, li in todo:
        spec = synth.CONFIGS[cfg].fc[li]
        W, v = synth.fc_weights(spec, synth.CONFIGS[cfg].seed)
        buf = cdn.compress_dense(W, spec.density, spec.r, spec.k, v)
        del W
        ms = [cdn.Model(0) for _ in range(R)]
        for m in ms:
            m.load_layer(buf, cdn.LayerDesc.fc(False))
        st = ms[0].stats(0)
        kname = ms[0].kernel_name(0, 1)
        a = synth.fc_inputs(spec.cols, 1, 0)
        x = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)
        y = torch.zeros((spec.rows, 1), dtype=torch.float32, device=dev)
        ms[0].layer_forward(0, x, 1, 1, y, 1, stream=sp)
        torch.cuda.synchronize()
        row, col, sym = cdn.debug_host_walk(buf)
        from oracle import cdni as ocdni
        cb = np.asarray(ocdni.deserialize(buf)[0].codebook, dtype=np.float64)
        real = sym != 0
        ref = np.zeros(spec.rows)
        np.add.at(ref, row[real], cb[sym[real]] * a[0, col[real]].astype(np.float64))
        ref += v
        yy = y.cpu().numpy()[:, 0]
        err = float(np.abs(yy - ref).max() / np.abs(ref).max())
        for m in ms:
            m.layer_forward(0, x, 1, 1, y, 1, stream=sp)
        samples = []
        for _ in range(7):
            flush.zero_()
            torch.cuda.synchronize()
            torch.cuda._sleep(3_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for m in ms:
                m.layer_forward(0, x, 1, 1, y, 1, stream=sp)
            e1.record(stream)
            torch.cuda.synchronize()
            samples.append(e0.elapsed_time(e1) / R)
        t = float(np.median(samples))
        algo = st["algo_bytes_fixed"] + 4 * spec.cols + 4 * spec.rows
        out[f"{cfg}_{spec.name}"] = {"kernel": kname, "us": t * 1e3, "frac": algo / (t / 1e3) / 1e9 / hbm,
                                     "rel_err": err}
        print(cfg, spec.name, out[f"{cfg}_{spec.name}"], flush=True)
        for m in ms:
            m.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
