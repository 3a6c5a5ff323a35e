"""Host->device copy throughput from pinned memory on this box: one copy vs
chunked copies on 1, 2, 4 streams, at the C5 B=512 input size (51 MB).
JSON lines.  Usage: python scripts/h2d_probe.py"""
import json

import numpy as np
import torch


def main():
    dev = torch.device("cuda:0")
    n = 512 * 25088
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float32, device=dev)
    streams = [torch.cuda.Stream(dev) for _ in range(4)]
    main_s = torch.cuda.current_stream(dev)
    for chunks, ns in ((1, 1), (4, 1), (8, 1), (4, 2), (8, 2), (4, 4), (8, 4), (16, 4)):
        ts = []
        for r in range(25):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main_s)
            c = n // chunks
            evs = []
            for k in range(chunks):
                s = streams[k % ns]
                s.wait_event(e0) if k < ns else None
                with torch.cuda.stream(s):
                    d[k * c:(k + 1) * c].copy_(h[k * c:(k + 1) * c], non_blocking=True)
            for s in streams[:ns]:
                main_s.wait_stream(s)
            e1.record(main_s)
            torch.cuda.synchronize()
            if r >= 5:
                ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        print(json.dumps({"chunks": chunks, "streams": ns, "ms": t, "gbs": n * 4 / t / 1e6,
                          "min_ms": float(min(ts)), "max_ms": float(max(ts))}), flush=True)


if __name__ == "__main__":
    main()
