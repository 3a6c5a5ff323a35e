"""Multi-GPU readiness on one GPU: each rank's
compute of the C5 stack at B = 512 with row-block shards (all-gather after
each layer) or Megatron-style column blocks (reduce-scatter / reduce), timed
through shard-only handles
(rank r of G, no communicator) -- cdn_layer_forward per layer on the rank's
rows, tensor-core policy as in bench.py, L2 flushed before each step.  The
slowest rank per G bounds the sharded compute; the all-gathers it would add
(4 rows_r B bytes per rank per layer into every rank) are estimated at the
measured NVLink peer bandwidth (770 GB/s per direction, B200_PROFILING.md).
Writes one JSON object (profiles/r02_shard_timing.json)."""
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
    dev = torch.device("cuda:0")
    s = torch.cuda.Stream(dev)
    torch.cuda.set_stream(s)
    B = 512
    cfg = synth.CONFIGS["C5"]
    bufs = []
    for spec in cfg.fc:
        W, v = synth.fc_weights(spec, cfg.seed)
        bufs.append(cdn.compress_dense(W, spec.density, spec.r, spec.k, v))
        del W
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    mode = sys.argv[1] if len(sys.argv) > 1 else "rows"
    out = {"B": B, "mode": mode,
           "workload": f"C5 fc6/fc7/fc8 {mode} shards, cdn_layer_forward per layer, tensor-core policy", "per_G": {}}
    for G in (1, 2, 4, 8):
        ranks = []
        for r in range(G):
            m = cdn.Model(0, rank=r, world=G)
            if mode == "cols":
                m.set_sharding(cdn.CDN_SHARD_COLS)
            for spec, buf in zip(cfg.fc, bufs):
                m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
            m.set_kernel_policy(0, 16)
            st = [m.stats(i) for i in range(3)]
            xs = [torch.from_numpy(np.ascontiguousarray(
                synth.fc_inputs(spec.cols, B, 0)[:, st[i]["col_begin"]:max(st[i]["col_end"], st[i]["col_begin"] + 1)].T))
                .to(dev) for i, spec in enumerate(cfg.fc)]
            ys = [torch.zeros((st[i]["row_end"] - st[i]["row_begin"], B), dtype=torch.float32, device=dev)
                  for i in range(3)]

            def step():
                for i in range(3):
                    m.layer_forward(i, xs[i], B, B, ys[i], B, stream=s.cuda_stream)
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            # the rank's step captured once as a CUDA graph (as infer replays its
            # calls): launch gaps out of the per-rank compute time
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                step()
            ts, te = [], []
            for _ in range(10):
                for replay, acc in ((True, ts), (False, te)):
                    flush.zero_()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    if replay:
                        g.replay()
                    else:
                        step()
                    e1.record(s)
                    torch.cuda.synchronize()
                    acc.append(e0.elapsed_time(e1))
            rows = [st[i]["row_end"] - st[i]["row_begin"] for i in range(3)]
            cols = [st[i]["col_end"] - st[i]["col_begin"] for i in range(3)]
            ranks.append({"rank": r, "rows": rows, "cols": cols, "ms": float(np.median(ts)),
                          "ms_eager": float(np.median(te))})
            del g
            m.close()
        worst = max(x["ms"] for x in ranks)
        # rows: all-gather of fc6 and fc7 outputs (fc8's scores go to rank 0 only), each
        # rank receives (G-1) slabs of rows_r x B fp32 per layer; cols: reduce-scatter of
        # fc6 / fc7 partials (each rank sends / receives (G-1) blocks of per x B) and the
        # reduce of fc8's to rank 0 -- the same bytes per layer
        ag_bytes = sum((G - 1) * 4.0 * B * ((spec.rows + G - 1) // G) for spec in cfg.fc[:2])
        ag_ms = ag_bytes / 770e9 * 1e3 if G > 1 else 0.0
        out["per_G"][G] = {"ranks": ranks, "max_rank_ms": worst, "allgather_bytes_in_per_rank": ag_bytes,
                           "allgather_ms_at_770GBs": ag_ms}
        print(G, worst, ag_ms, flush=True)
    t1 = out["per_G"][1]["max_rank_ms"]
    for G, v in out["per_G"].items():
        v["compute_speedup"] = t1 / v["max_rank_ms"]
        v["speedup_no_overlap_est"] = t1 / (v["max_rank_ms"] + v["allgather_ms_at_770GBs"])
        v["speedup_full_overlap_est"] = t1 / max(v["max_rank_ms"], v["allgather_ms_at_770GBs"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
