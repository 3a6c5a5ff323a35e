"""Debug: fused split scales vs a separate max pass (bits must agree)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth
import torch
import paper_1711_00244_b200 as cdn
from test_gpu_parity import config_layer
dev = torch.device("cuda:0")
cfg = synth.CONFIGS["C3"]
outs = {}
for fuse in ("1", "0"):
    os.environ["CDN_TC_FUSE_SCALES"] = fuse
    m = cdn.Model(0)
    for i, spec in enumerate(cfg.fc):
        _, _, buf = config_layer("C3", i)
        m.load_layer(buf, cdn.LayerDesc.fc(spec.relu))
    for K, plan in ((300, [50, 100, 100]), (200, [8, 16, 32]), (256, [256, 256, 256])):
        m.set_plan(plan)
        a = synth.fc_inputs(cfg.fc[0].cols, K, 1)
        host = np.zeros((K, 1000), np.float32)
        m.infer(a, K, host, on_device=False)
        xi = torch.from_numpy(a).to(dev)
        so = torch.zeros((K, 1000), dtype=torch.float32, device=dev)
        m.infer(xi, K, so, on_device=True)
        so2 = torch.zeros((K, 1000), dtype=torch.float32, device=dev)
        m.infer(xi, K, so2, on_device=True)
        torch.cuda.synchronize()
        d = so.cpu().numpy()
        outs[(fuse, K)] = d
        print(fuse, K, plan, "host==dev", np.array_equal(host, d), "dev==dev2", np.array_equal(d, so2.cpu().numpy()),
              "kernels", [m.kernel_name(i, plan[i]) for i in range(3)], flush=True)
        if not np.array_equal(host, d):
            bad = np.argwhere(host != d)
            print("  mismatch rows(images)", np.unique(bad[:, 0])[:20], "count", len(bad))
    m.close()
for K in (300, 200, 256):
    print("fused==unfused", K, np.array_equal(outs[("1", K)], outs[("0", K)]))
