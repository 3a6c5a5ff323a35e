import time, json, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth, paper_1711_00244_b200 as cdn
from paper_1711_00244_b200 import build
build.build()
cfg = synth.CONFIGS["C5"]
m = cdn.Model(0)
for i, spec in enumerate(cfg.fc):
    W, v = synth.fc_weights(spec, cfg.seed)
    m.load_layer(cdn.compress_dense(W, spec.density, spec.r, spec.k, v), cdn.LayerDesc.fc(spec.relu))
B = 512
m.set_plan([B] * 3)
dev = torch.device("cuda:0")
a = synth.fc_inputs(cfg.fc[0].cols, B, cfg.seed)
x = torch.from_numpy(a).to(dev); s_out = torch.zeros((B, cfg.fc[-1].rows), device=dev)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st); sp = st.cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(5): m.infer(x, B, s_out, on_device=True, stream=sp)
torch.cuda.synchronize()
def timed(fn, n=20):
    tot = 0.0
    for _ in range(n):
        flush.zero_(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); fn(); e1.record(st); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n
print("eager ms/step", timed(lambda: m.infer(x, B, s_out, on_device=True, stream=sp)))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
    m.infer(x, B, s_out, on_device=True, stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("graph ms/step", timed(lambda: g.replay()))
