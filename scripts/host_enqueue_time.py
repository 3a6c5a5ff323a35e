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
for _ in range(5): m.infer(x, B, s_out, on_device=True, stream=sp)
torch.cuda.synchronize()
for rep in range(5):
    torch.cuda._sleep(5_000_000)   # keep GPU busy so the host measurement is pure enqueue
    t0 = time.perf_counter(); m.infer(x, B, s_out, on_device=True, stream=sp); t1 = time.perf_counter()
    torch.cuda.synchronize()
    print("host enqueue us", (t1 - t0) * 1e6)
# GPU time with host ahead
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(20_000_000)
e0.record(st)
for _ in range(10): m.infer(x, B, s_out, on_device=True, stream=sp)
e1.record(st)
torch.cuda.synchronize()
print("gpu ms per step (host ahead, back to back, no flush)", e0.elapsed_time(e1) / 10)
# the same step replayed from a CUDA graph captured around infer (potential of graph launch)
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g, stream=st, capture_error_mode="relaxed"):
        m.infer(x, B, s_out, on_device=True, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = s_out.clone()
    torch.cuda._sleep(20_000_000)
    e0.record(st)
    for _ in range(10):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    print("graph replay ms per step", e0.elapsed_time(e1) / 10)
    m.infer(x, B, s_out, on_device=True, stream=sp); torch.cuda.synchronize()
    print("graph result matches eager:", bool(torch.equal(ref, s_out)))
except Exception as ex:
    print("capture failed:", ex)
