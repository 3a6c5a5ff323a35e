import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import synth
import paper_1711_00244_b200 as cdn
from oracle import cdni, compress
sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
from test_gpu_conv import conv_case
cfg = synth.CONFIGS["C4"]
m = cdn.Model(0)
hw = 227
for i, spec in enumerate(cfg.conv):
    _, c, buf, v = conv_case(i)
    m.load_layer(buf, cdn.LayerDesc.conv(spec.in_ch, hw, hw, spec.kh, spec.kw, spec.stride, spec.pad, spec.groups, relu=True, lrn=spec.lrn, pool_k=3 if spec.pool else 0, pool_s=2 if spec.pool else 0))
    hw = m.out_shape(i)[0]
for spec in cfg.fc:
    W, v = synth.fc_weights(spec, cfg.seed)
    c = compress.compress_layer(W, spec.density, spec.r, spec.k, v)
    m.load_layer(cdni.serialize([c.layer]), cdn.LayerDesc.fc(spec.relu))
print([m.kernel_name(i, 8) for i in range(8)])
print("memory model", m.memory_model(32))
print("profile", np.array(m.profile(32, 3)).reshape(8, 32)[:, [0, 1, 3, 7, 15, 31]])
m.set_memory_budget(128 << 20)
try:
    print(m.plan(32))
except Exception as e:
    print("plan failed", e)
