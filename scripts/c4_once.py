import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth, paper_1711_00244_b200 as cdn
from paper_1711_00244_b200 import build
build.build()
import bench
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
cdn.kernel_timer(False)
r = bench.bench_c4(cdn, torch, dev, flush, 3)
print(r)
