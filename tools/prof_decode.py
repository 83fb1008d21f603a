"""Minimal launch sequence of the decode-sized projection for ncu captures and single-launch
timing: SHAPE (cfg2 | paper), L; a few eager launches (the capture takes one), then the
median CUDA-event time of isolated launches.   python tools/prof_decode.py cfg2 64"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd

shape, L = sys.argv[1], int(sys.argv[2])
n, nprob = (16, 2) if shape == "cfg2" else (128, 1)
d, d_h = 512, 128
dev = torch.device("cuda:0")
x = torch.randn(L, d, device=dev).half()
cs = [(torch.randn(d - d_h, n * d_h, device=dev) / 8).half() for _ in range(nprob)]
specs = [(c, d_h, n, t) for c, t in zip(cs, [bd.Tag.FIRST, bd.Tag.LAST])]
outs = [torch.empty(L, n * d_h, device=dev, dtype=torch.half) for _ in range(nprob)]
ts = []
for i in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    bd.fused_kv_proj_grouped(x, specs, outs=outs, check_finite=False)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"{shape} L={L}: isolated launch median {ts[len(ts) // 2]:.2f} us (min {ts[0]:.2f})")
