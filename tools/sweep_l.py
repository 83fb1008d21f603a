"""Development aid: CUDA-graph timing of the grouped K'+V' projection at several token
counts (separates the per-launch fixed cost from the per-tile cost).  Not a bench."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd

d, d_h, n = 512, 128, 16
dtype = torch.float16
dev = torch.device("cuda:0")
label = sys.argv[1] if len(sys.argv) > 1 else ""
Ls = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [256, 1024, 2048, 4096, 8192, 16384]
ck = (torch.randn(d - d_h, n * d_h, device=dev) / 8).to(dtype)
cv = (torch.randn(d - d_h, n * d_h, device=dev) / 8).to(dtype)
for L in Ls:
    x = torch.randn(L, d, device=dev).to(dtype)
    k = torch.empty(L, n * d_h, device=dev, dtype=dtype)
    v = torch.empty(L, n * d_h, device=dev, dtype=dtype)

    def step():
        bd.fused_kv_proj_grouped(x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)],
                                 outs=[k, v], check_finite=False)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=s):
        for _ in range(40):
            step()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            g.replay()
            b.record(s)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 40 * 1e3)
    print(f"{label} L={L} us={best:.2f}", flush=True)
