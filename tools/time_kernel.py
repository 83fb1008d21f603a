"""Quick CUDA-event timing of the cfg2 K'+V' grouped projection (development aid;
the contract numbers come from bench.py).  Usage: time_kernel.py [label] [--dense]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd

L, d, d_h, n = 8192, 512, 128, 16
dtype = torch.float16
dev = torch.device("cuda:0")
R = 5
xs = [torch.randn(L, d, device=dev).to(dtype) for _ in range(R)]
cks = [(torch.randn(d - d_h, n * d_h, device=dev) / 8).to(dtype) for _ in range(R)]
cvs = [(torch.randn(d - d_h, n * d_h, device=dev) / 8).to(dtype) for _ in range(R)]
ks = [torch.empty(L, n * d_h, device=dev, dtype=dtype) for _ in range(R)]
vs = [torch.empty(L, n * d_h, device=dev, dtype=dtype) for _ in range(R)]
ws = [(torch.randn(d, 2 * n * d_h, device=dev) / 8).to(dtype) for _ in range(R)]
outs = [torch.empty(L, 2 * n * d_h, device=dev, dtype=dtype) for _ in range(R)]


def step(i):
    j = i % R
    bd.fused_kv_proj_grouped(xs[j], [(cks[j], d_h, n, bd.Tag.FIRST), (cvs[j], d_h, n, bd.Tag.LAST)],
                             outs=[ks[j], vs[j]])


def dense(i):
    j = i % R
    torch.matmul(xs[j], ws[j], out=outs[j])


def timeit(fn):
    for i in range(10):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=s):
        for i in range(50):
            fn(i)
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            g.replay()
            b.record(s)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 50 * 1e3)
    return best


label = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else ""
print(f"{label} bd us/step {timeit(step):.2f}", flush=True)
if "--dense" in sys.argv:
    print(f"{label} dense cublas us/step {timeit(dense):.2f}", flush=True)
