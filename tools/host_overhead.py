"""Development aid: host-side cost per eager call of the grouped K'+V' projection (ctypes
wrapper + C ABI + tensor-map encoding + launch), vs the device time.  Not a bench."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import _native as N

L, d, d_h, n = 8192, 512, 128, 16
dev = torch.device("cuda:0")
x = torch.randn(L, d, device=dev).half()
ck = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
cv = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
k = torch.empty(L, n * d_h, device=dev, dtype=torch.half)
v = torch.empty_like(k)
specs = [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)]
for _ in range(20):
    bd.fused_kv_proj_grouped(x, specs, outs=[k, v])
torch.cuda.synchronize()
R = 200
t0 = time.perf_counter()
for _ in range(R):
    bd.fused_kv_proj_grouped(x, specs, outs=[k, v])
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"python API: host {1e6 * (t1 - t0) / R:.1f} us/call, wall incl. drain {1e6 * (t2 - t0) / R:.1f} us/call")
# raw C ABI (problems prebuilt): isolates the library's own host cost
lib = N.load()
probs = (N.KvProblem * 2)()
for i, (c, tag) in enumerate([(ck, 0), (cv, 1)]):
    o = k if i == 0 else v
    probs[i] = N.KvProblem(x.data_ptr(), c.data_ptr(), o.data_ptr(), d, n * d_h, n * d_h, L, d, d_h, n,
                           d_h if tag == 0 else 0, 0 if tag == 0 else d - d_h)
stream = torch.cuda.current_stream().cuda_stream
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(R):
    lib.bd_kv_proj_grouped(probs, 2, N.BD_F16, 0, None, stream)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"C ABI: host {1e6 * (t1 - t0) / R:.1f} us/call, wall incl. drain {1e6 * (t2 - t0) / R:.1f} us/call")
import os
if os.environ.get("NOPROF"): sys.exit(0)
import cProfile
import pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(R):
    bd.fused_kv_proj_grouped(x, specs, outs=[k, v])
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
