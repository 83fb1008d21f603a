"""Development aid: can the kernels read x from / write K', V' to pinned host memory
directly (UVA), and what does that do to the end-to-end step?"""
import sys, time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import _native as N
from paper_2510_01718_b200.kv_proj import _problem, _on_device

L, d, d_h, n = 8192, 512, 128, 16
dev = torch.device("cuda:0")
ck = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
cv = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
xh = torch.randn(L, d).half().pin_memory()
kh = torch.empty(L, n * d_h, dtype=torch.half).pin_memory()
vh = torch.empty_like(kh).pin_memory()
specs = [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)]
ref = bd.fused_kv_proj_grouped(xh.to(dev), specs)
lib = N.load()


def zc_call(x_ptr_tensor):
    probs = (N.KvProblem * 2)()
    for i, (c, tag) in enumerate([(ck, bd.Tag.FIRST), (cv, bd.Tag.LAST)]):
        o = kh if i == 0 else vh
        probs[i] = _problem(x_ptr_tensor, c, o, d_h, n, tag)
    st = _on_device(dev, lib.bd_kv_proj_grouped_ex, probs, 2, N.BD_F16, 0, 0, None)
    return st


for name, xsrc in (("x in HBM, out pinned host", xh.to(dev)), ("x and out pinned host", xh)):
    st = zc_call(xsrc)
    torch.cuda.synchronize()
    print(name, "status", st, N.last_error() if st else "",
          "equal:", torch.equal(kh.to(dev), ref[0]) and torch.equal(vh.to(dev), ref[1]))
    if st == 0:
        for _ in range(3):
            zc_call(xsrc)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(20):
            zc_call(xsrc)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 20
        print(f"   {dt*1e3:.3f} ms/step  {L/dt/1e6:.2f} M tok/s")
t = time.perf_counter()
for _ in range(20):
    bd.fused_kv_proj_grouped_host(xh, specs, outs=[kh, vh])
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 20
print(f"staged host pipeline: {dt*1e3:.3f} ms/step  {L/dt/1e6:.2f} M tok/s")
