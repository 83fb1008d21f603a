"""Minimal driver for ncu: runs the cfg2 K'+V' grouped projection (and, with --dense,
the cuBLAS comparator) a few times.  Never used for timing numbers."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd

L, d, d_h, n = 8192, 512, 128, 16
dtype = torch.bfloat16 if "--bf16" in sys.argv else torch.float16
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
dev = torch.device("cuda:0")
x = torch.randn(L, d, device=dev).to(dtype)
ck = (torch.randn(d - d_h, n * d_h, device=dev) / 8).to(dtype)
cv = (torch.randn(d - d_h, n * d_h, device=dev) / 8).to(dtype)
w = (torch.randn(d, 2 * n * d_h, device=dev) / 8).to(dtype)
for _ in range(reps):
    bd.fused_kv_proj_grouped(x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)])
    if "--dense" in sys.argv:
        torch.matmul(x, w)
torch.cuda.synchronize()
print("done")
