"""Development aid: one traced launch of the cfg2 K'+V' projection (BD_TC_TRACE=1)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d, d_h, n = 512, 128, 16
dev = torch.device("cuda:0")
x = torch.randn(L, d, device=dev).half()
ck = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
cv = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
for _ in range(3):
    bd.fused_kv_proj_grouped(x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)])
torch.cuda.synchronize()
