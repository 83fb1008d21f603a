"""Development aid: one launch of the cfg2 K'+V' projection with an instrumented build
(BD_LIB_PATH=exp/v3stamp.so BD_STAMPS=1) printing pair 0's per-role clock stamps."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import os
import torch

import paper_2510_01718_b200 as bd

L, d, d_h, n = 8192, 512, 128, 16
dev = torch.device("cuda:0")
x = torch.randn(L, d, device=dev).half()
ck = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
cv = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
stamps = os.environ.pop("BD_STAMPS", None)
for _ in range(int(os.environ.get("WARM", "5"))):
    bd.fused_kv_proj_grouped(x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)])
if os.environ.get("WARM") is None:
    torch.cuda.synchronize()
if stamps:
    os.environ["BD_STAMPS"] = stamps
bd.fused_kv_proj_grouped(x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)])
torch.cuda.synchronize()
