"""Development aid: launches for ncu — the small-L kernel (paper shape L=64 and cfg2 L=64)
and the fused-norm cfg2 launch."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd

dev = torch.device("cuda:0")
d, d_h = 512, 128
x = torch.randn(8192, d, device=dev).half()
c128 = (torch.randn(d - d_h, 128 * d_h, device=dev) / 8).half()
ck = (torch.randn(d - d_h, 16 * d_h, device=dev) / 8).half()
cv = (torch.randn(d - d_h, 16 * d_h, device=dev) / 8).half()
gamma = 0.5 + torch.rand(d, device=dev)
fk = bd.fold_rmsnorm(ck, gamma, d_h, bd.Tag.FIRST)
fv = bd.fold_rmsnorm(cv, gamma, d_h, bd.Tag.LAST)
for _ in range(3):
    bd.fused_kv_proj(x[:64].contiguous(), c128, d_h, 128, bd.Tag.FIRST, check_finite=False)
    bd.fused_kv_proj_grouped(x[:64].contiguous(), [(ck, d_h, 16, bd.Tag.FIRST), (cv, d_h, 16, bd.Tag.LAST)])
    bd.fused_rmsnorm_kv_proj_grouped(x, [(fk[0], fk[1], d_h, 16, bd.Tag.FIRST),
                                         (fv[0], fv[1], d_h, 16, bd.Tag.LAST)], 1e-6)
torch.cuda.synchronize()
print("done")
