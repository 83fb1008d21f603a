"""Development aid: cfg2 K'+V' with the RMSNorm fused vs RMSNorm (torch) + projection."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import benchmark as B
from paper_2510_01718_b200.mla import _rms_norm

L, d, d_h, n, eps = 8192, 512, 128, 16, 1e-6
dev = torch.device("cuda:0")
x = torch.randn(L, d, device=dev).half()
gamma = (0.5 + torch.rand(d, device=dev))
ck = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
cv = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
fk = bd.fold_rmsnorm(ck, gamma, d_h, bd.Tag.FIRST)
fv = bd.fold_rmsnorm(cv, gamma, d_h, bd.Tag.LAST)
specs_f = [(fk[0], fk[1], d_h, n, bd.Tag.FIRST), (fv[0], fv[1], d_h, n, bd.Tag.LAST)]
specs = [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)]
k = torch.empty(L, n * d_h, device=dev, dtype=torch.half)
v = torch.empty_like(k)
g16 = gamma.half()
t_fused = B.time_operator_ns(lambda: bd.fused_rmsnorm_kv_proj_grouped(x, specs_f, eps, outs=[k, v], check_finite=False), inner=20)
t_proj = B.time_operator_ns(lambda: bd.fused_kv_proj_grouped(x, specs, outs=[k, v], check_finite=False), inner=20)
t_unf = B.time_operator_ns(lambda: bd.fused_kv_proj_grouped(_rms_norm(x, g16, eps), specs, outs=[k, v], check_finite=False), inner=20)
print(f"fused norm+proj {t_fused/1e3:.2f} us | proj alone {t_proj/1e3:.2f} us | torch rmsnorm + proj {t_unf/1e3:.2f} us")
