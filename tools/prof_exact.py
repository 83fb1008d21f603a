import sys; sys.path.insert(0, ".")
import torch, paper_2510_01718_b200 as bd
dev = torch.device("cuda")
x = torch.randn(256, 512, device=dev); ck = torch.randn(448, 512, device=dev) / 8; cv = torch.randn(448, 512, device=dev) / 8
for _ in range(3):
    bd.fused_kv_proj_grouped(x, [(ck, 64, 8, bd.Tag.FIRST), (cv, 64, 8, bd.Tag.LAST)])
torch.cuda.synchronize()
