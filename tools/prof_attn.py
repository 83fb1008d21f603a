import math, sys, torch
sys.path.insert(0, '.')
from paper_2510_01718_b200 import mla as M
L, H = 8192, 16
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q = torch.randn(L, H, 192, device=dev, generator=g).half()
k = torch.randn(H, L, 128, device=dev, generator=g).half()
kpe = torch.randn(L, 64, device=dev, generator=g).half()
v = torch.randn(H, L, 128, device=dev, generator=g).half()
out = torch.empty(L, H, 128, device=dev, dtype=torch.half)
for _ in range(3):
    M.mla_attention(q, k, kpe, v, scale=1 / math.sqrt(192), out=out)
torch.cuda.synchronize()
