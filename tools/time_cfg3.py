"""Development aid: cfg3 (Llama-2-7B K+V, BF16, d=4096) and cfg4 GEMM timing vs cuBLAS."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import benchmark as B

label = sys.argv[1] if len(sys.argv) > 1 else ""
L = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
d, d_h, n = 4096, 128, 32
x = torch.randn(L, d, device=dev, generator=g).to(torch.bfloat16)
ck = (torch.randn(d - d_h, n * d_h, device=dev, generator=g) / 64).to(torch.bfloat16)
cv = (torch.randn(d - d_h, n * d_h, device=dev, generator=g) / 64).to(torch.bfloat16)
w = (torch.randn(d, 2 * n * d_h, device=dev, generator=g) / 64).to(torch.bfloat16)
ko = torch.empty(L, n * d_h, device=dev, dtype=torch.bfloat16)
vo = torch.empty_like(ko)
do = torch.empty(L, 2 * n * d_h, device=dev, dtype=torch.bfloat16)
bd_ns = B.time_operator_ns(lambda: bd.fused_kv_proj_grouped(
    x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)], outs=[ko, vo]), inner=3)
dn_ns = B.time_operator_ns(lambda: torch.matmul(x, w, out=do), inner=3)
fl = 2 * 2 * L * (d - d_h) * n * d_h
print(f"{label} cfg3 L={L}: bd {bd_ns/1e3:.1f} us ({fl/bd_ns/1e3:.0f} TF)  cublas {dn_ns/1e3:.1f} us  ratio {dn_ns/bd_ns:.3f}")
