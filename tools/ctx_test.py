import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2510_01718_b200 as bd
from paper_2510_01718_b200.benchmark import ring_size, time_ring_us
dev = torch.device("cuda:0")
F, Lt = bd.Tag.FIRST, bd.Tag.LAST
def paper(L, tag):
    d, d_h, n = 512, 128, 128
    K, N = d - d_h, n * d_h
    R = ring_size(2 * (L * d + K * N + L * N))
    sets = [(torch.randn(L, d, device=dev).half(), (torch.randn(K, N, device=dev) / 8).half(),
             torch.empty(L, N, device=dev, dtype=torch.half)) for _ in range(R)]
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, F)], outs=[s[2]], check_finite=False) for s in sets]
    us = time_ring_us(calls, 613, reps=11)
    del sets, calls; torch.cuda.empty_cache()
    return us
print(tag := "fresh", [round(paper(L, 0), 2) for L in (64, 128, 64)], flush=True)
# cfg3-like heavy BF16 streaming-A run
L, d, d_h, n = 65536, 4096, 128, 32
K, N = d - d_h, n * d_h
bf = torch.bfloat16
sets = [(torch.randn(L, d, device=dev).to(bf), (torch.randn(K, N, device=dev) / 64).to(bf), (torch.randn(K, N, device=dev) / 64).to(bf),
         torch.empty(L, N, device=dev, dtype=bf), torch.empty(L, N, device=dev, dtype=bf)) for _ in range(2)]
for _ in range(3):
    for s in sets:
        bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, F), (s[2], d_h, n, Lt)], outs=[s[3], s[4]], check_finite=False)
torch.cuda.synchronize()
del sets; torch.cuda.empty_cache()
print("after cfg3", [round(paper(L, 0), 2) for L in (64, 128, 64, 64)], flush=True)
# flush L2 with a plain write of 512 MB
buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
buf.fill_(1); torch.cuda.synchronize(); del buf; torch.cuda.empty_cache()
print("after flush", [round(paper(L, 0), 2) for L in (64, 128, 64)], flush=True)
