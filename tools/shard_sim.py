"""Per-rank work of the head-sharded weak-scaling bench, simulated on one GPU: rank r of g
projects g x 8192 tokens for 16/g heads of K' and of V' (cfg2), cold-L2 ring, CUDA graph.
The kernel time per rank at g = 1, 2, 4, 8 is what the multi-GPU bench's efficiency is
made of (there is no collective in its timed region).   python tools/shard_sim.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200.benchmark import ring_size, time_ring_us

dev = torch.device("cuda", 0)
d, d_h, K = 512, 128, 384
g0 = torch.Generator(device=dev).manual_seed(0)
base = None
for g in (1, 2, 4, 8):
    L, n = 8192 * g, 16 // g
    N = n * d_h
    R = ring_size(2 * (L * d + 2 * K * N + 2 * L * N))
    sets = [(torch.randn(L, d, device=dev, generator=g0).half(),
             (torch.randn(K, N, device=dev, generator=g0) / 8).half(),
             (torch.randn(K, N, device=dev, generator=g0) / 8).half(),
             torch.empty(L, N, device=dev, dtype=torch.half),
             torch.empty(L, N, device=dev, dtype=torch.half)) for _ in range(R)]
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, bd.Tag.FIRST),
                                                         (s[2], d_h, n, bd.Tag.LAST)],
                                                  outs=[s[3], s[4]], check_finite=False)
             for s in sets]
    us = time_ring_us(calls, max(R, 40))
    base = base or us
    print(f"g={g}: {L} tokens x {n}+{n} heads per rank: {us:.2f} us per step "
          f"(weak-scaling efficiency of the kernel {base / us:.3f})", flush=True)
    del sets, calls
    torch.cuda.empty_cache()
