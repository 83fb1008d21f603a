"""Time the FP32/FP64 exact kernel (kv_proj_exact.cu) on a few shapes: graph-timed ring
of buffer sets larger than L2.  BD_LIB_PATH selects the library (A/B against xb/ builds).
    python tools/time_exact.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2510_01718_b200 as bd  # noqa: E402
from paper_2510_01718_b200.benchmark import ring_size, time_ring_us  # noqa: E402

F, Lt = bd.Tag.FIRST, bd.Tag.LAST
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(5)
for (L, d, d_h, n, dt) in [(256, 512, 64, 8, torch.float32), (1024, 512, 128, 16, torch.float32),
                           (8192, 512, 128, 16, torch.float32), (32768, 512, 128, 16, torch.float32),
                           (8192, 512, 128, 16, torch.float64)]:
    K, N = d - d_h, n * d_h
    es = torch.finfo(dt).bits // 8
    R = ring_size(es * (L * d + 2 * K * N + 2 * L * N))
    sets = [(torch.randn(L, d, device=dev, generator=g).to(dt),
             (torch.randn(K, N, device=dev, generator=g) / 8).to(dt),
             (torch.randn(K, N, device=dev, generator=g) / 8).to(dt),
             torch.empty(L, N, device=dev, dtype=dt), torch.empty(L, N, device=dev, dtype=dt))
            for _ in range(R)]
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, F), (s[2], d_h, n, Lt)],
                                                  outs=[s[3], s[4]], check_finite=False)
             for s in sets]
    us = time_ring_us(calls, max(R, 8 if L >= 8192 else 200))
    mul_add = 2 * L * K * N
    print(f"L={L:6d} n={n:2d} d_h={d_h:3d} {str(dt)[6:]}: {us:9.1f} us  "
          f"{2 * mul_add / us / 1e6:6.1f} TFLOP/s (mul+add)", flush=True)
    del sets, calls
