"""Graph-timed cfg2-shape K'+V' at L = 256 / 512 (small-L pair kernel) with x as a view of
an allocation 64x taller (so the UNSHARED_A build's per-pair row offsets stay in bounds);
run once with the normal build and once with BD_LIB_PATH=<UNSHARED_A build>."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200.benchmark import time_ring_us

dev = torch.device("cuda", 0)
d, d_h, n = 512, 128, 16
for L in (256, 512):
    sets = []
    for _ in range(24):
        big = torch.randn(L * 64, d, device=dev).half()
        sets.append((big[:L], (torch.randn(384, 2048, device=dev) / 8).half(),
                     (torch.randn(384, 2048, device=dev) / 8).half(),
                     torch.empty(L, 2048, device=dev, dtype=torch.half),
                     torch.empty(L, 2048, device=dev, dtype=torch.half)))
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, bd.Tag.FIRST),
                                                         (s[2], d_h, n, bd.Tag.LAST)],
                                                  outs=[s[3], s[4]], check_finite=False)
             for s in sets]
    print(f"L={L}: {time_ring_us(calls, 48):.2f} us", flush=True)
