"""Development aid: graph-timed FP16 projection at short and full lengths (cold-L2 ring,
benchmark.time_ring_us) for A/B of library builds (BD_LIB_PATH).  Paper k_proj shape
(d = 512, 128 heads x 128, tag FIRST) and cfg2 K'+V'.   python tools/time_short.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2510_01718_b200 as bd  # noqa: E402
from paper_2510_01718_b200.benchmark import ring_size, time_ring_us  # noqa: E402

F, Lt = bd.Tag.FIRST, bd.Tag.LAST
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(3)
h = torch.float16
cases = [("paper", L, 128, 1) for L in (64, 128, 256, 512, 1024, 4096)] + \
        [("cfg2", L, 16, 2) for L in (64, 128, 160, 256, 384, 512, 640, 768, 1024, 8192)]
if os.environ.get("TIME_SHORT_CASES"):  # e.g. "cfg2:640,cfg2:1024"
    cases = [(c.split(":")[0], int(c.split(":")[1]), 128 if c.startswith("paper") else 16,
              1 if c.startswith("paper") else 2) for c in os.environ["TIME_SHORT_CASES"].split(",")]
out = []
for name, L, n, probs in cases:
    d, d_h = 512, 128
    K, N = d - d_h, n * d_h
    R = ring_size(2 * (L * d + probs * (K * N + L * N)))
    sets = [(torch.randn(L, d, device=dev, generator=g).to(h),
             [(torch.randn(K, N, device=dev, generator=g) / 8).to(h) for _ in range(probs)],
             [torch.empty(L, N, device=dev, dtype=h) for _ in range(probs)]) for _ in range(R)]
    calls = [lambda s=s: bd.fused_kv_proj_grouped(
        s[0], [(c, d_h, n, t) for c, t in zip(s[1], (F, Lt))], outs=s[2], check_finite=False)
        for s in sets]
    us = time_ring_us(calls, max(R, int(2000 / max(1.0, L / 256))))
    out.append(f"{name} L={L}: {us:.2f}")
    del sets, calls
print(" | ".join(out), flush=True)
