"""Development aid: A/B timing of the cfg2 K'+V' launch (and the fused-RMSNorm variant)
exactly as bench.py times it — cold-L2 ring of buffer sets, CUDA graph, CUDA events.
Run once per build with BD_LIB_PATH=xb/<build>.so, interleaving builds:

    for i in 1 2; do for b in base new; do BD_LIB_PATH=xb/$b.so python tools/ab_cfg2.py $b; done; done
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200.benchmark import ring_size, time_ring_us

label = sys.argv[1] if len(sys.argv) > 1 else ""
what = sys.argv[2].split(",") if len(sys.argv) > 2 else ["kv", "norm"]
L, d, d_h, n = 8192, 512, 128, 16
K, N = d - d_h, n * d_h
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(5)
R = ring_size(2 * (L * d + 2 * K * N + 2 * L * N))
sets = [(torch.randn(L, d, device=dev, generator=g).half(),
         (torch.randn(K, N, device=dev, generator=g) / 8).half(),
         (torch.randn(K, N, device=dev, generator=g) / 8).half(),
         torch.empty(L, N, device=dev, dtype=torch.half),
         torch.empty(L, N, device=dev, dtype=torch.half)) for _ in range(R)]
out = []
if "kv" in what:
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, bd.Tag.FIRST), (s[2], d_h, n, bd.Tag.LAST)],
                                                  outs=[s[3], s[4]], check_finite=False) for s in sets]
    out.append(f"kv {time_ring_us(calls, 200):.2f}")
if "norm" in what:
    gam = torch.rand(d, device=dev, generator=g) + 0.5
    rk = torch.rand(d_h, device=dev, generator=g) + 0.5
    rv = torch.rand(d_h, device=dev, generator=g) + 0.5
    calls = [lambda s=s: bd.fused_rmsnorm_kv_proj_grouped(
        s[0], [(s[1], rk, d_h, n, bd.Tag.FIRST), (s[2], rv, d_h, n, bd.Tag.LAST)], 1e-6,
        outs=[s[3], s[4]], check_finite=False) for s in sets]
    out.append(f"norm {time_ring_us(calls, 200):.2f}")
print(label, " ".join(out), "us", flush=True)
