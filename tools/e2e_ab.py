"""Development aid: the end-to-end host path (fused_kv_proj_grouped_host, cfg2) with the
shipped row-block plan (equal blocks) vs a short first block (1/16 of L, so the first
copy-out starts earlier), interleaved in one process (wall clock per step, as bench.py's
e2e).  Measured: equal 1.35 ms, short-first 1.39 ms per step; equal blocks at chunks =
2 / 3 / 4 / 6: 1.40–1.42 / 1.38–1.41 / 1.37–1.39 / 1.40 ms (4, the default, is best).
Add ("short1st", short_first) to the plan list to repeat the first comparison."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2510_01718_b200 as bd  # noqa: E402
from paper_2510_01718_b200 import kv_proj as KP  # noqa: E402

dev = torch.device("cuda")
L, d, d_h, n = 8192, 512, 128, 16
ck = (torch.randn(384, 2048, device=dev) / 8).half()
cv = (torch.randn(384, 2048, device=dev) / 8).half()
xh = [torch.randn(L, d).half().pin_memory() for _ in range(2)]
kh = [torch.empty(L, 2048).half().pin_memory() for _ in range(2)]
vh = [torch.empty(L, 2048).half().pin_memory() for _ in range(2)]
specs = [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)]
shipped = KP._chunk_bounds


def short_first(L, chunks):
    if chunks == 1 or L <= 512:
        return [(0, L)]
    first = min(L, max(256, (L // 16) // 256 * 256))
    step = -(-(-(-(L - first) // (chunks - 1))) // 256) * 256
    return [(0, first)] + [(r, min(L, r + step)) for r in range(first, L, step)]


for rnd in range(3):
    for name, plan in (("shipped", shipped),):
        KP._chunk_bounds = plan
        for c in (2, 3, 4, 6):
            for i in range(3):
                bd.fused_kv_proj_grouped_host(xh[i % 2], specs, outs=[kh[i % 2], vh[i % 2]], chunks=c)
            torch.cuda.synchronize()
            t = time.perf_counter()
            for i in range(40):
                bd.fused_kv_proj_grouped_host(xh[i % 2], specs, outs=[kh[i % 2], vh[i % 2]], chunks=c)
            dt = (time.perf_counter() - t) / 40
            print(f"{name:8s} chunks {c}: {dt * 1e3:.3f} ms/step  {L / dt / 1e6:.2f} M tok/s", flush=True)
KP._chunk_bounds = shipped
