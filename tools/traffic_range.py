"""DRAM traffic per launch of the benched cfg2 kernel, over a multi-launch range on the
bench's cold-L2 ring (the `roofline.traffic` evidence).

A single-launch ncu capture undercounts writes: most of the 67 MB of K'/V' is still
dirty in the 126 MB L2 when the kernel ends and is written back during LATER kernels.
Over a range of R launches cycling through the bench's ring, steady-state write-backs
(the previous launches' outputs evicted by this one) replace them, so the range total
divided by R is the per-launch traffic of the steady state the bench times.

    ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,\
gpu__time_duration.sum --csv --log-file gpurun_out/traffic.csv \
        python tools/traffic_range.py [--impl bd|dense] [--launches 40]
"""

from __future__ import annotations

import argparse
import math
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2510_01718_b200 as bd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["bd", "dense"], default="bd")
    ap.add_argument("--launches", type=int, default=40)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    L, d, d_h, n = 8192, 512, 128, 16
    K, N = d - d_h, n * d_h
    set_bytes = 2 * (L * d + 2 * K * N + 2 * L * N)
    R = max(2, math.ceil(2 * 126 * 2 ** 20 / set_bytes) + 1)  # same ring as bench.py
    g = torch.Generator(device=dev).manual_seed(1234)
    xs = [torch.randn(L, d, device=dev, generator=g).half() for _ in range(R)]
    if a.impl == "bd":
        cks = [(torch.randn(K, N, device=dev, generator=g) / 8).half() for _ in range(R)]
        cvs = [(torch.randn(K, N, device=dev, generator=g) / 8).half() for _ in range(R)]
        kos = [torch.empty(L, N, device=dev, dtype=torch.half) for _ in range(R)]
        vos = [torch.empty(L, N, device=dev, dtype=torch.half) for _ in range(R)]

        def step(j):
            bd.fused_kv_proj_grouped(xs[j], [(cks[j], d_h, n, bd.Tag.FIRST),
                                             (cvs[j], d_h, n, bd.Tag.LAST)],
                                     outs=[kos[j], vos[j]], check_finite=False)
    else:
        ws = [(torch.randn(d, 2 * N, device=dev, generator=g) / 8).half() for _ in range(R)]
        dos = [torch.empty(L, 2 * N, device=dev, dtype=torch.half) for _ in range(R)]

        def step(j):
            torch.matmul(xs[j], ws[j], out=dos[j])
    for i in range(2 * R):  # reach the steady state of the ring
        step(i % R)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for i in range(a.launches):
        step(i % R)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"{a.impl}: {a.launches} launches over a ring of {R} sets "
          f"({R * set_bytes / 2 ** 20:.0f} MiB)")


if __name__ == "__main__":
    main()
