"""Decode-sized L: our launch (whatever the library routes to; BD_DECODE=0 selects the
older small-L / persistent kernels) vs cuBLAS, FP16/BF16, the paper's n = 128 shape and
cfg2's 16 + 16 heads, on cold-L2 rings, CUDA-graph timed.  Prints one line per point.

    python tools/decode_ab.py [L ...]
"""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2510_01718_b200 as bd  # noqa: E402
from paper_2510_01718_b200.benchmark import ring_size, time_ring_us  # noqa: E402


def point(dtype, n, nprob, L, dev, g):
    d, d_h = 512, 128
    K, N = d - d_h, n * d_h
    R = ring_size(2 * (L * d + nprob * (K * N + L * N)))
    sets = [(torch.randn(L, d, device=dev, generator=g).to(dtype),
             [(torch.randn(K, N, device=dev, generator=g) / 8).to(dtype) for _ in range(nprob)],
             [torch.empty(L, N, device=dev, dtype=dtype) for _ in range(nprob)]) for _ in range(R)]
    tags = [bd.Tag.FIRST, bd.Tag.LAST][:nprob]
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(c, d_h, n, t) for c, t in zip(s[1], tags)],
                                                  outs=s[2], check_finite=False) for s in sets]
    inner = max(R, 400)
    import os
    if os.environ.get("ISO"):
        us = iso_us(calls[0], dev)
        ds = [(sets[0][0], (torch.randn(d, nprob * N, device=dev, generator=g) / 8).to(dtype),
               torch.empty(L, nprob * N, device=dev, dtype=dtype))]
        dus = iso_us(lambda: torch.matmul(ds[0][0], ds[0][1], out=ds[0][2]), dev)
        return us, dus, 2 * (L * d + nprob * (K * N + L * N)) / (us * 1e-6) / 1e9
    us = time_ring_us(calls, inner)
    ds = [(s[0], (torch.randn(d, nprob * N, device=dev, generator=g) / 8).to(dtype),
           torch.empty(L, nprob * N, device=dev, dtype=dtype)) for s in sets]
    dus = time_ring_us([lambda s=s: torch.matmul(s[0], s[1], out=s[2]) for s in ds], inner)
    nbytes = 2 * (L * d + nprob * (K * N + L * N))
    return us, dus, nbytes / (us * 1e-6) / 1e9


def iso_us(fn, dev, reps=15):
    """Isolated launch latency: L2 flushed (256 MB written) before each call, the call
    bracketed by CUDA events on the current stream; median of reps."""
    import statistics
    flush = torch.empty(256 * 2 ** 20 // 4, device=dev)
    ts = []
    for _ in range(reps + 2):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts[2:])


def main():
    Ls = [int(a) for a in sys.argv[1:]] or [1, 16, 64, 128, 256]
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    import os
    dts = [torch.float16, torch.bfloat16][:int(os.environ.get("NDT", "2"))]
    for name, n, nprob in (("paper", 128, 1), ("cfg2", 16, 2)):
        for dtype in dts:
            for L in Ls:
                us, dus, gbs = point(dtype, n, nprob, L, dev, g)
                print(f"{name:5s} {str(dtype)[6:]:8s} L={L:4d}  ours {us:6.2f} us  cublas {dus:6.2f} us"
                      f"  x{dus / us:5.3f}  {gbs:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
