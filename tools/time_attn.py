"""cfg5 attention core and block timing: the tcgen05 MLA attention kernel vs torch SDPA
(cuDNN) on the same inputs; then the BD MLA block with each attention (and head groups).
    python tools/time_attn.py [L] [H]
"""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_01718_b200 import mla as M  # noqa: E402
from paper_2510_01718_b200.benchmark import time_ring_us  # noqa: E402
from torch.nn.attention import sdpa_kernel  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn(L, H, 192, device=dev, generator=g).half()
    k = torch.randn(H, L, 128, device=dev, generator=g).half()
    kpe = torch.randn(L, 64, device=dev, generator=g).half()
    v = torch.randn(H, L, 128, device=dev, generator=g).half()
    out = torch.empty(L, H, 128, device=dev, dtype=torch.half)
    scale = 1 / math.sqrt(192)
    flops = H * (L * (L + 128) / 2) * 2 * (192 + 128)
    us = time_ring_us([lambda: M.mla_attention(q, k, kpe, v, scale=scale, out=out)], 5)
    kk = torch.cat([k, kpe[None].expand(H, L, 64)], -1)
    qt = q.transpose(0, 1)[None]

    def sd():
        with sdpa_kernel(M._BACKENDS):
            torch.nn.functional.scaled_dot_product_attention(qt, kk[None], v[None], is_causal=True,
                                                             scale=scale)
    sus = time_ring_us([sd], 5)
    print(f"attention L={L} H={H}: ours {us:.1f} us ({flops / us / 1e6:.0f} TFLOP/s), "
          f"SDPA {sus:.1f} us ({flops / sus / 1e6:.0f} TFLOP/s)", flush=True)
    if L < 8192:
        return
    w = M.gen_random_mla(1234)
    p = M.mla_prepare(w).to(dev, torch.float16)
    wd = w.to(dev, torch.float16)
    hid = torch.randn(L, 2048, device=dev, generator=g).half()
    for name, fn in (("dense sdpa", lambda: M.mla_forward(hid, wd)),
                     ("bd sdpa", lambda: M.bd_mla_forward(hid, p)),
                     ("bd bd-attn", lambda: M.bd_mla_forward(hid, p, attention="bd")),
                     ("bd bd-attn G=2", lambda: M.bd_mla_forward(hid, p, attention="bd", head_group=2)),
                     ("bd bd-attn G=4", lambda: M.bd_mla_forward(hid, p, attention="bd", head_group=4))):
        t = time_ring_us([fn], 3)
        print(f"block {name:16s} {t / 1e3:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
