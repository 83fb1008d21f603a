"""Development aid: does NVML polling (the bench's clock sampler) perturb short launches?
Times the paper k_proj shape at L = 64 / 128 (graph ring, as tools/time_short.py) with no
sampler and with a sampler thread polling every 2 ms and every 20 ms."""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2510_01718_b200 as bd  # noqa: E402
from paper_2510_01718_b200.benchmark import ring_size, time_ring_us  # noqa: E402
import pynvml  # noqa: E402

dev = torch.device("cuda:0")
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def poll(stop, period):
    while not stop.is_set():
        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        time.sleep(period)


def run(L, inner):
    d, d_h, n = 512, 128, 128
    K, N = d - d_h, n * d_h
    R = ring_size(2 * (L * d + K * N + L * N))
    sets = [(torch.randn(L, d, device=dev).half(), (torch.randn(K, N, device=dev) / 8).half(),
             torch.empty(L, N, device=dev, dtype=torch.half)) for _ in range(R)]
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, bd.Tag.FIRST)], outs=[s[2]],
                                                  check_finite=False) for s in sets]
    return time_ring_us(calls, inner, reps=11)


for mode in ("none", "2ms", "20ms", "none"):
    stop = threading.Event()
    t = None
    if mode != "none":
        t = threading.Thread(target=poll, args=(stop, 0.002 if mode == "2ms" else 0.02), daemon=True)
        t.start()
    res = [f"L={L} inner={inner}: {run(L, inner):.2f}" for L in (64, 128) for inner in (613, 2000)]
    stop.set()
    if t:
        t.join()
    print(f"{mode:5s}", " | ".join(res), flush=True)
