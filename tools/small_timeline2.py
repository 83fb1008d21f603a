"""Development aid: where a decode-sized launch's time goes, from the stamped small-L
kernel (tools/instrument_small.py -> xb/stl.so; run with BD_LIB_PATH=xb/stl.so).
Runs a CUDA graph of back-to-back launches on a cold-L2 ring (like the bench's decode
sweep), then prints, per launch of the last 8: entry spread, PDL release after the
previous launch's last CTA end, and the median per-CTA phase durations.

    python tools/small_timeline2.py SHAPE L     (SHAPE: cfg2 | paper)
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import _native
from paper_2510_01718_b200.benchmark import ring_size

import os
shape, L = sys.argv[1], int(sys.argv[2])
mode = os.environ.get("RING", "cold")  # cold | warm (R = 1) | warmx (x shared by every set)
n, nprob = (16, 2) if shape == "cfg2" else (128, 1)
d, d_h = 512, 128
K, N = d - d_h, n * d_h
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
dtype = torch.float16
R = ring_size(2 * (L * d + nprob * (K * N + L * N))) if mode != "warm" else 1
sets = [(torch.randn(L, d, device=dev, generator=g).to(dtype),
         [(torch.randn(K, N, device=dev, generator=g) / 8).to(dtype) for _ in range(nprob)],
         [torch.empty(L, N, device=dev, dtype=dtype) for _ in range(nprob)]) for _ in range(R)]
if mode == "warmx":
    sets = [(sets[0][0],) + s[1:] for s in sets]
tags = [bd.Tag.FIRST, bd.Tag.LAST][:nprob]
calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(c, d_h, n, t) for c, t in zip(s[1], tags)],
                                              outs=s[2], check_finite=False) for s in sets]
for f in calls:
    f()
torch.cuda.synchronize()
stream = torch.cuda.Stream()
graph = torch.cuda.CUDAGraph()
inner = max(R, 200)
with torch.cuda.graph(graph, stream=stream):
    for i in range(inner):
        calls[i % len(calls)]()
graph.replay()
torch.cuda.synchronize()
lib = _native.load()
lib.bd_debug_small_reset()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(stream):
    a.record(stream)
    graph.replay()
    b.record(stream)
torch.cuda.synchronize()
print(f"{shape} L={L} ring={mode}: {a.elapsed_time(b) * 1e3 / inner:.2f} us/launch (graph of {inner}, ring {R})")
buf = (ctypes.c_ulonglong * (8 * 512 * 8))()
lib.bd_debug_small_timeline(buf)
tl = np.frombuffer(buf, dtype=np.uint64).reshape(8, 512, 8).astype(np.float64)
tl[tl == 0] = np.nan  # stamps a CTA does not take (pair peers: no MMA issuer)
ncta = int((~np.isnan(tl[0, :, 0])).sum())
tl = tl[:, :ncta]
order = np.argsort(np.nanmin(tl[:, :, 0], axis=1))
tl = tl[order]
t0 = np.nanmin(tl[0, :, 0])
med = lambda v: int(np.nanmedian(v))
mn = lambda v: int(np.nanmin(v))
mx = lambda v: int(np.nanmax(v))
print(f"CTAs per launch: {ncta}")
print("launch | entry min..max | release(min,max) after prev last end | last end | "
      "median: prologue, wait->landed, landed->mma done, epilogue, end sync | CTA end spread")
prev_end = None
for j in range(8):
    e = tl[j] - t0
    rel = (mn(e[:, 2]) - prev_end, mx(e[:, 2]) - prev_end) if prev_end is not None else (0, 0)
    print(f"{j} | {mn(e[:, 0]):6d}..{mx(e[:, 0]):6d} | {rel[0]:5d},{rel[1]:5d} | {mx(e[:, 6]):6d} | "
          f"{med(e[:, 1] - e[:, 0]):5d} {med(e[:, 3] - e[:, 2]):5d} {med(e[:, 4] - e[:, 3]):5d} "
          f"{med(e[:, 5] - e[:, 4]):5d} {med(e[:, 6] - e[:, 5]):5d} | {mx(e[:, 6]) - mn(e[:, 6]):5d}")
    prev_end = mx(e[:, 6])
print("absolute (ns): launch | entry min/max | release min/max | first kb landed min/max | last kb min/max | "
      "epi done min/max | next release - last epi done")
for j in range(8):
    e = tl[j] - t0
    gap = mn(tl[j + 1, :, 2] - t0) - mx(e[:, 5]) if j < 7 else 0
    print(j, "|", " | ".join(f"{mn(e[:, k]):6d} {mx(e[:, k]):6d}" for k in (0, 2, 7, 3, 5)), "|", gap)
e = tl[4] - tl[4, :, 2:3]
print("launch 4, per-CTA (rel. to its PDL release) percentiles 0/50/100:")
for k, name in ((3, "last k-block landed"), (4, "MMA done"), (5, "epilogue done"), (6, "end")):
    print(f"  {name:20s}", np.nanpercentile(e[:, k], [0, 50, 100]).astype(int))
