"""Development aid: how much of a cfg2 step is outside the kernel's CTA lifetime?

Run with BD_LIB_PATH=exp/tl.so (tools/instrument.py build).  A CUDA graph replays
`inner` K'+V' launches over a ring of R buffer sets (R=1 warm, R=5 cold); the per-launch
time from CUDA events is compared with the last launch's span from its CTA stamps
(first CTA entry .. last CTA's final store drained, globaltimer ns)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import _native

L, d, d_h, n = 8192, 512, 128, 16
dev = torch.device("cuda:0")
lib = _native.load()
for R in (1, 5):
    sets = [(torch.randn(L, d, device=dev).half(), (torch.randn(d - d_h, n * d_h, device=dev) / 8).half(),
             (torch.randn(d - d_h, n * d_h, device=dev) / 8).half(),
             torch.empty(L, n * d_h, device=dev, dtype=torch.half),
             torch.empty(L, n * d_h, device=dev, dtype=torch.half)) for _ in range(R)]
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, bd.Tag.FIRST), (s[2], d_h, n, bd.Tag.LAST)],
                                                  outs=[s[3], s[4]], check_finite=False) for s in sets]
    for f in calls * 3:
        f()
    torch.cuda.synchronize()
    inner = 40
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(inner):
            calls[i % R]()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    spans = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            g.replay()
            b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / inner)
        buf = (ctypes.c_ulonglong * (148 * 96))()
        lib.bd_debug_timeline(buf)
        tl = np.frombuffer(buf, dtype=np.uint64).reshape(148, 96).astype(np.int64)
        spans.append((tl[:, 41].max() - tl[:, 0].min()) / 1e3)
        rel = tl[:, 45].min()
        last = (tl, rel)
    print(f"R={R}: per-launch {np.median(ts):.2f} us (graph of {inner}), last launch CTA span "
          f"{np.median(spans):.2f} us -> outside the span {np.median(ts) - np.median(spans):.2f} us")
    tl, rel = last
    lead = np.arange(0, 148, 2)
    print("  PDL release spread (ns):", int(tl[:, 45].max() - rel),
          " CTA entry before release (ns) p0/50/100:", np.percentile(rel - tl[:, 0], [0, 50, 100]).astype(int))
    print("  pair end after release (ns) p0/10/50/90/100:",
          np.percentile(tl[lead, 41] - rel, [0, 10, 50, 90, 100]).astype(int))
    print("  first TMA after release (clk) p50/100:",
          np.percentile(tl[lead, 7] - tl[lead, 6], [50, 100]).astype(int))
