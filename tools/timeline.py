"""Development aid: per-CTA timeline of one cfg2 K'+V' launch from the instrumented build
(tools/instrument.py -> exp/tl.so; run with BD_LIB_PATH=exp/tl.so).  Prints medians over
the pairs with a full tile count of: prologue stamps, each tile's MMA window (post
tempty-wait .. last MMA issued), the epilogue window (tfull .. done), B-wait clocks.
SM clocks relative to each CTA's entry.  Not a bench."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import _native

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
back_to_back = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16
single = len(sys.argv) > 4 and sys.argv[4] == "single"
d, d_h = 512, 128
dev = torch.device("cuda:0")
x = torch.randn(L, d, device=dev).half()
ck = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
cv = (torch.randn(d - d_h, n * d_h, device=dev) / 8).half()
k = torch.empty(L, n * d_h, device=dev, dtype=torch.half)
v = torch.empty_like(k)
specs = [(ck, d_h, n, bd.Tag.FIRST)] + ([] if single else [(cv, d_h, n, bd.Tag.LAST)])
for _ in range(10):
    bd.fused_kv_proj_grouped(x, specs, outs=[k, v][:len(specs)])
torch.cuda.synchronize()
for _ in range(back_to_back):
    bd.fused_kv_proj_grouped(x, specs, outs=[k, v][:len(specs)])
torch.cuda.synchronize()
lib = _native.load()
buf = (ctypes.c_ulonglong * (148 * 96))()
assert lib.bd_debug_timeline(buf) == 0
tl = np.frombuffer(buf, dtype=np.uint64).reshape(148, 96).astype(np.int64)
g0 = tl[:, 0].min()
print(f"L={L} back_to_back={back_to_back}")
print(f"CTA start spread (ns): 0 .. {tl[:, 0].max() - g0}; end (ns): "
      f"{tl[::2, 41].min() - g0} .. {tl[::2, 41].max() - g0}")
lead = np.arange(0, 148, 2)
nt = tl[lead, 42]
full = lead[nt == np.bincount(nt).argmax()]
rel = tl[full] - tl[full, 1:2]
med = lambda a: np.median(a, axis=0).astype(int)
print("tiles per pair:", np.bincount(nt))
print("prologue (prefetch, mbar-init, tmem-alloc, cluster-sync, pdl, first-TMA):",
      med(rel[:, 2:8]))
T = int(np.bincount(nt).argmax())
print("producer: first decode done, first a_empty passed:", med(rel[:, 43:45]))
print("mma window start:", med(rel[:, 8:8 + T]))
print("mma issued      :", med(rel[:, 16:16 + T]))
print("epi start (tfull):", med(rel[:, 24:24 + T]))
print("epi end         :", med(rel[:, 32:32 + T]))
print("b_full wait clks:", med(tl[full, 48:48 + T]))
print("end (clk):", int(np.median(rel[:, 40])), " ns per clk ~",
      float(np.median((tl[full, 41] - tl[full, 0]) / (tl[full, 40] - tl[full, 1]))))
endns = tl[full, 41] - g0
print("7-tile pair end (ns) percentiles 0/25/50/75/100:", np.percentile(endns, [0, 25, 50, 75, 100]).astype(int))
first_mma = rel[:, 8]
print("first MMA window start (clk) percentiles:", np.percentile(first_mma, [0, 25, 50, 75, 100]).astype(int))
per_tile = (rel[:, 32 + T - 1] - rel[:, 32]) / (T - 1)
print("epi-end period per tile (clk) percentiles:", np.percentile(per_tile, [0, 25, 50, 75, 100]).astype(int))
order = np.argsort(endns)[-5:]
print("slowest pairs (cta, end ns, first mma clk, period):",
      [(int(full[i]), int(endns[i]), int(first_mma[i]), int(per_tile[i])) for i in order])

if tl.shape[1] > 64 and (tl[full, 64] > 0).any():
    for base, name in ((64, "warp 2 (SMSP2)"), (80, "warp 4 (SMSP0, shared with the producer)")):
        e = tl[full, base:base + 13]
        rel_e = e - e[:, 11:12]  # relative to 'before tfull wait'
        m = np.median(rel_e, axis=0).astype(int)
        print(f"epilogue tile 3, {name}: tfull-wait-done {m[12]}, first-ld {m[1]} |",
              "after chunk c: ", [m[2], m[4], m[6], m[8]], "| loads ready c=1..3:", [m[3], m[5], m[7]],
              "| loop end", m[9], "| barrier done", m[10])

# straddling: does the pair's contiguous tile range cross a (problem, row-block) boundary
# (16 tiles per row-block per problem at cfg2) — i.e. load A twice?
if not single and L == 8192 and n == 16:
    units = 74
    tot = 512
    lead_all = np.arange(0, 148, 2)
    ends = tl[lead_all, 41] - g0
    rows = []
    for u in range(units):
        tb, te = u * tot // units, (u + 1) * tot // units
        rows.append((te - tb, int(tb // 16 != (te - 1) // 16), int(ends[u])))
    arr = np.array(rows)
    for nt in (6, 7):
        for st in (0, 1):
            sel = (arr[:, 0] == nt) & (arr[:, 1] == st)
            if sel.any():
                print(f"tiles={nt} straddle={st}: pairs {sel.sum():2d}, end ns median "
                      f"{int(np.median(arr[sel, 2]))}, max {int(arr[sel, 2].max())}")
