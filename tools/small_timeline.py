"""Development aid: per-CTA stamps of the small-L kernel (exp/smalltl.so)."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import _native
L = int(sys.argv[1]); n = int(sys.argv[2]); single = len(sys.argv) > 3
d, d_h = 512, 128
dev = torch.device("cuda:0")
x = torch.randn(L, d, device=dev).half()
cs = [(torch.randn(d - d_h, n * d_h, device=dev) / 8).half() for _ in range(1 if single else 2)]
specs = [(c, d_h, n, t) for c, t in zip(cs, [bd.Tag.FIRST, bd.Tag.LAST])]
for _ in range(30):
    bd.fused_kv_proj_grouped(x, specs)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (148 * 64))()
_native.load().bd_debug_timeline(buf)
tl = np.frombuffer(buf, dtype=np.uint64).reshape(148, 64).astype(np.int64)
ncta = int((tl[:, 13] > 0).sum())
t = tl[:ncta]
rel = t - t[:, 1:2]
med = lambda a: int(np.median(a))
print(f"L={L} n={n} ctas={ncta} start spread ns {t[:,0].max()-t[:,0].min()} end spread {t[:,13].max()-t[:,0].min()}")
print("setup", med(rel[:, 2]), "pdl", med(rel[:, 3]), "kb ready", [med(rel[:, 4 + k]) for k in range(6)],
      "mma done", med(rel[:, 10]), "epi end", med(rel[:, 11]), "end", med(rel[:, 12]))
end_ns = t[:, 13] - t[:, 0].min()
print("CTA end ns percentiles 0/10/50/90/100:", np.percentile(end_ns, [0, 10, 50, 90, 100]).astype(int))
print("kb0 ready clk percentiles:", np.percentile(rel[:, 4], [0, 10, 50, 90, 100]).astype(int))
print("last kb ready clk percentiles:", np.percentile(rel[:, 9], [0, 10, 50, 90, 100]).astype(int))
print("epi end clk percentiles:", np.percentile(rel[:, 11], [0, 10, 50, 90, 100]).astype(int))
