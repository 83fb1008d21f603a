"""Development aid: per-tile timeline of the MLA attention kernel's first work item on CTA 0
(a stamped build from tools/instrument_attn.py; run with
BD_LIB_PATH=xb/attnstamp.so).   python tools/attn_timeline.py [L]"""
import ctypes
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2510_01718_b200 import _native
from paper_2510_01718_b200 import mla as M

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H = 16
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q = torch.randn(L, H, 192, device=dev, generator=g).half()
k = torch.randn(H, L, 128, device=dev, generator=g).half()
kpe = torch.randn(L, 64, device=dev, generator=g).half()
v = torch.randn(H, L, 128, device=dev, generator=g).half()
out = torch.empty(L, H, 128, device=dev, dtype=torch.half)
for _ in range(3):
    M.mla_attention(q, k, kpe, v, scale=1 / math.sqrt(192), out=out)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (6 * 64))()
_native.load().bd_debug_attn_timeline(buf)
t = np.frombuffer(buf, dtype=np.int64).reshape(6, 64).astype(np.int64)
t0 = t[:, 0].min()
r = t - t0
print("j | K issued | V issued | S_j issued (MMA) | softmax saw S_j | P_j published | MMA saw P_j")
for j in range(0, 64, 4):
    print(f"{j:2d} | " + " | ".join(f"{r[k_, j]:7d}" for k_ in (0, 1, 3, 4, 5, 2)))
per = np.diff(t[5, 8:60]).mean()
print(f"P period (clk, tiles 8..60): {per:.0f};  softmax busy (S seen -> P published): "
      f"{(t[5, 8:60] - t[4, 8:60]).mean():.0f};  S issued -> softmax saw it: {(t[4, 8:60] - t[3, 8:60]).mean():.0f};"
      f"  P published -> MMA saw P: {(t[2, 8:60] - t[5, 8:60]).mean():.0f};  K issue -> S issue: {(t[3, 8:60] - t[0, 8:60]).mean():.0f}")
