"""Development aid: paper k_proj shape (n=128, d=512, d_h=128, FP16) at small L through the
reference's benchmark harness (CUDA graph, median) — ours vs cuBLAS.  Not a bench."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2510_01718_b200 import benchmark as B

label = sys.argv[1] if len(sys.argv) > 1 else ""
seq = tuple(int(v) for v in sys.argv[2].split(",")) if len(sys.argv) > 2 else (64, 128, 256, 512, 1024)
recs = B.kv_proj_benchmark(512, 128, 128, seq, dtype=torch.float16, inner=10)
for r in recs:
    if r.operator == B.FUSED_OPERATOR:
        print(f"{label} L={r.seq_len}: {r.median_ns / 1e3:.2f} us  speedup {r.speedup_vs_baseline:.3f}")
