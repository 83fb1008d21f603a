"""The reference's own numba kernel beside the C port (oracle/bd_oracle.c) on the same
host, same inputs: shows the port — the timed CPU baseline on the GPU box, where
/root/reference does not exist — is a fair stand-in for the reference's CPU path.

Build container only (imports bdattn from /root/reference without writing into it,
SURVEY App. C):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tools/ref_vs_port_cpu.py > profiles/r02_ref_vs_port_cpu.json

Workload: cfg2 (DSV2-Lite kv_b_proj) K'+V', FP32, on a token sample (the kernel is
independent 8-row blocks, linear in L), 1 thread and all threads, median of 5 after 2
warm-ups (ref bench.py:85-99 protocol).  Outputs are also compared bit for bit.
"""

from __future__ import annotations

import json
import os
import statistics
import sys
import time
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import bdattn as ref  # noqa: E402
from oracle import oracle as O  # noqa: E402


def med(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def main():
    L, d, d_h, n = int(os.environ.get("SAMPLE_L", "1024")), 512, 128, 16
    rng = O.Rng(2024)
    x = O.rand_gaussian(rng, L, d, np.float32)
    ck = (O.rand_gaussian(rng, d - d_h, n * d_h, np.float32) / 8).astype(np.float32)
    cv = (O.rand_gaussian(rng, d - d_h, n * d_h, np.float32) / 8).astype(np.float32)
    X, CK, CV = ref.Tensor2D(x), ref.Tensor2D(ck), ref.Tensor2D(cv)
    rows = []
    all_threads = O.default_threads()
    for threads in sorted({1, all_threads}):
        ref.set_thread_count(threads)

        def run_ref():
            ref.fused_kv_proj(X, CK, d_h, n, ref.Tag.FIRST)
            ref.fused_kv_proj(X, CV, d_h, n, ref.Tag.LAST)

        def run_port():
            O.fused_kv_proj_ref(x, ck, d_h, n, "first", threads=threads)
            O.fused_kv_proj_ref(x, cv, d_h, n, "last", threads=threads)

        t_ref, t_port = med(run_ref), med(run_port)
        rows.append({"threads": threads, "ref_numba_ms": t_ref * 1e3, "port_c_ms": t_port * 1e3,
                     "ref_tokens_per_s": L / t_ref, "port_tokens_per_s": L / t_port,
                     "port_over_ref_speed": t_ref / t_port})
    same_k = np.array_equal(ref.fused_kv_proj(X, CK, d_h, n, ref.Tag.FIRST).data,
                            O.fused_kv_proj_ref(x, ck, d_h, n, "first", threads=all_threads))
    same_v = np.array_equal(ref.fused_kv_proj(X, CV, d_h, n, ref.Tag.LAST).data,
                            O.fused_kv_proj_ref(x, cv, d_h, n, "last", threads=all_threads))
    model = next((ln.split(":", 1)[1].strip() for ln in Path("/proc/cpuinfo").read_text().splitlines()
                  if ln.startswith("model name")), None)
    print(json.dumps({
        "workload": f"cfg2 K'+V' FP32, {L}-token sample (d=512, d_h=128, 16+16 heads)",
        "host": {"model": model, "cpu_count": os.cpu_count(), "affinity": all_threads},
        "numba": __import__("numba").__version__, "rows": rows,
        "outputs_bit_identical": bool(same_k and same_v)}, indent=1))


if __name__ == "__main__":
    main()
