"""Per-CTA %globaltimer timeline of the decode kernel (kv_proj_decode.cu, BD_DC_STAMPS
build) in its steady state: a CUDA graph of back-to-back launches over a cold ring,
then the stamps of the last launches, relative to the previous launch's last CTA exit.

    nvcc ... -DBD_DC_STAMPS -o xb/dc_stamps.so csrc/*.cu      (tools/build_variant.sh)
    BD_LIB_PATH=xb/dc_stamps.so python tools/decode_timeline.py [paper|cfg2] L
Events: 0 entry, 1 init done, 2 producer past griddep_wait, 3 first k-block landed,
4 last MMA issued, 5 epilogue saw MMAs done, 6 stores drained, 7 exit.
"""

import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2510_01718_b200 as bd  # noqa: E402
from paper_2510_01718_b200 import _native as N  # noqa: E402
from paper_2510_01718_b200.benchmark import ring_size  # noqa: E402


def main():
    shape = sys.argv[1] if len(sys.argv) > 1 else "paper"
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    d, d_h = 512, 128
    n, nprob = (128, 1) if shape == "paper" else (16, 2)
    dev = torch.device("cuda", 0)
    K, Nc = d - d_h, n * d_h
    R = ring_size(2 * (L * d + nprob * (K * Nc + L * Nc)))
    g = torch.Generator(device=dev).manual_seed(0)
    sets = [(torch.randn(L, d, device=dev, generator=g).half(),
             [(torch.randn(K, Nc, device=dev, generator=g) / 8).half() for _ in range(nprob)],
             [torch.empty(L, Nc, device=dev, dtype=torch.half) for _ in range(nprob)])
            for _ in range(R)]
    tags = [bd.Tag.FIRST, bd.Tag.LAST][:nprob]

    def call(s):
        bd.fused_kv_proj_grouped(s[0], [(c, d_h, n, t) for c, t in zip(s[1], tags)], outs=s[2],
                                 check_finite=False)
    for s in sets:
        call(s)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    inner = max(R, 40)
    with torch.cuda.graph(graph, stream=stream):
        for i in range(inner):
            call(sets[i % R])
    graph.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(stream)
        graph.replay()
        b.record(stream)
    torch.cuda.synchronize()
    print(f"{shape} L={L}: {a.elapsed_time(b) * 1e3 / inner:.2f} us/launch (graph of {inner})")
    lib = N.load()
    buf = np.zeros((4, 512, 16), dtype=np.uint64)
    lib.bd_debug_decode_stamps.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    rc = lib.bd_debug_decode_stamps(buf.ctypes.data, buf.nbytes)
    assert rc == 0, rc
    # launches were numbered by the host: the last `inner` launches; find the 4 slots'
    # order by their entry times
    used = [(int(buf[s, :, 0][buf[s, :, 0] > 0].min()), s) for s in range(4)]
    used.sort()
    grid = int((buf[used[-1][1], :, 0] > 0).sum())
    print(f"grid {grid} CTAs")
    prev_end = None
    for _, s in used:
        st = buf[s, :grid].astype(np.int64)
        base = prev_end if prev_end is not None else int(st[:, 0].min())
        rel = (st - base) / 1e3
        names = ["entry", "init", "wait", "kb0", "mma", "done", "drain", "exit"]
        line = "  ".join(f"{nm} {np.min(rel[:, k]):6.2f}/{np.median(rel[:, k]):6.2f}/{np.max(rel[:, k]):6.2f}"
                         for k, nm in enumerate(names))
        print(f"slot {s}: (us rel. to prev launch's last exit; min/med/max)  {line}")
        kbs = [k for k in range(8, 16) if (st[:, k] > 0).all() and (st[:, k] >= st[:, 0]).all()]
        print("    k-block landed (median us): " +
              " ".join(f"kb{k - 8} {np.median(rel[:, k]):.2f}" for k in kbs))
        prev_end = int(st[:, 7].max())


if __name__ == "__main__":
    main()
