"""Measure every BASELINE.json config beside the bench's headline (cfg2) on one B200,
plus the paper's Table 4/5 k_proj sweep, and write the results under profiles/.

    python tools/sweep_configs.py [--out profiles/r01] [--quick]

cfg1  reference CPU test shape (d=512, 8 heads, d_h=64, 256 tokens), FP32 exact kernel,
      K'+V' in one launch
cfg3  Llama-2-7B K/V (d=4096, 32 x 128), BF16, 65536 tokens: BD K'+V' (tags FIRST/LAST,
      one launch, K = 3968 streams) vs cuBLAS X @ [W_k | W_v] (4096 x 8192)
cfg4  BD low-rank linear 4096 -> 1024 -> 4096, FP16, 32768 tokens vs the two-GEMM low-rank
      layer (cuBLAS) and the dense 4096 x 4096 layer (cuBLAS)
paper n=128, d=512, d_h=128, FP16 and BF16, L = 64 ... 65536, the
      reference's CSV schema (paper_2510_01718_b200.benchmark)
All timings: CUDA graphs of back-to-back calls, CUDA events, median of 5.  Inputs are
random (timing depends on shapes only, like the reference's bench, bench.py:113-116).
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import benchmark as B


def tf(flops, ns):
    return flops / (ns * 1e-9) / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r01")
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    peak = B.measured_peak_tflops()
    g = torch.Generator(device=dev).manual_seed(0)
    res = {"peak_tflops": peak}

    # ---- cfg1: FP32 exact path (reference CPU test shape)
    x = torch.randn(256, 512, device=dev, generator=g)
    ck = torch.randn(448, 512, device=dev, generator=g) / 8
    cv = torch.randn(448, 512, device=dev, generator=g) / 8
    ns = B.time_operator_ns(lambda: bd.fused_kv_proj_grouped(
        x, [(ck, 64, 8, bd.Tag.FIRST), (cv, 64, 8, bd.Tag.LAST)]))
    res["cfg1_fp32_exact"] = {"tokens": 256, "us": ns / 1e3, "tokens_per_s": 256 / (ns * 1e-9),
                              "gflops": tf(2 * 2 * 256 * 448 * 512, ns) * 1e3}

    # ---- cfg3: Llama-2-7B K/V, BF16, 65536 tokens
    L, d, d_h, n = (16384 if args.quick else 65536), 4096, 128, 32
    x = torch.randn(L, d, device=dev, generator=g).to(torch.bfloat16)
    ck = (torch.randn(d - d_h, n * d_h, device=dev, generator=g) / 64).to(torch.bfloat16)
    cv = (torch.randn(d - d_h, n * d_h, device=dev, generator=g) / 64).to(torch.bfloat16)
    w = (torch.randn(d, 2 * n * d_h, device=dev, generator=g) / 64).to(torch.bfloat16)
    ko = torch.empty(L, n * d_h, device=dev, dtype=torch.bfloat16)
    vo = torch.empty_like(ko)
    do = torch.empty(L, 2 * n * d_h, device=dev, dtype=torch.bfloat16)
    bd_ns = B.time_operator_ns(lambda: bd.fused_kv_proj_grouped(
        x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)], outs=[ko, vo]), inner=3)
    dn_ns = B.time_operator_ns(lambda: torch.matmul(x, w, out=do), inner=3)
    fl = 2 * 2 * L * (d - d_h) * n * d_h
    res["cfg3_llama2_7b_kv_bf16"] = {
        "tokens": L, "bd_us": bd_ns / 1e3, "dense_cublas_us": dn_ns / 1e3,
        "bd_tokens_per_s": L / (bd_ns * 1e-9), "speedup_vs_dense": dn_ns / bd_ns,
        "flop_ratio": d / (d - d_h), "bd_tflops": tf(fl, bd_ns), "bd_roofline_frac": tf(fl, bd_ns) / peak,
        "dense_tflops": tf(2 * L * d * 2 * n * d_h, dn_ns)}
    del x, ck, cv, w, ko, vo, do

    # ---- cfg4: BD low-rank linear, FP16, 32768 tokens
    L, din, r, dout = (8192 if args.quick else 32768), 4096, 1024, 4096
    u = torch.randn(din, r, device=dev, generator=g) / 32
    v = torch.randn(dout, r, device=dev, generator=g) / 32
    basis = (torch.randn(din, r, device=dev, generator=g) / 32).half()
    coeff = (torch.randn(r, dout - r, device=dev, generator=g) / 32).half()
    fac = bd.BDFactors(axis=bd.Axis.COLUMN, tag=bd.Tag.FIRST, basis=basis.cpu().numpy(),
                       coeff=coeff.cpu().numpy(), orig_rows=din, orig_cols=dout, rank=r,
                       residual=0.0, rank_deficient=False)
    layer = bd.BDLinearLayer(fac, basis, coeff)
    x = torch.randn(L, din, device=dev, generator=g).half()
    y = torch.empty(L, dout, device=dev, dtype=torch.float16)
    uh, vth = u.half(), v.t().contiguous().half()
    h = torch.empty(L, r, device=dev, dtype=torch.float16)
    yl = torch.empty(L, dout, device=dev, dtype=torch.float16)
    wd = (torch.randn(din, dout, device=dev, generator=g) / 64).half()
    yd = torch.empty(L, dout, device=dev, dtype=torch.float16)

    def lowrank():
        torch.matmul(x, uh, out=h)
        torch.matmul(h, vth, out=yl)

    bd_ns = B.time_operator_ns(lambda: bd.bd_linear_forward(x, layer, out=y), inner=3)
    lr_ns = B.time_operator_ns(lowrank, inner=3)
    dn_ns = B.time_operator_ns(lambda: torch.matmul(x, wd, out=yd), inner=3)
    fl_bd = 2 * L * din * r + 2 * L * r * (dout - r)
    res["cfg4_lowrank_bd_linear_fp16"] = {
        "tokens": L, "bd_us": bd_ns / 1e3, "lowrank_cublas_us": lr_ns / 1e3,
        "dense_cublas_us": dn_ns / 1e3, "bd_tokens_per_s": L / (bd_ns * 1e-9),
        "speedup_vs_lowrank": lr_ns / bd_ns, "speedup_vs_dense": dn_ns / bd_ns,
        "bd_tflops": tf(fl_bd, bd_ns), "bd_roofline_frac": tf(fl_bd, bd_ns) / peak,
        "flop_ratio_vs_lowrank": (2 * L * din * r + 2 * L * r * dout) / fl_bd}
    del x, y, h, yl, wd, yd

    # ---- paper Table 4 / 5 sweep (n=128, d=512, d_h=128)
    seq = B.DEFAULT_SEQ_LENS if not args.quick else (64, 1024, 8192)
    for dt, name in ((torch.float16, "fp16"), (torch.bfloat16, "bf16")):
        recs = B.kv_proj_benchmark(512, 128, 128, seq, dtype=dt, inner=10)
        B.write_csv(f"{args.out}_paper_kproj_{name}.csv", recs)
        fused = [r_ for r_ in recs if r_.operator == B.FUSED_OPERATOR]
        res[f"paper_kproj_{name}"] = {str(r_.seq_len): {"Mtok_s": r_.tokens_per_sec / 1e6,
                                                         "speedup": r_.speedup_vs_baseline,
                                                         "roofline_frac": r_.roofline_frac}
                                      for r_ in fused}
    Path(f"{args.out}_configs.json").write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
