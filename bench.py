#!/usr/bin/env python
"""Benchmark of the BD K/V projection (BASELINE.json metric) — one JSON line on rank 0.

Workload (BASELINE config 2): DeepSeek-V2-Lite MLA kv_b_proj, kv_lora_rank d = 512,
16 heads x (128 K_nope + 128 V), d_h = 128, FP16, 8192 tokens per GPU, random-init
weights.  One step = the BD projection of K' AND V' (two problems, different tags, one
kernel launch) for the step's tokens:

    K' = X[:, S_k] + X[:, ~S_k] C_k,   V' = X[:, S_v] + X[:, ~S_v] C_v

Arms
  default            our kernel (libbd_kvproj.so via the package API), device-resident
                     inputs -> `value`; the same call with pinned HOST buffers and the
                     H2D/D2H copies inside the timed region -> `e2e`; cuBLAS dense
                     projection with the original 512 x 4096 weight -> `baselines`.
  --impl reference   the reference's CPU algorithm (the C oracle restatement; the
                     reference is Python+numba and cannot travel to the GPU box) on all
                     host threads, rank 0 only.

Multi-GPU (torchrun): head-sharded weak scaling — rank r owns heads [r n/g, (r+1) n/g) of
C_k and C_v and projects g x 8192 tokens, so per-GPU work is fixed and no collective sits
on the data path; the step time is the max over ranks.

L2 hygiene: the timed loop cycles through a ring of R buffer sets (x, C_k, C_v, K', V')
whose total exceeds 2x the 126 MB L2, so no step finds its inputs in L2 from the
previous use of the same buffers.
"""

from __future__ import annotations

import argparse
import contextlib
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "BD K/V-proj tokens/s & speedup vs dense cuBLAS proj (DSV2-Lite FP16), 1-8 GPU"
L2_BYTES = 126 * 2 ** 20

CFG2 = dict(L=8192, d=512, d_h=128, n_heads=16)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dtype", choices=["fp16", "bf16"], default="fp16")
    ap.add_argument("--tokens", type=int, default=CFG2["L"], help="tokens per GPU per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-block", action="store_true",
                    help="skip the DeepSeek-V2-Lite BDA block measurement (config 5)")
    ap.add_argument("--block-tokens", type=int, default=32768)
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other BASELINE configs and the paper sweep (N=1 only)")
    ap.add_argument("--gather", choices=["both", "none", "nccl", "fused"], default="both",
                    help="time the head all-gather paths (SURVEY 8(e)) after the projection")
    return ap.parse_args()


@contextlib.contextmanager
def stdout_to_stderr():
    """Point fd 1 at stderr for the duration: NCCL may print its banner on stdout at
    init, and the driver reads exactly ONE JSON line there."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        yield
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["bf16_tflops"], d["hbm_gbs"], "measured"
    return 1590.0, 6650.0, "fallback"  # B200_PROFILING.md fallback figures


def load_sustained_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["bf16_tflops_sustained"])
    except Exception:
        return 1400.0  # B200_PROFILING.md: sustained ~1.4 PFLOP/s under the power cap


def kernel_source_sha16() -> str:
    import hashlib
    src = ROOT / "paper_2510_01718_b200" / "csrc" / "kv_proj_tc.cu"
    return hashlib.sha256(src.read_bytes()).hexdigest()[:16]


def load_traffic():
    """DRAM bytes per launch of the dominant kernel: ncu over a 40-launch range on the
    bench's cold ring (tools/traffic_range.py, profiles/traffic_cfg2.json) — only if it
    was measured on THIS kernel source (sha256 of kv_proj_tc.cu), else None."""
    p = ROOT / "profiles" / "traffic_cfg2.json"
    try:
        d = json.loads(p.read_text())
    except Exception:
        return None
    if d.get("kv_proj_tc_sha16") != kernel_source_sha16():
        return None
    return d.get("bd_bytes_per_launch")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.ok = False
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.002)

    def sample(self):
        try:
            self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
            r = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t is not None:
            self._stop.set()
            self._t.join()
            self.sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": int(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU legs
def cpu_oracle_run(x16, ck16, cv16, d_h, n, threads):
    """Reference algorithm (C restatement of attention.py:249-270) on float32 inputs,
    K' and V' — the reference has no 16-bit path."""
    from oracle import oracle as O
    O.fused_kv_proj_ref(x16, ck16, d_h, n, "first", threads=threads)
    O.fused_kv_proj_ref(x16, cv16, d_h, n, "last", threads=threads)


def make_cpu_inputs(L, d, d_h, n):
    import numpy as np
    from oracle import oracle as O
    rng = O.Rng(2024)
    x = O.rand_gaussian(rng, L, d, np.float32)
    ck = (O.rand_gaussian(rng, d - d_h, n * d_h, np.float32) / 8).astype(np.float32)
    cv = (O.rand_gaussian(rng, d - d_h, n * d_h, np.float32) / 8).astype(np.float32)
    return x, ck, cv


def cpu_baseline(L, d, d_h, n, budget_s=12.0):
    """Time the reference algorithm on the host: full-L steps until ~budget_s."""
    from oracle import oracle as O
    threads = O.default_threads()
    x, ck, cv = make_cpu_inputs(L, d, d_h, n)
    cpu_oracle_run(x[:64], ck, cv, d_h, n, threads)  # warm
    times = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(times) < 3:
        t0 = time.perf_counter()
        cpu_oracle_run(x, ck, cv, d_h, n, threads)
        times.append(time.perf_counter() - t0)
        if len(times) >= 50:
            break
    med = statistics.median(times)
    return {"value": L / med, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"{len(times)} full steps of cfg2 K'+V' (L={L}, FP32, C restatement of "
                      f"ref attention.py:249-270), median {med * 1e3:.1f} ms/step",
            "cpu": cpu_info(), "one_thread": cpu_one_thread(L, d, d_h, n)}


def cpu_info() -> dict:
    model = None
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        aff = os.cpu_count()
    return {"model": model, "cpu_count": os.cpu_count(), "affinity": aff}


def cpu_one_thread(L, d, d_h, n, sample_L=1024):
    """The same algorithm on ONE host thread (a bounded token sample, scaled)."""
    from oracle import oracle as O
    x, ck, cv = make_cpu_inputs(sample_L, d, d_h, n)
    cpu_oracle_run(x[:64], ck, cv, d_h, n, 1)
    t0 = time.perf_counter()
    cpu_oracle_run(x, ck, cv, d_h, n, 1)
    dt = time.perf_counter() - t0
    return {"value": sample_L / dt, "unit": "tokens/s", "cores": 1, "kind": "port",
            "sample": f"{sample_L} tokens of cfg2 K'+V' on 1 thread, {dt * 1e3:.0f} ms"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O
    d, d_h, n = CFG2["d"], CFG2["d_h"], CFG2["n_heads"]
    L = args.tokens * world  # same whole-job tokens per step as our arm
    threads = O.default_threads()
    x, ck, cv = make_cpu_inputs(L, d, d_h, n)
    # each step is a bounded sample of the step's tokens, scaled to the full step:
    # the kernel is independent 8-row blocks (attention.py:254-257), linear in L.
    sample_L = min(L, 8192)
    for _ in range(args.warmup):
        cpu_oracle_run(x[:sample_L], ck, cv, d_h, n, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_oracle_run(x[:sample_L], ck, cv, d_h, n, threads)
        times.append(time.perf_counter() - t0)
    total = sum(times) * (L / sample_L)
    value = args.steps * L / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": "cfg2 DSV2-Lite kv_b_proj K'+V' (d=512, d_h=128, 16+16 heads)",
                   "tokens_per_step": L, "sample_tokens_per_step": sample_L},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": f"{sample_L} of {L} tokens per step, scaled by L/sample "
                                   "(work is linear in L)",
                         "cpu": cpu_info(),
                         "one_thread": cpu_one_thread(L, d, d_h, n),
                         "port_vs_numba": "profiles/r02_ref_vs_port_cpu.json (the reference's "
                                          "own numba kernel beside this C port, build container)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2510_01718_b200 as bd
    from paper_2510_01718_b200 import _native as N

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        with stdout_to_stderr():
            dist.init_process_group("nccl", device_id=dev)
    dtype = torch.float16 if args.dtype == "fp16" else torch.bfloat16
    d, d_h, n_total = CFG2["d"], CFG2["d_h"], CFG2["n_heads"]
    if n_total % world:
        raise SystemExit(f"{n_total} heads do not shard over {world} GPUs")
    n = n_total // world              # heads of K (and of V) owned by this rank
    L = args.tokens * world           # head-sharded weak scaling: tokens grow with g
    K = d - d_h
    N_cols = n * d_h

    # ring of buffer sets exceeding 2x L2
    set_bytes = 2 * (L * d + 2 * K * N_cols + 2 * L * N_cols)
    R = max(2, math.ceil(2 * L2_BYTES / set_bytes) + 1)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    xs = [torch.randn(L, d, device=dev, generator=g).to(dtype) for _ in range(R)]
    cks = [(torch.randn(K, N_cols, device=dev, generator=g) / 8).to(dtype) for _ in range(R)]
    cvs = [(torch.randn(K, N_cols, device=dev, generator=g) / 8).to(dtype) for _ in range(R)]
    kos = [torch.empty(L, N_cols, device=dev, dtype=dtype) for _ in range(R)]
    vos = [torch.empty(L, N_cols, device=dev, dtype=dtype) for _ in range(R)]
    # dense comparator: original kv_b_proj weight (d x 2 N), one cuBLAS GEMM per step
    ws = [(torch.randn(d, 2 * N_cols, device=dev, generator=g) / 8).to(dtype) for _ in range(R)]
    dos = [torch.empty(L, 2 * N_cols, device=dev, dtype=dtype) for _ in range(R)]

    def bd_step(i):
        j = i % R
        bd.fused_kv_proj_grouped(xs[j], [(cks[j], d_h, n, bd.Tag.FIRST),
                                         (cvs[j], d_h, n, bd.Tag.LAST)],
                                 outs=[kos[j], vos[j]], check_finite=False)

    def dense_step(i):
        j = i % R
        torch.matmul(xs[j], ws[j], out=dos[j])

    stream = torch.cuda.Stream(device=dev)

    def capture(step_fn, k):
        for i in range(3):  # warm the path (attributes, cuBLAS handles) outside capture
            step_fn(i)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        before = N.launch_count()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(k):
                step_fn(i)
        return graph, N.launch_count() - before

    def timed(graph_w, graph_t):
        graph_w.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            s.record(stream)
            graph_t.replay()
            e.record(stream)
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # dense cuBLAS comparator first (also settles clocks)
    gdw, _ = capture(dense_step, args.warmup)
    gdt, _ = capture(dense_step, args.steps)
    dense_ms = statistics.median(timed(gdw, gdt) for _ in range(3))

    gbw, _ = capture(bd_step, args.warmup)
    gbt, launches = capture(bd_step, args.steps)
    sampler = ClockSampler(local)
    sampler.start()
    # `value`: median of 3 timed runs of exactly K steps (the burst protocol of the
    # dense comparator above and of the burst peak).  Then the same K-step run repeated
    # back to back for ~0.5 s under the clock sampler: the sustained (power-capped)
    # figure, reported beside it against the sustained peak.
    runs = [timed(gbw, gbt) for _ in range(3)]
    bd_ms = statistics.median(runs)
    sus = []
    t_end = time.perf_counter() + 0.5
    while time.perf_counter() < t_end and len(sus) < 5000:
        sus.append(timed(gbw, gbt))
    sus_ms = statistics.median(sus)
    kern_ms = bd_ms / args.steps  # the step is exactly one launch of the kernel

    ms_per_step = bd_ms / args.steps
    # L already counts every rank's tokens: each rank projects all L tokens for its heads
    value = L / (ms_per_step * 1e-3)
    dense_value = L / (dense_ms / args.steps * 1e-3)

    flops = 2 * 2 * L * K * N_cols  # K' and V', this rank (multiply FLOPs)
    bytes_alg = 2 * (L * d + 2 * K * N_cols + 2 * L * N_cols)
    peak_tf, peak_hbm, peak_kind = load_peaks()
    achieved_tf = flops / (kern_ms * 1e-3) / 1e12
    traffic = load_traffic()

    configs = None
    if world == 1 and not args.no_configs:
        configs = run_configs(torch, dev, peak_tf, peak_hbm)
    sampler.stop()

    gather = None
    if args.gather != "none":
        gather = run_gather(args, bd, torch, dist, dev, rank, world, dtype)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, bd, torch, dist, dev, world, dtype, L, d, d_h, n, cks[0], cvs[0])

    block = None
    if not args.no_block:
        block = run_block(args, torch, dist, dev, rank, world, dtype, stream)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(L, d, d_h, n)
        if configs is not None and "cfg2_fp32_exact" in configs:
            ex = configs["cfg2_fp32_exact"]
            ex["speedup_vs_cpu_port"] = ex["tokens_per_s"] / cpu["value"]

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (N(0,1) activations, random-init C_k/C_v and dense weight)",
        "config": {
            "workload": "cfg2: DSV2-Lite MLA kv_b_proj K'+V' (d=kv_lora_rank 512, d_h=128, "
                        "16 K heads + 16 V heads, K tag FIRST, V tag LAST), one launch/step",
            "tokens_per_step": L, "d": d, "d_h": d_h, "heads_per_gpu": n,
            "parallelism": f"head-sharded x{world}" if world > 1 else "single GPU",
            "l2": f"ring of {R} buffer sets, {R * set_bytes / 2**20:.0f} MiB > 2x126 MiB L2",
        },
        "roofline": {
            "bound": "tensor", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
            "frac": achieved_tf / peak_tf, "traffic": traffic,
            "peak_kind": f"{peak_kind} burst bf16/fp16 dense",
            "kernel_us": kern_ms * 1e3,
            "hbm_gbs": bytes_alg / (kern_ms * 1e-3) / 1e9, "hbm_peak_gbs": peak_hbm,
            "algorithmic_bytes": bytes_alg, "algorithmic_flops": flops,
        },
        "baselines": {
            "dense_cublas": {"value": dense_value, "unit": "tokens/s",
                             "ms_per_step": dense_ms / args.steps,
                             "what": "torch.matmul(x, W_kvb 512x4096) FP16, same ring"},
            "speedup_vs_dense_cublas": value / dense_value,
            "flop_ratio": d / (d - d_h),
        },
        "gpu_launches": launches,
        "clocks": sampler.summary(),
    }
    sus_tf = flops / (sus_ms / args.steps * 1e-3) / 1e12
    peak_sus = load_sustained_peak()
    line["sustained"] = {
        "runs": len(sus), "seconds": round(sum(sus) * 1e-3, 3),
        "ms_per_step_median": sus_ms / args.steps,
        "ms_per_step_p10_p90": [statistics.quantiles(sus, n=10)[0] / args.steps,
                                statistics.quantiles(sus, n=10)[-1] / args.steps] if len(sus) > 10 else None,
        "tokens_per_s": L / (sus_ms / args.steps * 1e-3), "achieved_tflops": sus_tf,
        "peak_sustained_tflops": peak_sus,
        "frac_of_sustained_peak": sus_tf / peak_sus if peak_sus else None}
    if e2e is not None:
        line["e2e"] = e2e
    if configs is not None:
        line["configs"] = configs
    if gather is not None:
        line["gather"] = gather
    if block is not None:
        line["block"] = block
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_block(args, torch, dist, dev, rank, world, dtype, stream):
    """BASELINE config 5: DeepSeek-V2-Lite MLA attention block (q_proj, kv_a + RMSNorm,
    BD kv_b_proj as ONE grouped launch, RoPE, causal SDPA, o_proj), random-init weights,
    `--block-tokens` tokens, heads sharded over the ranks (all_reduce of the output),
    vs the dense block with the original kv_b_proj weight (cuBLAS).  Strong scaling:
    the token count is fixed as g grows."""
    from paper_2510_01718_b200 import mla as M
    cfg = M.DSV2_LITE
    w = M.gen_random_mla(1234)
    p = M.mla_prepare(w)  # offline, CPU (global tags), then shard
    if world > 1:
        p = M.shard_bd_mla(p, world, rank)
    p = p.to(dev, dtype)
    wd = w.to(dev, dtype)
    L = args.block_tokens
    g = torch.Generator(device=dev).manual_seed(99)
    hid = torch.randn(L, cfg.hidden, device=dev, generator=g).to(dtype)
    steps, warm = 10, 3

    def time_fn(fn):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    bd_ms = time_fn(lambda: M.bd_mla_forward(hid, p))
    dense_ms = time_fn(lambda: M.mla_forward(hid, wd)) if world == 1 else None
    # the tcgen05 MLA attention kernel reading K'/V' head-major in place:
    # whole block, and in head groups of 4 through the L2 ring of group buffers
    bd_attn_ms = time_fn(lambda: M.bd_mla_forward(hid, p, attention="bd"))
    bd_attn_g4_ms = time_fn(lambda: M.bd_mla_forward(hid, p, attention="bd", head_group=4))
    out = {"workload": "cfg5: DeepSeek-V2-Lite MLA block (hidden 2048, 16 heads, kv_lora 512, "
                       "nope/rope/v 128/64/128), causal, random-init, BD kv_b_proj",
           "tokens": L, "heads_per_gpu": cfg.n_heads // world, "scaling": "strong",
           "bd_ms": bd_ms, "bd_tokens_per_s": L / (bd_ms * 1e-3),
           "bd_flops_per_gpu": M.block_flops(L, cfg, cfg.n_heads // world, bd=True),
           "qk_tag": p.qk_tag.value, "vo_tag": p.vo_tag.value,
           "bd_attention": {"ms": bd_attn_ms, "head_group_4_ms": bd_attn_g4_ms,
                            "what": "BD block with attention='bd' (csrc/mla_attn.cu) instead of "
                                    "cuDNN SDPA; head_group_4: K'/V' of 4 heads at a time "
                                    "through an L2-sized ring"}}
    if dense_ms is not None:
        out.update({"dense_ms": dense_ms, "dense_tokens_per_s": L / (dense_ms * 1e-3),
                    "speedup_vs_dense": dense_ms / bd_ms})
        out["breakdown"] = block_breakdown(torch, M, hid, w, wd, p, time_fn, dense_ms, bd_ms)
    return out


def block_breakdown(torch, M, hid, w, wd, p, time_fn, dense_ms, bd_ms):
    """Where the BD block's gain over the dense block comes from:
    the kv_b projection itself (BD kernel head-major vs cuBLAS, same tokens), the fused
    kv_a_layernorm (the BD block with fuse_norm=False), and the rest — the head-major
    K'/V' written straight into the SDPA operands instead of the dense block's
    view/reshape/cat copies."""
    from paper_2510_01718_b200.kv_proj import fused_kv_proj_grouped
    cfg = w.cfg
    L, H = hid.shape[0], cfg.n_heads
    unfused_ms = time_fn(lambda: M.bd_mla_forward(hid, p, fuse_norm=False))
    c_kv = torch.randn(L, cfg.kv_lora_rank, device=hid.device, dtype=hid.dtype)
    kvb = torch.empty(L, wd.w_kvb.shape[1], device=hid.device, dtype=hid.dtype)
    dense_proj_ms = time_fn(lambda: torch.matmul(c_kv, wd.w_kvb, out=kvb))
    kb = torch.empty(H, L, cfg.qk_nope, device=hid.device, dtype=hid.dtype)
    vb = torch.empty(H, L, cfg.v_head, device=hid.device, dtype=hid.dtype)
    specs = [(p.c_qk, cfg.qk_nope, H, p.qk_tag), (p.c_vo, cfg.v_head, H, p.vo_tag)]
    bd_proj_ms = time_fn(lambda: fused_kv_proj_grouped(c_kv, specs, outs=[kb, vb], out_layout="head",
                                                      check_finite=False))
    proj = dense_proj_ms - bd_proj_ms
    norm = unfused_ms - bd_ms
    return {"dense_ms": dense_ms, "bd_ms": bd_ms, "bd_unfused_norm_ms": unfused_ms,
            "kv_b_proj_dense_ms": dense_proj_ms, "kv_b_proj_bd_ms": bd_proj_ms,
            "gain_ms": {"kv_b_projection": proj, "fused_rmsnorm": norm,
                        "layout_and_rest": dense_ms - bd_ms - proj - norm},
            "note": "gain = dense_ms - bd_ms split by source; the BD FLOP saving is 0.54% of "
                    "the block (SURVEY 8(d)), the projection term is what BD itself buys"}


# ----------------------------------------------------------------------------- configs
def _roof(flops, nbytes, us, peak_tf, peak_hbm):
    """Roofline of one call: the bound is the resource its arithmetic intensity hits."""
    tf = flops / (us * 1e-6) / 1e12
    gbs = nbytes / (us * 1e-6) / 1e9
    ridge = peak_tf * 1e12 / (peak_hbm * 1e9)
    bound = "tensor" if flops / nbytes >= ridge else "hbm"
    frac = tf / peak_tf if bound == "tensor" else gbs / peak_hbm
    return {"bound": bound, "frac": round(frac, 4), "tflops": round(tf, 1), "hbm_gbs": round(gbs, 1)}


def run_configs(torch, dev, peak_tf, peak_hbm):
    """The other BASELINE configs and the paper's k_proj sweep, each against cuBLAS in
    the same dtype, every call on a cold-L2 ring (buffer sets > 2x L2), CUDA-graph
    timed (benchmark.time_ring_us).  N = 1, rank 0; inside the bench's clock sampler."""
    import paper_2510_01718_b200 as bd
    from paper_2510_01718_b200.benchmark import ring_size, time_ring_us
    from oracle import oracle as O
    F, Lt = bd.Tag.FIRST, bd.Tag.LAST
    g = torch.Generator(device=dev).manual_seed(77)

    def rnd(shape, dtype, scale=1.0):
        return (torch.randn(*shape, device=dev, generator=g) * scale).to(dtype)

    def inner_for(est_us, R):
        return max(R, min(2000, int(3000 / max(est_us, 1.0)) + 1))

    res = {}
    # cfg1: the FP32 exact kernel (bit-identical to the reference) vs the FP32 reference
    # on one host thread — the like-for-like arm
    L, d, d_h, n = 256, 512, 64, 8
    K, N = d - d_h, n * d_h
    f32 = torch.float32
    R = ring_size(4 * (L * d + 2 * K * N + 2 * L * N))
    sets = [(rnd((L, d), f32), rnd((K, N), f32, 1 / 8), rnd((K, N), f32, 1 / 8),
             torch.empty(L, N, device=dev), torch.empty(L, N, device=dev)) for _ in range(R)]
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, F), (s[2], d_h, n, Lt)],
                                                  outs=[s[3], s[4]], check_finite=False)
             for s in sets]
    us = time_ring_us(calls, inner_for(40, R))
    x32, ck32, cv32 = (t.cpu().numpy() for t in sets[0][:3])
    t0 = time.perf_counter()
    for _ in range(3):
        O.fused_kv_proj_ref(x32, ck32, d_h, n, "first", threads=1)
        O.fused_kv_proj_ref(x32, cv32, d_h, n, "last", threads=1)
    cpu_us = (time.perf_counter() - t0) / 3 * 1e6
    res["cfg1_fp32_exact"] = {
        "workload": "cfg1: d=512, 8 heads x 64, 256 tokens, K'+V' one launch, FP32 exact kernel "
                    "(bit-identical to the reference rounding sequence)",
        "us": round(us, 3), "tokens_per_s": L / (us * 1e-6),
        "cpu_ref_1thread_us": round(cpu_us, 1), "speedup_vs_cpu_ref_1thread": cpu_us / us,
        "note": "FP32 CUDA-core path (no FMA, reference order): latency-bound at L=256"}
    del sets, calls

    # cfg2 in FP32 on the exact kernel: the headline workload in the reference's own
    # precision and rounding sequence — the like-for-like arm against the CPU port
    # (cpu_baseline below times the same workload, FP32, on the host threads)
    L, d, d_h, n = 8192, 512, 128, 16
    K, N = d - d_h, n * d_h
    R = ring_size(4 * (L * d + 2 * K * N + 2 * L * N))
    sets = [(rnd((L, d), f32), rnd((K, N), f32, 1 / 8), rnd((K, N), f32, 1 / 8),
             torch.empty(L, N, device=dev), torch.empty(L, N, device=dev)) for _ in range(R)]
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, F), (s[2], d_h, n, Lt)],
                                                  outs=[s[3], s[4]], check_finite=False)
             for s in sets]
    us = time_ring_us(calls, max(R, 8))
    res["cfg2_fp32_exact"] = {
        "workload": "cfg2 K'+V' (8192 tokens, 16 + 16 heads x 128, d = 512) in FP32 on the exact "
                    "kernel (bit-identical to the reference rounding sequence)",
        "us": round(us, 1), "tokens_per_s": L / (us * 1e-6),
        "note": "like-for-like with cpu_baseline (same workload, FP32); FP32 CUDA-core path, "
                "no FMA (the reference's order)"}
    del sets, calls

    # cfg3: Llama-2-7B K/V, 65536 tokens, BF16 (K = 3968 streams, round-robin tiles)
    L, d, d_h, n = 65536, 4096, 128, 32
    K, N = d - d_h, n * d_h
    bf = torch.bfloat16
    sets = [(rnd((L, d), bf), rnd((K, N), bf, 1 / 64), rnd((K, N), bf, 1 / 64),
             torch.empty(L, N, device=dev, dtype=bf), torch.empty(L, N, device=dev, dtype=bf))
            for _ in range(2)]
    calls = [lambda s=s: bd.fused_kv_proj_grouped(s[0], [(s[1], d_h, n, F), (s[2], d_h, n, Lt)],
                                                  outs=[s[3], s[4]], check_finite=False)
             for s in sets]
    us = time_ring_us(calls, 4)
    dsets = [(s[0], rnd((d, 2 * N), bf, 1 / 64), torch.empty(L, 2 * N, device=dev, dtype=bf))
             for s in sets]
    del calls
    sets = None
    dcalls = [lambda s=s: torch.matmul(s[0], s[1], out=s[2]) for s in dsets]
    dus = time_ring_us(dcalls, 4)
    flops = 2 * 2 * L * K * N
    res["cfg3"] = {"workload": "cfg3: Llama-2-7B K/V (d=4096, 32 x 128), 65536 tokens, BF16, "
                               "K'+V' one launch", "us": round(us, 1),
                   "tokens_per_s": L / (us * 1e-6), "dense_cublas_us": round(dus, 1),
                   "speedup_vs_dense_cublas": dus / us,
                   "roofline": _roof(flops, 2 * (L * d + 2 * K * N + 2 * L * N), us, peak_tf, peak_hbm)}
    del dsets, dcalls
    torch.cuda.empty_cache()

    # cfg4: BD low-rank linear 4096 -> 1024 -> 4096, 32768 tokens, FP16
    L, din, r, dout = 32768, 4096, 1024, 4096
    h16 = torch.float16
    basis, coeff = rnd((din, r), h16, 1 / 64), rnd((r, dout - r), h16, 1 / 32)
    fac = bd.BDFactors(axis=bd.Axis.COLUMN, tag=Lt, basis=basis.double().cpu().numpy(),
                       coeff=coeff.double().cpu().numpy(), orig_rows=din,
                       orig_cols=dout, rank=r, residual=0.0, rank_deficient=False)
    layer = bd.BDLinearLayer(fac, basis, coeff)
    U, Vt, W = rnd((din, r), h16, 1 / 64), rnd((r, dout), h16, 1 / 32), rnd((din, dout), h16, 1 / 64)
    sets = [(rnd((L, din), h16), torch.empty(L, dout, device=dev, dtype=h16),
             torch.empty(L, r, device=dev, dtype=h16)) for _ in range(2)]
    us = time_ring_us([lambda s=s: bd.bd_linear_forward(s[0], layer, out=s[1], check_finite=False)
                       for s in sets], 4)

    def lowrank(s):
        torch.matmul(s[0], U, out=s[2])
        torch.matmul(s[2], Vt, out=s[1])
    lus = time_ring_us([lambda s=s: lowrank(s) for s in sets], 4)
    dus = time_ring_us([lambda s=s: torch.matmul(s[0], W, out=s[1]) for s in sets], 4)
    flops = 2 * L * (din * r + r * (dout - r))
    res["cfg4"] = {"workload": "cfg4: BD low-rank linear 4096 -> rank 1024 -> 4096, 32768 tokens, "
                               "FP16 (two tcgen05 GEMMs, h written into y and re-read)",
                   "us": round(us, 1), "tokens_per_s": L / (us * 1e-6),
                   "lowrank_cublas_us": round(lus, 1), "speedup_vs_lowrank_cublas": lus / us,
                   "dense_cublas_us": round(dus, 1), "speedup_vs_dense_cublas": dus / us,
                   "roofline": _roof(flops, 2 * (2 * L * din + 2 * L * dout + din * r + r * dout),
                                     us, peak_tf, peak_hbm)}
    del sets, layer, basis, coeff, U, Vt, W
    torch.cuda.empty_cache()

    # the paper's k_proj sweep (ref bench.py:102-162, Tables 4/5): n=128 heads,
    # d=512, d_h=128, tag FIRST, L = 64 ... 65536, FP16 and BF16; plus cfg2's shape
    # (16 + 16 heads, K'+V' one launch) at decode-sized L
    def sweep(dtype, d, d_h, n, Ls, grouped):
        K, N = d - d_h, n * d_h
        pts = []
        for L in Ls:
            nprob = 2 if grouped else 1
            set_bytes = 2 * (L * d + nprob * (K * N + L * N))
            R = ring_size(set_bytes)
            sets = [(rnd((L, d), dtype), [rnd((K, N), dtype, 1 / 8) for _ in range(nprob)],
                     [torch.empty(L, N, device=dev, dtype=dtype) for _ in range(nprob)])
                    for _ in range(R)]
            tags = [F, Lt][:nprob]
            calls = [lambda s=s: bd.fused_kv_proj_grouped(
                s[0], [(c, d_h, n, t) for c, t in zip(s[1], tags)], outs=s[2], check_finite=False)
                for s in sets]
            est = 4 + 2 * L * d * N * nprob / 1.2e9
            inner = inner_for(est, R)
            # decode-sized points last a few µs: more replays for a stable median
            reps = 11 if est < 20 else 5
            if L == Ls[0]:  # the sweep's first graph: one discarded measurement (warm-up)
                time_ring_us(calls, inner, reps=reps)
            us = time_ring_us(calls, inner, reps=reps)
            dsets = [(s[0], rnd((d, nprob * N), dtype, 1 / 8),
                      torch.empty(L, nprob * N, device=dev, dtype=dtype)) for s in sets]
            del calls
            sets = None
            dus = time_ring_us([lambda s=s: torch.matmul(s[0], s[1], out=s[2]) for s in dsets], inner,
                               reps=reps)
            del dsets
            flops = 2 * L * K * N * nprob
            nbytes = 2 * (L * d + nprob * (K * N + L * N))
            pts.append({"L": L, "us": round(us, 2), "cublas_us": round(dus, 2),
                        "speedup_vs_cublas": round(dus / us, 4),
                        "tokens_per_s": L / (us * 1e-6),
                        "roofline": _roof(flops, nbytes, us, peak_tf, peak_hbm)})
            torch.cuda.empty_cache()
        return pts

    paper_Ls = [64 * 2 ** i for i in range(11)]
    for name, dt in (("fp16", torch.float16), ("bf16", torch.bfloat16)):
        pts = sweep(dt, 512, 128, 128, paper_Ls, grouped=False)
        res[f"paper_kproj_{name}"] = {
            "workload": f"paper Table {4 if name == 'fp16' else 5} shape: k_proj, d=512, 128 heads "
                        f"x 128, tag FIRST, {name.upper()}, vs cuBLAS X @ W_k (512 x 16384)",
            "points": pts,
            "mean_speedup_vs_cublas": statistics.mean(p["speedup_vs_cublas"] for p in pts),
            "paper_mean_speedup_a6000": 1.32 if name == "fp16" else 1.34}
    res["cfg2_small_l_fp16"] = {
        "workload": "cfg2 shape (16 + 16 heads x 128, d=512), K'+V' one launch, decode-sized L, "
                    "FP16, vs cuBLAS X @ W_kvb (512 x 4096)",
        "points": sweep(torch.float16, 512, 128, 16, [64, 128, 256, 512], grouped=True)}
    return res


def run_gather(args, bd, torch, dist, dev, rank, world, dtype):
    """The head all-gather paths of SURVEY 8(e), timed at every N (exercised at N = 1):
    `nccl` = head-major projection of this rank's heads + one all_gather_into_tensor per
    problem; `fused` = the all-gather fused into the projection's epilogue over
    symmetric (peer) memory + one symmetric-memory barrier.  Per step, cfg2 K'+V',
    tokens_per_gpu tokens (the full-width K'/V' every rank ends up holding)."""
    from paper_2510_01718_b200 import parallel as P
    d, d_h, n_total = CFG2["d"], CFG2["d_h"], CFG2["n_heads"]
    n = n_total // world
    L = args.tokens
    K = d - d_h
    with stdout_to_stderr():
        return _run_gather(args, bd, torch, dist, dev, rank, world, dtype, P, d, d_h, n_total,
                           n, L, K)


def _run_gather(args, bd, torch, dist, dev, rank, world, dtype, P, d, d_h, n_total, n, L, K):
    own_pg = False
    if not dist.is_initialized():
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                world_size=1, device_id=dev)
        own_pg = True
    g = torch.Generator(device=dev).manual_seed(4321)
    x = torch.randn(L, d, device=dev, generator=g).to(dtype)
    ck = (torch.randn(K, n * d_h, device=dev, generator=g) / 8).to(dtype)
    cv = (torch.randn(K, n * d_h, device=dev, generator=g) / 8).to(dtype)
    specs = [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)]
    full_bytes = 2 * 2 * L * n_total * d_h  # K' + V', full width, 16-bit
    out = {"tokens_per_gpu": L, "world": world,
           "ingress_bytes_per_gpu": full_bytes * (world - 1) // world,
           "full_width_bytes": full_bytes}
    steps = 20

    def time_eager(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            fn()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) * 1e3

    def all_ok(ok: bool) -> bool:
        """Every rank agrees before a timed collective loop: a rank that failed locally
        must not leave the others blocked in a barrier (the multi-GPU paths have only run
        on one device here, so they are guarded rather than trusted)."""
        t = torch.tensor([1 if ok else 0], device=dev, dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    modes = ["nccl", "fused"] if args.gather == "both" else [args.gather]
    if "nccl" in modes:
        def nccl_step():
            kh, vh = bd.fused_kv_proj_grouped(x, specs, out_layout="head", check_finite=False)
            P.all_gather_heads(kh, d_h)
            P.all_gather_heads(vh, d_h)
        try:
            if not all_ok(True):
                raise RuntimeError("a rank could not start the NCCL gather")
            us = time_eager(nccl_step)
            out["nccl"] = {"us": round(us, 2), "tokens_per_s": L * world / (us * 1e-6),
                           "what": "projection (head-major) + NCCL all_gather_into_tensor x2"}
        except Exception as exc:  # report, never hide
            out["nccl"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if "fused" in modes:
        sg, local_err = None, None
        try:
            sg = P.SymmetricGather([(n_total, L, d_h), (n_total, L, d_h)], dtype)
            # one un-timed projection with the fused gather (no barrier yet): a launch
            # error shows up here, on this rank, before any rank enters a collective
            P.fused_allgather_kv_proj(x, specs, sg.peers, sg.rank)
            torch.cuda.synchronize()
        except Exception as exc:
            local_err = f"{type(exc).__name__}: {exc}"[:300]
        try:
            if not all_ok(local_err is None):
                raise RuntimeError(local_err or "another rank could not set up the fused gather")
            sg.barrier()

            def fused_step():
                P.fused_allgather_kv_proj(x, specs, sg.peers, sg.rank)
                sg.barrier()
            us = time_eager(fused_step)
            # parity of the gathered buffers against the plain projection (this rank's planes)
            kh, vh = bd.fused_kv_proj_grouped(x, specs, out_layout="head", check_finite=False)
            ok = bool(torch.equal(sg.local[0][rank * n:(rank + 1) * n], kh)
                      and torch.equal(sg.local[1][rank * n:(rank + 1) * n], vh))
            out["fused"] = {"us": round(us, 2), "tokens_per_s": L * world / (us * 1e-6),
                            "own_planes_bit_identical": ok,
                            "what": "bd_kv_proj_grouped_allgather: epilogue TMA-stores every box "
                                    "to all ranks' symmetric buffers + symm-mem barrier"}
        except Exception as exc:
            out["fused"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if own_pg:
        dist.destroy_process_group()
    return out


def run_e2e(args, bd, torch, dist, dev, world, dtype, L, d, d_h, n, ck, cv):
    """Same metric through the public API with pinned HOST buffers: every step copies its
    x in (H2D), runs the grouped projection, and reads K', V' back (D2H)."""
    N_cols = n * d_h
    x_host = [torch.randn(L, d).to(dtype).pin_memory() for _ in range(2)]
    k_host = [torch.empty(L, N_cols, dtype=dtype).pin_memory() for _ in range(2)]
    v_host = [torch.empty(L, N_cols, dtype=dtype).pin_memory() for _ in range(2)]
    specs = [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)]
    steps = max(3, min(args.steps, 50))

    def step(i):
        bd.fused_kv_proj_grouped_host(x_host[i % 2], specs, outs=[k_host[i % 2], v_host[i % 2]])

    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for i in range(steps):
        step(i)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    esz = 2
    return {"value": L / (ms / steps * 1e-3), "unit": "tokens/s",
            "h2d_bytes_per_step": L * d * esz, "d2h_bytes_per_step": 2 * L * N_cols * esz,
            "steps": steps, "api": "fused_kv_proj_grouped_host (pinned host x -> K', V')"}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
