"""Parity harness of the drop-in API (ref: pkg/src/bdattn/verify.py, tensor.py:377-419).

* ``Rng`` / ``rand_gaussian`` — the reference's seeded sources: PCG64 keyed through
  SeedSequence(seed, spawn_key), values drawn in float64 and rounded, so one seed gives
  the same model at every precision and in the reference itself.
* ``gen_random_mha`` — Gaussian weights at scale 1/sqrt(d) with the scale rounded to the
  operand precision first (ref verify.py:83-99, tensor.py:292-295).
* ``max_relative_error`` / ``EQUIVALENCE_THRESHOLDS`` / ``equivalence_check`` /
  ``reconstruction_error_report`` — the reference's metrics, run on the GPU forward.

These are part of the package API (the reference exports them) — not the CPU oracle.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from .attention import BDAWeights, MHAWeights, bda_forward, bda_prepare, mha_forward
from .decompose import Tag, blas_matmul

# ref verify.py:23 (P64 / P32), extended with the 16-bit kernel tolerances of
# SURVEY.md App. A for the kernel-level parity of fused_kv_proj.
EQUIVALENCE_THRESHOLDS = {torch.float64: 1e-10, torch.float32: 1e-4}
KERNEL_MAXREL = {torch.float16: 1e-3, torch.bfloat16: 8e-3}

_NP = {torch.float64: np.float64, torch.float32: np.float32, torch.float16: np.float16}


class Rng:
    """Deterministic random source (ref tensor.py:377-405)."""

    def __init__(self, seed: int, _spawn_key: tuple[int, ...] = ()):
        self._seed = int(seed)
        self._spawn_key = tuple(_spawn_key)
        ss = np.random.SeedSequence(self._seed, spawn_key=self._spawn_key)
        self._generator = np.random.Generator(np.random.PCG64(ss))

    @property
    def seed(self) -> int:
        return self._seed

    def derive(self, index: int) -> "Rng":
        return Rng(self._seed, self._spawn_key + (int(index),))

    def standard_normal(self, rows: int, cols: int) -> np.ndarray:
        return self._generator.standard_normal((rows, cols))

    def __repr__(self) -> str:
        key = "".join(f",{k}" for k in self._spawn_key)
        return f"Rng(seed={self._seed}{key})"


def _to_torch(a: np.ndarray, dtype: torch.dtype, device) -> torch.Tensor:
    if dtype == torch.bfloat16:  # numpy has no bfloat16: round from float64 in torch
        return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dtype)
    return torch.from_numpy(np.ascontiguousarray(a.astype(_NP[dtype], copy=False))).to(device)


def rand_gaussian(rng: Rng, rows: int, cols: int, dtype: torch.dtype = torch.float64,
                  device="cpu") -> torch.Tensor:
    """i.i.d. N(0,1), drawn in float64 then rounded (ref tensor.py:408-419)."""
    if rows < 1 or cols < 1:
        raise ValueError(f"rand_gaussian needs positive dims, got {rows}x{cols}")
    return _to_torch(rng.standard_normal(rows, cols), dtype, device)


def _scaled_gaussian(rng: Rng, rows: int, cols: int, s: float, dtype, device) -> torch.Tensor:
    vals = rng.standard_normal(rows, cols)
    if dtype in (torch.float64, torch.float32, torch.float16):
        t = _NP[dtype]
        return torch.from_numpy(np.ascontiguousarray(vals.astype(t) * t(s))).to(device)
    # bfloat16: round the draw, multiply by the rounded scale in float32, round again
    v = torch.from_numpy(vals).to(torch.bfloat16)
    return (v.float() * float(torch.tensor(s, dtype=torch.bfloat16))).to(torch.bfloat16).to(device)


def gen_random_mha(rng: Rng, d: int, d_h: int, n_heads: int,
                   dtype: torch.dtype = torch.float64, device="cpu") -> MHAWeights:
    """Gaussian projection weights at scale 1/sqrt(d) (ref verify.py:83-99)."""
    if d_h >= d:
        raise ValueError(f"d_h ({d_h}) must be < d ({d})")
    s = 1.0 / math.sqrt(d)
    width = n_heads * d_h
    w_q = _scaled_gaussian(rng, d, width, s, dtype, device)
    w_k = _scaled_gaussian(rng, d, width, s, dtype, device)
    w_v = _scaled_gaussian(rng, d, width, s, dtype, device)
    w_o = _scaled_gaussian(rng, width, d, s, dtype, device)
    return MHAWeights(d=d, n_heads=n_heads, d_h=d_h, w_q=w_q, w_k=w_k, w_v=w_v, w_o=w_o)


def max_relative_error(result: torch.Tensor, reference: torch.Tensor) -> float:
    """max |result - reference| / max |reference|, in float64 (ref verify.py:74-80)."""
    r = torch.as_tensor(result).detach().to("cpu", torch.float64)
    ref = torch.as_tensor(reference).detach().to("cpu", torch.float64)
    diff = float((r - ref).abs().max())
    denom = float(ref.abs().max())
    return diff if denom == 0.0 else diff / denom


@dataclass(frozen=True)
class TrialSummary:
    trials: int
    failures: int
    worst_value: float
    threshold: float

    def __post_init__(self):
        if not 0 <= self.failures <= self.trials:
            raise ValueError("failures must lie in [0, trials]")

    @property
    def ok(self) -> bool:
        return self.failures == 0


def equivalence_check(rng: Rng, d: int, d_h: int, n_heads: int, seq_len: int,
                      dtype: torch.dtype = torch.float64, trials: int = 20,
                      threshold: float | None = None, device="cuda") -> TrialSummary:
    """Fresh model per trial, BDA (GPU kernel) vs MHA end to end (ref verify.py:158-187)."""
    thr = EQUIVALENCE_THRESHOLDS[dtype] if threshold is None else float(threshold)
    failures, worst = 0, 0.0
    for t in range(trials):
        stream = rng.derive(t)
        w = gen_random_mha(stream, d, d_h, n_heads, dtype, device)
        prepared = bda_prepare(w)
        x = rand_gaussian(stream, seq_len, d, dtype, device)
        err = max_relative_error(bda_forward(x, prepared), mha_forward(x, w))
        worst = max(worst, err)
        failures += err > thr
    return TrialSummary(trials=trials, failures=int(failures), worst_value=worst, threshold=thr)


class Target(Enum):
    QK = "qk"
    VO = "vo"


@dataclass(frozen=True)
class ErrorReport:
    mse: float
    nmse: float
    max_rel: float
    per_head: tuple[tuple[float, float], ...]
    precision: torch.dtype


def _np(t: torch.Tensor) -> np.ndarray:
    """Host array in the tensor's own precision: the reference forms the per-head
    products in the layer precision (verify.py:102-124, ``_fast_matmul``) and widens
    only the results to 64 bit (:136-137)."""
    return np.ascontiguousarray(t.detach().to("cpu").numpy())


def reconstruction_error_report(w: MHAWeights, prepared: BDAWeights,
                                target: Target) -> ErrorReport:
    """Per-head MSE/NMSE of the prepared factors vs the exact products
    (ref verify.py:103-155)."""
    if (w.d, w.n_heads, w.d_h) != (prepared.d, prepared.n_heads, prepared.d_h):
        raise ValueError("weight geometries differ between model and prepared form")
    d_h = w.d_h
    wq, wk, wv, wo = (_np(t) for t in (w.w_q, w.w_k, w.w_v, w.w_o))
    bqk, cqk, cvo, bvo = (_np(t) for t in (prepared.b_qk, prepared.c_qk, prepared.c_vo,
                                            prepared.b_vo))
    per_head, max_rel = [], 0.0
    for i in range(w.n_heads):
        lo, hi = i * d_h, (i + 1) * d_h
        if target is Target.QK:
            ref = blas_matmul(wq[:, lo:hi], wk[:, lo:hi].T)
            basis, coeff = bqk[:, lo:hi], cqk[:, lo:hi].T
            rebuilt = blas_matmul(basis, coeff)
            parts = [basis, rebuilt] if prepared.qk_tag is Tag.FIRST else [rebuilt, basis]
            recon = np.concatenate(parts, axis=1)
        else:
            ref = blas_matmul(wv[:, lo:hi], wo[lo:hi, :])
            basis, coeff = bvo[lo:hi, :], cvo[:, lo:hi]
            rebuilt = blas_matmul(coeff, basis)
            parts = [basis, rebuilt] if prepared.vo_tag is Tag.FIRST else [rebuilt, basis]
            recon = np.concatenate(parts, axis=0)
        ref = ref.astype(np.float64)
        diff = recon.astype(np.float64) - ref
        mse = float(np.mean(diff * diff))
        power = float(np.mean(ref * ref))
        nmse = mse / power if power > 0.0 else (0.0 if mse == 0.0 else math.inf)
        per_head.append((mse, nmse))
        peak = float(np.abs(ref).max())
        dmax = float(np.abs(diff).max())
        max_rel = max(max_rel, dmax / peak if peak > 0.0 else dmax)
    n = len(per_head)
    return ErrorReport(mse=sum(m for m, _ in per_head) / n, nmse=sum(s for _, s in per_head) / n,
                       max_rel=max_rel, per_head=tuple(per_head), precision=prepared.precision)
