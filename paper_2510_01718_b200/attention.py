"""Multi-head attention and its basis-decomposed (BD) form on the GPU.

Mirrors the reference module (ref: pkg/src/bdattn/attention.py) name for name:
``MHAWeights``, ``BDAWeights``, ``mha_forward``, ``bda_prepare``, ``fused_kv_proj``,
``bda_forward``, ``attention_scores``.  Differences, all deliberate:

* tensors are ``torch.Tensor`` (any float dtype; FP16/BF16 allowed — the reference is
  P32/P64 only) and ``bda_forward`` runs on the GPU.  K' and V' are ONE
  launch of the BD kernel (libbd_kvproj.so, both tags in one grouped launch).  For
  FP16/BF16, Q' and the output projection are cuBLAS GEMMs and the per-head softmax
  attention is ``scaled_dot_product_attention``; for FP32/FP64 (the exactness path)
  every product runs on the exact kernel in the reference's rounding order;
* ``bda_prepare`` is the offline step and stays on the CPU in NumPy/SciPy (see
  decompose.py) with the reference's exact operation sequence, so the chosen tags
  (the basis S) are bit-identical; 16-bit models are prepared in FP64 and rounded.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np
import torch
import torch.nn.functional as F

from .decompose import Axis, BDFactors, Tag, bd_decompose_both, ordered_matmul
from .errors import PrecisionError, ShapeError
from .kv_proj import fused_kv_proj, fused_kv_proj_grouped
from .linear import matmul as _exact_matmul

__all__ = ["MHAWeights", "BDAWeights", "mha_forward", "bda_prepare", "fused_kv_proj",
           "bda_forward", "attention_scores", "select_tag", "merge_heads"]


def _shape(t: torch.Tensor) -> tuple[int, ...]:
    return tuple(int(s) for s in t.shape)


@dataclass(frozen=True)
class MHAWeights:
    """w_q, w_k, w_v: d x (n d_h); w_o: (n d_h) x d (ref attention.py:30-81)."""

    d: int
    n_heads: int
    d_h: int
    w_q: torch.Tensor
    w_k: torch.Tensor
    w_v: torch.Tensor
    w_o: torch.Tensor

    def __post_init__(self):
        if self.d_h >= self.d:
            raise ValueError(f"d_h ({self.d_h}) must be < d ({self.d})")
        if self.d_h < 1 or self.n_heads < 1:
            raise ValueError("d_h and n_heads must be positive")
        width = self.n_heads * self.d_h
        for name, t, shape in (("w_q", self.w_q, (self.d, width)),
                               ("w_k", self.w_k, (self.d, width)),
                               ("w_v", self.w_v, (self.d, width)),
                               ("w_o", self.w_o, (width, self.d))):
            if _shape(t) != shape:
                raise ShapeError(f"{name} has shape {_shape(t)}, expected {shape}")
        if len({t.dtype for t in (self.w_q, self.w_k, self.w_v, self.w_o)}) != 1:
            raise PrecisionError("all four projection matrices must share precision")

    @property
    def precision(self) -> torch.dtype:
        return self.w_q.dtype

    @property
    def param_count(self) -> int:
        return 4 * self.d * self.n_heads * self.d_h

    def cast(self, dtype: torch.dtype) -> "MHAWeights":
        return replace(self, **{k: getattr(self, k).to(dtype) for k in ("w_q", "w_k", "w_v", "w_o")})

    def to(self, device) -> "MHAWeights":
        return replace(self, **{k: getattr(self, k).to(device) for k in ("w_q", "w_k", "w_v", "w_o")})


@dataclass(frozen=True)
class BDAWeights:
    """Prepared BD parameter set (ref attention.py:84-140).

    b_qk d x (n d_h); c_qk, c_vo (d - d_h) x (n d_h) in the reference layout (the
    kernel's B operand, read MN-major with no transpose); b_vo (n d_h) x d.
    One tag per target for every head.
    """

    d: int
    n_heads: int
    d_h: int
    b_qk: torch.Tensor
    c_qk: torch.Tensor
    c_vo: torch.Tensor
    b_vo: torch.Tensor
    qk_tag: Tag
    vo_tag: Tag
    qk_candidate_residuals: tuple[float, float]
    vo_candidate_residuals: tuple[float, float]
    qk_deficient_heads: tuple[int, ...] = ()
    vo_deficient_heads: tuple[int, ...] = ()

    def __post_init__(self):
        if self.d_h >= self.d:
            raise ValueError(f"d_h ({self.d_h}) must be < d ({self.d})")
        width = self.n_heads * self.d_h
        rest = self.d - self.d_h
        for name, t, shape in (("b_qk", self.b_qk, (self.d, width)),
                               ("c_qk", self.c_qk, (rest, width)),
                               ("c_vo", self.c_vo, (rest, width)),
                               ("b_vo", self.b_vo, (width, self.d))):
            if _shape(t) != shape:
                raise ShapeError(f"{name} has shape {_shape(t)}, expected {shape}")
        if len({t.dtype for t in (self.b_qk, self.c_qk, self.c_vo, self.b_vo)}) != 1:
            raise PrecisionError("all prepared matrices must share precision")

    @property
    def precision(self) -> torch.dtype:
        return self.b_qk.dtype

    @property
    def param_count(self) -> int:
        width = self.n_heads * self.d_h
        return 2 * width * self.d + 2 * width * (self.d - self.d_h)

    @property
    def mean_residual_qk(self) -> float:
        return self.qk_candidate_residuals[0 if self.qk_tag is Tag.FIRST else 1]

    @property
    def mean_residual_vo(self) -> float:
        return self.vo_candidate_residuals[0 if self.vo_tag is Tag.FIRST else 1]

    def cast(self, dtype: torch.dtype) -> "BDAWeights":
        return replace(self, **{k: getattr(self, k).to(dtype)
                                for k in ("b_qk", "c_qk", "c_vo", "b_vo")})

    def to(self, device) -> "BDAWeights":
        return replace(self, **{k: getattr(self, k).to(device)
                                for k in ("b_qk", "c_qk", "c_vo", "b_vo")})


# --------------------------------------------------------------------------- forward
def _attend(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, n_heads: int, d_h: int,
            causal: bool = False) -> torch.Tensor:
    """Per-head softmax(q_i k_i^T / sqrt(d_h)) v_i, heads concatenated
    (ref attention.py:143-154).

    16-bit: one SDPA call over [n_heads, L, d_h] views (flash / cuDNN kernels).
    float32/float64 (the exactness path): the reference's own sequence — fixed-order
    products on the exact kernel, the scale rounded to the operand precision
    (ref tensor.py:292-295), a max-shifted softmax — so the block output tracks the
    reference to rounding of exp/sum only.
    """
    L = q.shape[0]
    if q.dtype in (torch.float32, torch.float64):
        inv = torch.tensor(1.0 / math.sqrt(d_h), dtype=q.dtype).item()
        mask = (torch.ones(L, L, dtype=torch.bool, device=q.device).triu(1) if causal else None)
        outs = []
        for i in range(n_heads):
            lo, hi = i * d_h, (i + 1) * d_h
            s = _exact_matmul(q[:, lo:hi].contiguous(), k[:, lo:hi].T.contiguous()) * inv
            if mask is not None:
                s = s.masked_fill(mask, float("-inf"))
            e = torch.exp(s - s.amax(dim=1, keepdim=True))
            outs.append(_exact_matmul(e / e.sum(dim=1, keepdim=True), v[:, lo:hi].contiguous()))
        return torch.cat(outs, dim=1)
    qh = q.view(L, n_heads, -1).transpose(0, 1)[None]  # [1, H, L, d_h]: fused SDPA kernels
    kh = k.view(L, n_heads, -1).transpose(0, 1)[None]
    vh = v.view(L, n_heads, -1).transpose(0, 1)[None]
    o = F.scaled_dot_product_attention(qh, kh, vh, is_causal=causal, scale=1.0 / math.sqrt(d_h))
    return o[0].transpose(0, 1).reshape(L, n_heads * vh.shape[-1])


def _proj(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """Dense projection: cuBLAS for 16-bit, the reference's fixed-order product on the
    exact kernel for float32/float64 (ref tensor.py:189-213)."""
    if x.dtype in (torch.float32, torch.float64):
        return _exact_matmul(x, w)
    return x @ w


def _check_input(x: torch.Tensor, d: int, dtype: torch.dtype) -> None:
    if x.dim() != 2 or x.shape[1] != d:
        raise ShapeError(f"input has {x.shape[-1] if x.dim() else 0} cols, model dim is {d}")
    if x.dtype != dtype:
        raise PrecisionError("input and weights must share precision")


def mha_forward(x: torch.Tensor, w: MHAWeights, *, causal: bool = False) -> torch.Tensor:
    """Baseline multi-head attention, L x d -> L x d (ref attention.py:157-166)."""
    _check_input(x, w.d, w.precision)
    q, k, v = _proj(x, w.w_q), _proj(x, w.w_k), _proj(x, w.w_v)
    return _proj(_attend(q, k, v, w.n_heads, w.d_h, causal), w.w_o)


def bda_forward(x: torch.Tensor, w: BDAWeights, *, causal: bool = False,
                check_finite: bool = True) -> torch.Tensor:
    """BD attention forward; output matches ``mha_forward`` (ref attention.py:298-307).

    K' and V' come from ONE launch of the BD kernel (two problems, each with its own
    tag) instead of the reference's two ``fused_kv_proj`` calls.  Like the reference,
    whose every ``Tensor2D`` result is finite-checked (tensor.py:112-113), a non-finite
    K', V' or output raises ``ValueError``; ``check_finite=False`` is the unchecked,
    sync-free (CUDA-graph capturable) fast path.
    """
    _check_input(x, w.d, w.precision)
    q = _proj(x, w.b_qk)
    specs = [(w.c_qk, w.d_h, w.n_heads, w.qk_tag), (w.c_vo, w.d_h, w.n_heads, w.vo_tag)]
    if x.dtype in (torch.float16, torch.bfloat16) and w.d_h % 64 == 0:
        # K', V' head-major [H, L, d_h]: SDPA's [1, H, L, d_h] operands, no transpose copy
        kh, vh = fused_kv_proj_grouped(x, specs, check_finite=check_finite, out_layout="head")
        L, H = x.shape[0], w.n_heads
        qh = q.view(L, H, w.d_h).transpose(0, 1)[None]
        o = F.scaled_dot_product_attention(qh, kh[None], vh[None], is_causal=causal,
                                           scale=1.0 / math.sqrt(w.d_h))
        out = _proj(o[0].transpose(0, 1).reshape(L, H * w.d_h), w.b_vo)
    else:
        k, v = fused_kv_proj_grouped(x, specs, check_finite=check_finite)
        out = _proj(_attend(q, k, v, w.n_heads, w.d_h, causal), w.b_vo)
    if check_finite and not bool(torch.isfinite(out).all()):
        raise ValueError("operation produced non-finite values")
    return out


def attention_scores(x: torch.Tensor, w: MHAWeights | BDAWeights, head: int) -> torch.Tensor:
    """Pre-softmax L x L scores of one head, unscaled (ref attention.py:310-325)."""
    if not isinstance(w, (MHAWeights, BDAWeights)):
        raise TypeError(f"expected MHAWeights or BDAWeights, got {type(w).__name__}")
    if not 0 <= head < w.n_heads:
        raise IndexError(f"head {head} out of range for {w.n_heads} heads")
    lo, hi = head * w.d_h, (head + 1) * w.d_h
    if isinstance(w, MHAWeights):
        q = _proj(x, w.w_q[:, lo:hi].contiguous())
        k = _proj(x, w.w_k[:, lo:hi].contiguous())
    else:
        q = _proj(x, w.b_qk[:, lo:hi].contiguous())
        # only this head's coefficient columns: the kernel is column-separable
        k = fused_kv_proj(x, w.c_qk[:, lo:hi], w.d_h, 1, w.qk_tag, check_finite=False)
    return _proj(q, k.T.contiguous())


# --------------------------------------------------------------------------- prep
def select_tag(candidates: list[tuple[BDFactors, BDFactors]],
               force_first: bool = False) -> tuple[Tag, tuple[float, float]]:
    """One tag for all heads: the smaller MEAN residual, ties to FIRST
    (ref attention.py:181-189).  Must see every head — a per-shard choice could
    differ, so head sharding happens after this."""
    n = len(candidates)
    mean_first = sum(f.residual for f, _ in candidates) / n
    mean_last = sum(l.residual for _, l in candidates) / n
    if force_first or mean_first <= mean_last:
        return Tag.FIRST, (mean_first, mean_last)
    return Tag.LAST, (mean_first, mean_last)


def merge_heads(qk_sel: list[BDFactors], vo_sel: list[BDFactors]):
    """Per-head factors -> (b_qk, c_qk, c_vo, b_vo) (ref attention.py:222-228)."""
    b_qk = np.concatenate([f.basis for f in qk_sel], axis=1)
    c_qk = np.concatenate([np.ascontiguousarray(f.coeff.T) for f in qk_sel], axis=1)
    c_vo = np.concatenate([f.coeff for f in vo_sel], axis=1)
    b_vo = np.concatenate([f.basis for f in vo_sel], axis=0)
    return b_qk, c_qk, c_vo, b_vo


def _host_array(t: torch.Tensor, dtype) -> np.ndarray:
    return np.ascontiguousarray(t.detach().to("cpu", dtype).numpy())


def bda_prepare(w: MHAWeights, *, force_first: bool = False,
                prepare_in_p64: bool = False) -> BDAWeights:
    """Offline preparation: per-head QK column BD and VO row BD at rank d_h, one
    shared tag per target by mean residual, merge (ref attention.py:192-246).

    Runs on the CPU (NumPy/SciPy).  float64 models prepare in float64; float32 in
    float32 unless ``prepare_in_p64``; float16/bfloat16 models always prepare in
    float64.  Results are rounded to the model dtype and placed on its device.
    """
    model_dtype = w.precision
    if model_dtype == torch.float64 or model_dtype == torch.float32 and not prepare_in_p64:
        work = torch.float64 if model_dtype == torch.float64 else torch.float32
    else:
        work = torch.float64
    wq, wk, wv, wo = (_host_array(t, work) for t in (w.w_q, w.w_k, w.w_v, w.w_o))
    qk_pairs, vo_pairs = [], []
    for i in range(w.n_heads):
        lo, hi = i * w.d_h, (i + 1) * w.d_h
        # ref _head_products (attention.py:169-178): fixed-order products
        qk = ordered_matmul(np.ascontiguousarray(wq[:, lo:hi]), np.ascontiguousarray(wk[:, lo:hi].T))
        vo = ordered_matmul(np.ascontiguousarray(wv[:, lo:hi]), np.ascontiguousarray(wo[lo:hi, :]))
        qk_pairs.append(bd_decompose_both(qk, w.d_h, Axis.COLUMN))
        vo_pairs.append(bd_decompose_both(vo, w.d_h, Axis.ROW))
    qk_tag, qk_means = select_tag(qk_pairs, force_first)
    vo_tag, vo_means = select_tag(vo_pairs, force_first)
    qk_sel = [p[0 if qk_tag is Tag.FIRST else 1] for p in qk_pairs]
    vo_sel = [p[0 if vo_tag is Tag.FIRST else 1] for p in vo_pairs]
    mats = merge_heads(qk_sel, vo_sel)
    dev = w.w_q.device
    b_qk, c_qk, c_vo, b_vo = (torch.from_numpy(np.ascontiguousarray(m)).to(dev, model_dtype)
                              for m in mats)
    return BDAWeights(
        d=w.d, n_heads=w.n_heads, d_h=w.d_h, b_qk=b_qk, c_qk=c_qk, c_vo=c_vo, b_vo=b_vo,
        qk_tag=qk_tag, vo_tag=vo_tag, qk_candidate_residuals=qk_means,
        vo_candidate_residuals=vo_means,
        qk_deficient_heads=tuple(i for i, f in enumerate(qk_sel) if f.rank_deficient),
        vo_deficient_heads=tuple(i for i, f in enumerate(vo_sel) if f.rank_deficient))
