"""DeepSeek-V2-Lite MLA attention block with a BD-rewritten ``kv_b_proj`` (BASELINE
config 5).

MLA (multi-head latent attention) projects the hidden state to a shared latent
``c_kv`` (kv_lora_rank = 512), RMS-normalises it and expands it per head with
``kv_b_proj`` into K_nope (128) and V (128); a decoupled RoPE part (64 dims) is computed
separately (``q_pe`` per head, ``k_pe`` shared).  Structure after transformers 5.5
``models/deepseek_v2/modeling_deepseek_v2.py:317-359`` [ext]; geometry from
BASELINE.json (hidden 2048, 16 heads, no q-LoRA).

BD applies to the no-RoPE part exactly as to MHA:

* QK, per head h: P_qk = W_q_nope^h (hidden x 128) @ W_uk^h^T (128 x 512) has rank 128;
  its COLUMN BD picks 128 latent dims S_k: basis B_qk^h = P_qk[:, S_k] replaces the
  head's q_nope weight and C^h (128 x 384) gives K'_h = c_kv[:, S_k] + c_kv[:, ~S_k] C^h^T.
* VO, per head h: P_vo = W_uv^h (512 x 128) @ W_o^h (128 x hidden); its ROW BD picks S_v:
  B_vo^h = P_vo[S_v, :] replaces the head's rows of o_proj and V'_h = c_kv[:, S_v] +
  c_kv[:, ~S_v] C_vo^h.
* One tag per target for all heads by mean residual (ref attention.py:181-189), so the
  K' and V' of all heads are ONE grouped launch of the BD kernel — exactly BASELINE
  config 2 — and kv_b_proj's 512 x 4096 weight becomes two 384 x 2048 coefficient
  matrices (25 % fewer weights, 4/3 fewer FLOPs in that GEMM).
* The RoPE channels are untouched: q_pe, k_pe and the 1/sqrt(192) softmax scale are
  the same in both forms, so scores are preserved exactly (in exact arithmetic).

Weights use the x @ W convention of the reference (row-major [in, out]).  Prep runs
offline on the CPU in float64 through the same decompose path as ``bda_prepare``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np
import torch
import torch.distributed as dist
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

from .attention import select_tag
from .decompose import Axis, Tag, bd_decompose_both, ordered_matmul
from . import _native as _N
from .errors import NativeLibraryError, PrecisionError, ShapeError
from .kv_proj import (_on_device, fold_rmsnorm, fused_kv_proj_grouped,
                      fused_rmsnorm_kv_proj_grouped)


# attention-core backends, in preference order (cuDNN first: it supports the MLA head
# dims 192/128 natively; math covers float64 test shapes)
_BACKENDS = [SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION,
             SDPBackend.EFFICIENT_ATTENTION, SDPBackend.MATH]


@dataclass(frozen=True)
class MLAConfig:
    hidden: int = 2048
    n_heads: int = 16
    kv_lora_rank: int = 512
    qk_nope: int = 128
    qk_rope: int = 64
    v_head: int = 128
    rope_theta: float = 10000.0
    rms_eps: float = 1e-6
    rope_interleaved: bool = True  # DeepSeek-V2: complex rotation of adjacent pairs

    @property
    def qk_head(self) -> int:
        return self.qk_nope + self.qk_rope


DSV2_LITE = MLAConfig()


@dataclass(frozen=True)
class MLAWeights:
    """Dense MLA block weights (x @ W layout)."""

    cfg: MLAConfig
    w_q: torch.Tensor      # hidden x H (nope + rope), per head [nope | rope]
    w_kva: torch.Tensor    # hidden x (kv_lora + rope):  [c_kv | k_pe]
    kva_norm: torch.Tensor  # kv_lora (RMSNorm weight)
    w_kvb: torch.Tensor    # kv_lora x H (nope + v), per head [k_nope | v]
    w_o: torch.Tensor      # H v x hidden

    def to(self, device=None, dtype=None) -> "MLAWeights":
        f = {k: getattr(self, k).to(device=device, dtype=dtype)
             for k in ("w_q", "w_kva", "kva_norm", "w_kvb", "w_o")}
        return replace(self, **f)


@dataclass(frozen=True)
class BDMLAWeights:
    """MLA block with the BD-rewritten kv_b_proj / q_nope / o_proj."""

    cfg: MLAConfig
    w_q: torch.Tensor       # hidden x H (nope + rope): per head [B_qk^h | W_q_rope^h]
    w_kva: torch.Tensor
    kva_norm: torch.Tensor
    c_qk: torch.Tensor      # (kv_lora - nope) x H nope, reference layout
    c_vo: torch.Tensor      # (kv_lora - v) x H v
    b_vo: torch.Tensor      # H v x hidden
    qk_tag: Tag
    vo_tag: Tag
    qk_candidate_residuals: tuple[float, float]
    vo_candidate_residuals: tuple[float, float]
    n_heads: int            # heads held (== cfg.n_heads unless head-sharded)
    # kv_a_layernorm folded into the coefficients for the fused-norm projection:
    # (c_qk_g, c_vo_g, qk_rep_gamma, vo_rep_gamma) — see kv_proj.fold_rmsnorm
    norm_fold: tuple | None = None

    def to(self, device=None, dtype=None) -> "BDMLAWeights":
        f = {k: getattr(self, k).to(device=device, dtype=dtype)
             for k in ("w_q", "w_kva", "kva_norm", "c_qk", "c_vo", "b_vo")}
        if self.norm_fold is not None:
            cq, cv, gq, gv = self.norm_fold
            f["norm_fold"] = (cq.to(device=device, dtype=dtype), cv.to(device=device, dtype=dtype),
                              gq.to(device=device), gv.to(device=device))
        return replace(self, **f)

    @property
    def kv_param_count(self) -> int:
        return int(self.c_qk.numel() + self.c_vo.numel())


def gen_random_mla(seed: int, cfg: MLAConfig = DSV2_LITE, dtype=torch.float64,
                   device="cpu") -> MLAWeights:
    """Random-init block: N(0,1)/sqrt(fan_in) weights, RMSNorm weight 1 (synthetic,
    no checkpoint is available offline)."""
    g = torch.Generator().manual_seed(seed)
    H = cfg.n_heads

    def w(i, o):
        return (torch.randn(i, o, generator=g, dtype=torch.float64) / math.sqrt(i)).to(device, dtype)

    return MLAWeights(cfg=cfg, w_q=w(cfg.hidden, H * cfg.qk_head),
                      w_kva=w(cfg.hidden, cfg.kv_lora_rank + cfg.qk_rope),
                      kva_norm=torch.ones(cfg.kv_lora_rank, dtype=dtype, device=device),
                      w_kvb=w(cfg.kv_lora_rank, H * (cfg.qk_nope + cfg.v_head)),
                      w_o=w(H * cfg.v_head, cfg.hidden))


def mla_prepare(w: MLAWeights, *, force_first: bool = False) -> BDMLAWeights:
    """Offline BD of the MLA block (float64 on the CPU, rounded to the model dtype)."""
    cfg, H = w.cfg, w.cfg.n_heads
    if cfg.qk_nope != cfg.v_head:
        raise ShapeError("the grouped K'/V' launch needs qk_nope == v_head")
    nope, rope, dv, r = cfg.qk_nope, cfg.qk_rope, cfg.v_head, cfg.kv_lora_rank
    f64 = lambda t: np.ascontiguousarray(t.detach().to("cpu", torch.float64).numpy())  # noqa: E731
    wq, wkvb, wo = f64(w.w_q), f64(w.w_kvb), f64(w.w_o)
    qk_pairs, vo_pairs = [], []
    for h in range(H):
        q0 = h * (nope + rope)
        k0 = h * (nope + dv)
        w_qn = np.ascontiguousarray(wq[:, q0:q0 + nope])             # hidden x 128
        w_uk_t = np.ascontiguousarray(wkvb[:, k0:k0 + nope].T)       # 128 x 512
        w_uv = np.ascontiguousarray(wkvb[:, k0 + nope:k0 + nope + dv])  # 512 x 128
        w_oh = np.ascontiguousarray(wo[h * dv:(h + 1) * dv, :])      # 128 x hidden
        qk_pairs.append(bd_decompose_both(ordered_matmul(w_qn, w_uk_t), nope, Axis.COLUMN))
        vo_pairs.append(bd_decompose_both(ordered_matmul(w_uv, w_oh), dv, Axis.ROW))
    qk_tag, qk_means = select_tag(qk_pairs, force_first)
    vo_tag, vo_means = select_tag(vo_pairs, force_first)
    qk_sel = [p[0 if qk_tag is Tag.FIRST else 1] for p in qk_pairs]
    vo_sel = [p[0 if vo_tag is Tag.FIRST else 1] for p in vo_pairs]
    wq_bd = wq.copy()
    for h, f in enumerate(qk_sel):  # B_qk^h replaces the head's q_nope weight
        wq_bd[:, h * (nope + rope):h * (nope + rope) + nope] = f.basis
    c_qk = np.concatenate([np.ascontiguousarray(f.coeff.T) for f in qk_sel], axis=1)
    c_vo = np.concatenate([f.coeff for f in vo_sel], axis=1)
    b_vo = np.concatenate([f.basis for f in vo_sel], axis=0)
    dev, dt = w.w_q.device, w.w_q.dtype
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    assert c_qk.shape == (r - nope, H * nope) and b_vo.shape == (H * dv, cfg.hidden)
    return mla_fold_norm(BDMLAWeights(
        cfg=cfg, w_q=t(wq_bd), w_kva=w.w_kva, kva_norm=w.kva_norm, c_qk=t(c_qk), c_vo=t(c_vo),
        b_vo=t(b_vo), qk_tag=qk_tag, vo_tag=vo_tag, qk_candidate_residuals=qk_means,
        vo_candidate_residuals=vo_means, n_heads=H))


def mla_fold_norm(w: BDMLAWeights) -> BDMLAWeights:
    """Attach kv_a_layernorm folded into the coefficients (``kv_proj.fold_rmsnorm``, in
    float64, rounded once to the weights' dtype) for the fused-norm projection."""
    cfg = w.cfg
    gamma = w.kva_norm.detach().to(torch.float64)
    cq, gq = fold_rmsnorm(w.c_qk.to(torch.float64), gamma, cfg.qk_nope, w.qk_tag)
    cv, gv = fold_rmsnorm(w.c_vo.to(torch.float64), gamma, cfg.v_head, w.vo_tag)
    dt = w.c_qk.dtype
    return replace(w, norm_fold=(cq.to(dt), cv.to(dt), gq, gv))


def shard_bd_mla(w: BDMLAWeights, world: int, rank: int) -> BDMLAWeights:
    """Heads [r H/g, (r+1) H/g): q columns, C columns, B_vo rows; w_kva replicated."""
    from .parallel import head_range
    cfg = w.cfg
    h0, h1 = head_range(w.n_heads, world, rank)
    qh, dn, dv = cfg.qk_head, cfg.qk_nope, cfg.v_head
    fold = None
    if w.norm_fold is not None:
        cq, cv, gq, gv = w.norm_fold
        fold = (cq[:, h0 * dn:h1 * dn].contiguous(), cv[:, h0 * dv:h1 * dv].contiguous(), gq, gv)
    return replace(w, norm_fold=fold, w_q=w.w_q[:, h0 * qh:h1 * qh].contiguous(),
                   c_qk=w.c_qk[:, h0 * dn:h1 * dn].contiguous(),
                   c_vo=w.c_vo[:, h0 * dv:h1 * dv].contiguous(),
                   b_vo=w.b_vo[h0 * dv:h1 * dv, :].contiguous(), n_heads=h1 - h0)


# --------------------------------------------------------------------------- forward
def _rms_norm(x: torch.Tensor, weight: torch.Tensor, eps: float) -> torch.Tensor:
    xf = x.to(torch.promote_types(x.dtype, torch.float32))
    y = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
    return (y * weight.float()).to(x.dtype)


def _rope(t: torch.Tensor, theta: float, interleaved: bool = True) -> torch.Tensor:
    """RoPE over the last dim of [L, ..., r] at positions 0..L-1, in float32.

    ``interleaved``: DeepSeek-V2's form — adjacent pairs (2i, 2i+1) are one complex
    number rotated by pos * theta^(-2i/r) (transformers ``modeling_deepseek_v2.py``
    ``apply_rotary_emb`` [ext]); otherwise rotate-half (Llama convention)."""
    L, r = t.shape[0], t.shape[-1]
    inv = 1.0 / (theta ** (torch.arange(0, r, 2, device=t.device, dtype=torch.int64).float() / r))
    ang = torch.arange(L, device=t.device, dtype=torch.float32)[:, None] * inv[None, :]
    if interleaved:
        tc = torch.view_as_complex(t.float().reshape(*t.shape[:-1], r // 2, 2).contiguous())
        rot = torch.polar(torch.ones_like(ang), ang).view((L,) + (1,) * (t.dim() - 2) + (r // 2,))
        return torch.view_as_real(tc * rot).flatten(-2).to(t.dtype)
    cos = torch.cat([ang.cos(), ang.cos()], -1)
    sin = torch.cat([ang.sin(), ang.sin()], -1)
    shape = (L,) + (1,) * (t.dim() - 2) + (r,)
    tf = t.float()
    rot = torch.cat([-tf[..., r // 2:], tf[..., :r // 2]], -1)
    return (tf * cos.view(shape) + rot * sin.view(shape)).to(t.dtype)


def _mla_attend(q_nope, q_pe, k_nope, k_pe, v, n_heads, cfg: MLAConfig, causal=True):
    """softmax([q_nope|q_pe][k_nope|k_pe]^T / sqrt(192)) v per head, one SDPA call."""
    L = q_nope.shape[0]
    q = torch.cat([q_nope.view(L, n_heads, cfg.qk_nope), q_pe.view(L, n_heads, cfg.qk_rope)], -1)
    k = torch.cat([k_nope.view(L, n_heads, cfg.qk_nope),
                   k_pe.view(L, 1, cfg.qk_rope).expand(L, n_heads, cfg.qk_rope)], -1)
    vh = v.view(L, n_heads, cfg.v_head)
    # [1, H, L, D] views; cuDNN's fused attention takes E=192 with Ev=128 directly
    # (3.6 ms at 32k tokens on B200, vs 18.7 ms for flash with V zero-padded to 192)
    with sdpa_kernel(_BACKENDS):
        o = F.scaled_dot_product_attention(q.transpose(0, 1)[None], k.transpose(0, 1)[None],
                                           vh.transpose(0, 1)[None], is_causal=causal,
                                           scale=1.0 / math.sqrt(cfg.qk_head))
    return o[0].transpose(0, 1).reshape(L, n_heads * cfg.v_head)


def _split_q(q: torch.Tensor, n_heads: int, cfg: MLAConfig):
    L = q.shape[0]
    qh = q.view(L, n_heads, cfg.qk_head)
    return qh[..., :cfg.qk_nope].reshape(L, -1), qh[..., cfg.qk_nope:]


def _latent(hidden: torch.Tensor, w_kva, kva_norm, cfg: MLAConfig):
    kv = hidden @ w_kva
    c_kv = _rms_norm(kv[:, :cfg.kv_lora_rank], kva_norm, cfg.rms_eps)
    return c_kv.contiguous(), kv[:, cfg.kv_lora_rank:]


def mla_forward(hidden: torch.Tensor, w: MLAWeights, *, causal: bool = True) -> torch.Tensor:
    """Dense MLA block (the baseline): cuBLAS kv_b_proj with the original weight."""
    cfg, H = w.cfg, w.cfg.n_heads
    q_nope, q_pe = _split_q(hidden @ w.w_q, H, cfg)
    c_kv, k_pe = _latent(hidden, w.w_kva, w.kva_norm, cfg)
    kvb = (c_kv @ w.w_kvb).view(-1, H, cfg.qk_nope + cfg.v_head)
    k_nope = kvb[..., :cfg.qk_nope].reshape(-1, H * cfg.qk_nope)
    v = kvb[..., cfg.qk_nope:].reshape(-1, H * cfg.v_head)
    rope = lambda t: _rope(t, cfg.rope_theta, cfg.rope_interleaved)  # noqa: E731
    o = _mla_attend(q_nope, rope(q_pe), k_nope, rope(k_pe), v,
                    H, cfg, causal)
    return o @ w.w_o


def mla_attention(q: torch.Tensor, k_nope: torch.Tensor, k_pe: torch.Tensor, v: torch.Tensor,
                  *, scale: float, causal: bool = True,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """MLA prefill attention on the tcgen05 kernel (``bd_mla_attention``, csrc/mla_attn.cu):

        out[t, h] = softmax_s(scale (q[t,h,:128] . k_nope[h,s] + q[t,h,128:] . k_pe[s])) v[h,s]

    ``q`` [L, H, 192] (last dim contiguous; any token / head strides), ``k_nope`` and ``v``
    head-major [H, L, 128] — the BD projection's ``out_layout="head"`` outputs, read in
    place — and ``k_pe`` [L, 64], the RoPE key shared by all heads (never broadcast).
    Returns [L, H, 128] (or writes ``out``).  FP16/BF16 CUDA tensors; no fallback.
    """
    if q.dim() != 3 or k_nope.dim() != 3 or v.dim() != 3 or k_pe.dim() != 2:
        raise ShapeError("q [L,H,192], k_nope [H,L,128], k_pe [L,64], v [H,L,128] expected")
    L, H, dq = q.shape
    if tuple(k_nope.shape) != (H, L, 128) or tuple(v.shape) != (H, L, 128) or \
            tuple(k_pe.shape) != (L, 64) or dq != 192:
        raise ShapeError(f"inconsistent shapes q{tuple(q.shape)} k_nope{tuple(k_nope.shape)} "
                         f"k_pe{tuple(k_pe.shape)} v{tuple(v.shape)}")
    dt = q.dtype
    if any(t.dtype != dt for t in (k_nope, k_pe, v)) or dt not in (torch.float16, torch.bfloat16):
        raise PrecisionError("mla_attention: q, k_nope, k_pe, v must share float16/bfloat16")
    if not all(t.is_cuda for t in (q, k_nope, k_pe, v)):
        raise NativeLibraryError("mla_attention needs CUDA tensors (no CPU fallback)")
    if any(t.stride(-1) != 1 for t in (q, k_nope, k_pe, v)):
        raise ShapeError("mla_attention: the last dimension must be contiguous")
    if out is None:
        out = torch.empty((L, H, 128), dtype=dt, device=q.device)
    elif tuple(out.shape) != (L, H, 128) or out.dtype != dt or out.stride(-1) != 1:
        raise ShapeError("out must be [L, H, 128] of q's dtype with a contiguous last dim")
    st = _on_device(q.device, _N.load().bd_mla_attention,
                    q.data_ptr(), q.stride(0), q.stride(1),
                    k_nope.data_ptr(), k_nope.stride(1), k_nope.stride(0),
                    k_pe.data_ptr(), k_pe.stride(0),
                    v.data_ptr(), v.stride(1), v.stride(0),
                    out.data_ptr(), out.stride(0), out.stride(1),
                    L, H, 128, 64, 128, float(scale), 1 if causal else 0,
                    _N.BD_F16 if dt == torch.float16 else _N.BD_BF16)
    _N.check(st, "bd_mla_attention")
    return out


def bd_mla_forward(hidden: torch.Tensor, w: BDMLAWeights, *, causal: bool = True,
                   group=None, fuse_norm: bool = True, attention: str = "sdpa",
                   head_group: int | None = None) -> torch.Tensor:
    """BD MLA block: K'_nope and V' of all (local) heads in ONE launch of the BD kernel,
    with kv_a_layernorm fused into it (``fuse_norm``, when the weights carry the fold:
    the raw latent is read once and never normalised in memory).  With head-sharded
    weights (``shard_bd_mla``) the partial outputs are summed with one all_reduce over
    ``group``.

    ``attention="sdpa"``: the attention core is torch SDPA (cuDNN) on [K'_nope | k_pe]
    per head.  ``attention="bd"`` (16-bit, DeepSeek-V2 head geometry): the tcgen05 kernel
    ``mla_attention`` reads K'_nope / V' head-major and the shared k_pe in place — no
    key concatenation, no RoPE-key broadcast — and, with ``head_group = G``, the block
    runs G heads at a time: the BD projection of a group's K'/V' into a 2-deep ring of
    group buffers sized to stay in L2, then the attention over them, so K'/V' go from the
    projection's epilogue to the attention's TMA loads through L2 instead of a round
    trip through HBM."""
    cfg, H = w.cfg, w.n_heads
    L = hidden.shape[0]
    if attention not in ("sdpa", "bd"):
        raise ValueError(f"attention must be 'sdpa' or 'bd', not {attention!r}")
    use_bd_attn = attention == "bd"
    if use_bd_attn and (hidden.dtype not in (torch.float16, torch.bfloat16) or cfg.qk_nope != 128
                        or cfg.qk_rope != 64 or cfg.v_head != 128):
        raise ShapeError("attention='bd' needs 16-bit activations and nope/rope/v = 128/64/128")
    q = hidden @ w.w_q
    # fused norm: exact kernel (float32/64) any shape; tensor cores need the latent row
    # resident (d_h in {64, 128}, kv_lora - d_h <= 384 — DeepSeek-V2-Lite's 128 / 384)
    fused = fuse_norm and w.norm_fold is not None and (
        hidden.dtype in (torch.float32, torch.float64)
        or (cfg.qk_nope in (64, 128) and cfg.v_head in (64, 128)
            and cfg.kv_lora_rank - min(cfg.qk_nope, cfg.v_head) <= 384))
    if fused:
        kv = hidden @ w.w_kva
        c_kv, k_pe = kv[:, :cfg.kv_lora_rank].contiguous(), kv[:, cfg.kv_lora_rank:]
    else:
        c_kv, k_pe = _latent(hidden, w.w_kva, w.kva_norm, cfg)
    rope = lambda t: _rope(t, cfg.rope_theta, cfg.rope_interleaved)  # noqa: E731

    def project(h0, h1, k_out, v_out):
        dn, dv = cfg.qk_nope, cfg.v_head
        if fused:
            cq, cv, gq, gv = w.norm_fold
            fused_rmsnorm_kv_proj_grouped(
                c_kv, [(cq[:, h0 * dn:h1 * dn], gq, dn, h1 - h0, w.qk_tag),
                       (cv[:, h0 * dv:h1 * dv], gv, dv, h1 - h0, w.vo_tag)], cfg.rms_eps,
                outs=[k_out, v_out], out_layout="head", check_finite=False)
        else:
            fused_kv_proj_grouped(
                c_kv, [(w.c_qk[:, h0 * dn:h1 * dn], dn, h1 - h0, w.qk_tag),
                       (w.c_vo[:, h0 * dv:h1 * dv], dv, h1 - h0, w.vo_tag)],
                outs=[k_out, v_out], out_layout="head", check_finite=False)

    if use_bd_attn:
        qv = q.view(L, H, cfg.qk_head)
        qv[..., cfg.qk_nope:] = rope(qv[..., cfg.qk_nope:])   # RoPE in place, no concat
        k_pe_r = rope(k_pe).contiguous()
        scale = 1.0 / math.sqrt(cfg.qk_head)
        o = torch.empty((L, H, cfg.v_head), dtype=q.dtype, device=q.device)
        G = H if head_group is None else max(1, min(H, int(head_group)))
        ring = [(torch.empty((G, L, cfg.qk_nope), dtype=q.dtype, device=q.device),
                 torch.empty((G, L, cfg.v_head), dtype=q.dtype, device=q.device))
                for _ in range(1 if G == H else 2)]
        for gi, h0 in enumerate(range(0, H, G)):
            h1 = min(H, h0 + G)
            kb, vb = ring[gi % len(ring)]
            kb, vb = kb[:h1 - h0], vb[:h1 - h0]
            project(h0, h1, kb, vb)
            mla_attention(qv[:, h0:h1], kb, k_pe_r, vb, scale=scale, causal=causal,
                          out=o[:, h0:h1])
        out = o.view(L, H * cfg.v_head) @ w.b_vo
    else:
        # The BD kernel writes K'_nope head-major straight into the first qk_nope columns
        # of the attention key buffer [H, L, nope + rope] (row stride nope + rope) and V'
        # head-major into [H, L, v]: the SDPA operands need no transpose or concatenation
        # copy of K'/V'; only the shared RoPE key part is broadcast into each head's tail.
        k_buf = torch.empty((H, L, cfg.qk_head), dtype=c_kv.dtype, device=c_kv.device)
        v_buf = torch.empty((H, L, cfg.v_head), dtype=c_kv.dtype, device=c_kv.device)
        project(0, H, k_buf[..., :cfg.qk_nope], v_buf)
        k_buf[..., cfg.qk_nope:] = rope(k_pe)[None]
        q_nope, q_pe = _split_q(q, H, cfg)
        q = torch.cat([q_nope.view(L, H, cfg.qk_nope), rope(q_pe).view(L, H, cfg.qk_rope)], -1)
        with sdpa_kernel(_BACKENDS):
            o = F.scaled_dot_product_attention(q.transpose(0, 1)[None], k_buf[None], v_buf[None],
                                               is_causal=causal, scale=1.0 / math.sqrt(cfg.qk_head))
        o = o[0].transpose(0, 1).reshape(L, H * cfg.v_head)
        out = o @ w.b_vo
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(out, group=group)
    return out


# --------------------------------------------------------------------------- checkpoints
# Hugging Face DeepseekV2Attention parameter names (transformers 5.5
# models/deepseek_v2/modeling_deepseek_v2.py:310-333 [ext]); nn.Linear stores [out, in],
# this module uses x @ W ([in, out]).
_HF_DENSE = ("q_proj.weight", "kv_a_proj_with_mqa.weight", "kv_a_layernorm.weight",
             "kv_b_proj.weight", "o_proj.weight")


def mla_config_from_hf(hf_config) -> MLAConfig:
    """MLAConfig from a transformers DeepseekV2Config (q-LoRA-free attention only)."""
    if getattr(hf_config, "q_lora_rank", None) is not None:
        raise ShapeError("q_lora_rank set: only the q_proj (no q-LoRA) attention is supported")
    rope = getattr(hf_config, "rope_parameters", None) or {}
    return MLAConfig(hidden=hf_config.hidden_size, n_heads=hf_config.num_attention_heads,
                     kv_lora_rank=hf_config.kv_lora_rank, qk_nope=hf_config.qk_nope_head_dim,
                     qk_rope=hf_config.qk_rope_head_dim, v_head=hf_config.v_head_dim,
                     rope_theta=float(rope.get("rope_theta", getattr(hf_config, "rope_theta", 10000.0))),
                     rms_eps=float(hf_config.rms_norm_eps), rope_interleaved=True)


def mla_from_hf(state: dict, cfg: MLAConfig, prefix: str = "") -> MLAWeights:
    """Dense MLAWeights from a DeepseekV2Attention state dict (keys under ``prefix``).
    kv_b_proj's rows are per head [k_nope | v] — already this module's column order."""
    missing = [k for k in _HF_DENSE if prefix + k not in state]
    if missing:
        raise ShapeError(f"state dict lacks {missing} under prefix {prefix!r}")
    g = lambda k: state[prefix + k].detach()  # noqa: E731
    H = cfg.n_heads
    w = MLAWeights(cfg=cfg, w_q=g("q_proj.weight").T.contiguous(),
                   w_kva=g("kv_a_proj_with_mqa.weight").T.contiguous(),
                   kva_norm=g("kv_a_layernorm.weight").contiguous(),
                   w_kvb=g("kv_b_proj.weight").T.contiguous(),
                   w_o=g("o_proj.weight").T.contiguous())
    want = {"w_q": (cfg.hidden, H * cfg.qk_head), "w_kva": (cfg.hidden, cfg.kv_lora_rank + cfg.qk_rope),
            "kva_norm": (cfg.kv_lora_rank,), "w_kvb": (cfg.kv_lora_rank, H * (cfg.qk_nope + cfg.v_head)),
            "w_o": (H * cfg.v_head, cfg.hidden)}
    for k, shp in want.items():
        if tuple(getattr(w, k).shape) != shp:
            raise ShapeError(f"{k}: shape {tuple(getattr(w, k).shape)}, expected {shp}")
    return w


def bd_mla_state_dict(w: BDMLAWeights, prefix: str = "") -> dict:
    """The rewritten checkpoint of one attention layer: q_proj carries B_qk in each head's
    nope columns, kv_b_proj is replaced by the two coefficient matrices (reference layout)
    and their tags, o_proj carries B_vo.  [out, in] like the original."""
    tag = lambda t: torch.tensor(0 if t is Tag.FIRST else 1, dtype=torch.int8)  # noqa: E731
    return {prefix + "q_proj.weight": w.w_q.T.contiguous(),
            prefix + "kv_a_proj_with_mqa.weight": w.w_kva.T.contiguous(),
            prefix + "kv_a_layernorm.weight": w.kva_norm.contiguous(),
            prefix + "kv_b_proj.c_qk": w.c_qk.contiguous(),
            prefix + "kv_b_proj.c_vo": w.c_vo.contiguous(),
            prefix + "kv_b_proj.qk_tag": tag(w.qk_tag),
            prefix + "kv_b_proj.vo_tag": tag(w.vo_tag),
            prefix + "o_proj.weight": w.b_vo.T.contiguous()}


def bd_mla_from_state_dict(state: dict, cfg: MLAConfig, prefix: str = "") -> BDMLAWeights:
    """Inverse of ``bd_mla_state_dict`` (candidate residuals are not stored: NaN)."""
    g = lambda k: state[prefix + k].detach()  # noqa: E731
    tag = lambda k: Tag.FIRST if int(g(k)) == 0 else Tag.LAST  # noqa: E731
    c_qk, c_vo = g("kv_b_proj.c_qk").contiguous(), g("kv_b_proj.c_vo").contiguous()
    H = c_qk.shape[1] // cfg.qk_nope
    if c_qk.shape != (cfg.kv_lora_rank - cfg.qk_nope, H * cfg.qk_nope) or \
            c_vo.shape != (cfg.kv_lora_rank - cfg.v_head, H * cfg.v_head):
        raise ShapeError(f"coefficient shapes {tuple(c_qk.shape)}, {tuple(c_vo.shape)} do not fit {cfg}")
    nan = (float("nan"), float("nan"))
    w = BDMLAWeights(cfg=cfg, w_q=g("q_proj.weight").T.contiguous(),
                     w_kva=g("kv_a_proj_with_mqa.weight").T.contiguous(),
                     kva_norm=g("kv_a_layernorm.weight").contiguous(), c_qk=c_qk, c_vo=c_vo,
                     b_vo=g("o_proj.weight").T.contiguous(), qk_tag=tag("kv_b_proj.qk_tag"),
                     vo_tag=tag("kv_b_proj.vo_tag"), qk_candidate_residuals=nan,
                     vo_candidate_residuals=nan, n_heads=H)
    return mla_fold_norm(w)


def rewrite_hf_checkpoint(state: dict, cfg: MLAConfig, *, dtype: torch.dtype | None = None,
                          force_first: bool = False) -> dict:
    """Rewrite every DeepseekV2Attention in a model state dict (keys ``...self_attn.``)
    to its BD form (offline, float64 prep, cast back to ``dtype`` or the stored dtype);
    all other entries pass through unchanged."""
    prefixes = sorted({k[:-len("kv_b_proj.weight")] for k in state if k.endswith("kv_b_proj.weight")})
    out = {k: v for k, v in state.items()
           if not any(k.startswith(p) and k[len(p):] in _HF_DENSE for p in prefixes)}
    for p in prefixes:
        dense = mla_from_hf(state, cfg, p)
        dt = dtype or dense.w_kvb.dtype
        bdw = mla_prepare(dense.to(dtype=torch.float64), force_first=force_first).to(dtype=dt)
        out.update(bd_mla_state_dict(bdw, p))
    return out


def block_flops(L: int, cfg: MLAConfig, n_heads: int | None = None, bd: bool = True,
                causal: bool = True) -> int:
    """Multiply-FLOPs of one block forward over L tokens for n_heads (default all)."""
    H = cfg.n_heads if n_heads is None else n_heads
    r = cfg.kv_lora_rank
    f = 2 * L * cfg.hidden * H * cfg.qk_head                         # q_proj
    f += 2 * L * cfg.hidden * (r + cfg.qk_rope)                       # kv_a (replicated)
    f += 2 * L * (r - (cfg.qk_nope if bd else 0)) * H * cfg.qk_nope   # K (nope)
    f += 2 * L * (r - (cfg.v_head if bd else 0)) * H * cfg.v_head     # V
    pairs = L * (L + 1) // 2 if causal else L * L
    f += 2 * pairs * H * (cfg.qk_head + cfg.v_head)                   # QK^T and PV
    f += 2 * L * H * cfg.v_head * cfg.hidden                          # o_proj
    return f
