"""Parity at BASELINE.json's FULL sizes (configs 2-5), through the C-ABI library.

* cfg2 (DSV2-Lite kv_b_proj, 8192 tokens, K' and V' in one launch): EVERY output element
  against the FP64 C oracle (oracle/bd_oracle.c, the restatement of ref
  attention.py:249-270) under the elementwise bound of test_kv_proj_gpu.py, FP16 and BF16.
* cfg3 (Llama-2-7B K/V, 65536 tokens, BF16) and cfg4 (BD low-rank layer, 32768 tokens,
  FP16): one row from EVERY 256-row block (the row's offset inside its block walks
  through all 256 positions across the blocks, so both CTAs of every pair and every
  TMEM lane quadrant are hit), all columns of it — every tile of the round-robin
  schedule (kv_proj_tc.cu, kRR) is checked against the FP64 oracle.
* cfg5 (DSV2-Lite MLA block, 32768-token causal prefill, FP16): the BD block's output
  max-abs error against a float64 dense block, with the dense FP16 block's error beside
  it — the north star's "attention-output max-abs error bound stated per config"
  (cfg1's FP32 bound, 1e-5 max-abs, is in test_callers_gpu.py).
"""

import math

import numpy as np
import pytest
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import mla as M
from oracle import oracle as O
from test_kv_proj_gpu import assert_tc_close

pytestmark = pytest.mark.gpu


def every_block_rows(L: int, block: int = 256) -> torch.Tensor:
    """One row per `block`-row block; offset (37 b) mod block walks all positions."""
    nb = (L + block - 1) // block
    rows = [min(L - 1, b * block + (37 * b) % block) for b in range(nb)]
    return torch.tensor(sorted(set(rows)))


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_cfg2_full_output_vs_fp64_oracle(dtype, cuda):
    L, d, d_h, n = 8192, 512, 128, 16
    g = torch.Generator().manual_seed(2)
    x = torch.randn(L, d, generator=g).to(dtype).to(cuda)
    ck = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    cv = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    k, v = bd.fused_kv_proj_grouped(x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)])
    assert_tc_close(k, x, ck, d_h, n, bd.Tag.FIRST)   # all 8192 x 2048 elements
    assert_tc_close(v, x, cv, d_h, n, bd.Tag.LAST)


def test_cfg3_llama_every_tile_vs_fp64_oracle(cuda):
    """65536 tokens x (32 heads x 128), d = 4096 (K = 3968 streams through the A ring,
    round-robin tile schedule), BF16, K' and V' in one launch."""
    L, d, d_h, n = 65536, 4096, 128, 32
    g = torch.Generator(device=cuda).manual_seed(33)
    x = torch.randn(L, d, generator=g, device=cuda).bfloat16()
    ck = (torch.randn(d - d_h, n * d_h, generator=g, device=cuda) / 64).bfloat16()
    cv = (torch.randn(d - d_h, n * d_h, generator=g, device=cuda) / 64).bfloat16()
    k, v = bd.fused_kv_proj_grouped(x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)])
    rows = every_block_rows(L).to(cuda)
    assert rows.numel() == L // 256
    assert_tc_close(k, x, ck, d_h, n, bd.Tag.FIRST, rows=rows)
    assert_tc_close(v, x, cv, d_h, n, bd.Tag.LAST, rows=rows)
    # the per-element bound above already holds on every sampled element; also: no
    # non-finite value anywhere in the 2 x 512 MiB output
    assert bool(torch.isfinite(k).all()) and bool(torch.isfinite(v).all())


def test_cfg4_lowrank_every_tile_vs_fp64(cuda):
    """BD low-rank layer W = A B (4096 x 4096, rank 1024) at 32768 tokens, FP16: both
    GEMMs (h = x B into y[:, S]; h C into the rest) on every 256-row block.  The oracle
    rounds h to FP16 like the kernel (h is stored in y and re-read as GEMM 2's A), so
    each GEMM is held to its own elementwise bound."""
    din, r, dout, L = 4096, 1024, 4096, 32768
    g = torch.Generator(device=cuda).manual_seed(7)
    basis = (torch.randn(din, r, generator=g, device=cuda) / 64).half()
    coeff = (torch.randn(r, dout - r, generator=g, device=cuda) / 32).half()
    fac = bd.BDFactors(axis=bd.Axis.COLUMN, tag=bd.Tag.LAST, basis=basis.double().cpu().numpy(),
                       coeff=coeff.double().cpu().numpy(), orig_rows=din, orig_cols=dout, rank=r,
                       residual=0.0, rank_deficient=False)
    layer = bd.BDLinearLayer(fac, basis, coeff)
    x = torch.randn(L, din, generator=g, device=cuda).half()
    y = bd.bd_linear_forward(x, layer)
    rows = every_block_rows(L).to(cuda)
    assert rows.numel() == L // 256
    ys = y[rows].double().cpu().numpy()
    xs = x[rows].double().cpu().numpy()
    B = basis.double().cpu().numpy()
    C = coeff.double().cpu().numpy()
    u, u32 = 2.0 ** -11, 2.0 ** -24
    h_got = ys[:, dout - r:]                       # LAST: y = [h C, h]
    h_ref = xs @ B
    bound_h = 2 * u * np.abs(h_ref) + 2 * din * u32 * (np.abs(xs) @ np.abs(B)) + 1e-30
    assert float((np.abs(h_got - h_ref) / bound_h).max()) <= 1.0
    hc_ref = h_got @ C                              # GEMM 2 on the kernel's own FP16 h
    bound_hc = 2 * u * np.abs(hc_ref) + 2 * r * u32 * (np.abs(h_got) @ np.abs(C)) + 1e-30
    assert float((np.abs(ys[:, :dout - r] - hc_ref) / bound_hc).max()) <= 1.0
    assert bool(torch.isfinite(y).all())


# ------------------------------------------------------------------ cfg5 block, 32k
def _dense_block_fp64_chunked(hid: torch.Tensor, w: M.MLAWeights, chunk: int = 2048):
    """mla_forward in float64 with the causal attention evaluated per head and per query
    chunk (the math SDPA would need 32768^2 x 16 x 8 B = 137 GB at once)."""
    cfg, H = w.cfg, w.cfg.n_heads
    L = hid.shape[0]
    q_nope, q_pe = M._split_q(hid @ w.w_q, H, cfg)
    c_kv, k_pe = M._latent(hid, w.w_kva, w.kva_norm, cfg)
    kvb = (c_kv @ w.w_kvb).view(L, H, cfg.qk_nope + cfg.v_head)
    rope = lambda t: M._rope(t, cfg.rope_theta, cfg.rope_interleaved)  # noqa: E731
    q = torch.cat([q_nope.view(L, H, cfg.qk_nope), rope(q_pe).view(L, H, cfg.qk_rope)], -1)
    k = torch.cat([kvb[..., :cfg.qk_nope],
                   rope(k_pe).view(L, 1, cfg.qk_rope).expand(L, H, cfg.qk_rope)], -1)
    v = kvb[..., cfg.qk_nope:]
    scale = 1.0 / math.sqrt(cfg.qk_head)
    o = torch.empty(L, H, cfg.v_head, dtype=hid.dtype, device=hid.device)
    for h in range(H):
        qh, kh, vh = q[:, h], k[:, h], v[:, h]
        for q0 in range(0, L, chunk):
            q1 = min(L, q0 + chunk)
            s = (qh[q0:q1] @ kh[:q1].T) * scale
            mask = torch.arange(q1, device=hid.device)[None, :] > torch.arange(q0, q1, device=hid.device)[:, None]
            s.masked_fill_(mask, float("-inf"))
            o[q0:q1, h] = torch.softmax(s, dim=-1) @ vh[:q1]
    return o.reshape(L, H * cfg.v_head) @ w.w_o


# Stated bounds (north star: "attention-output max-abs error bound stated per config"),
# cfg5 = DeepSeek-V2-Lite MLA block, 32768-token causal prefill, FP16, x_hidden ~ N(0, 1),
# BD block output vs the float64 dense block:
#   * random-init weights (N(0,1)/sqrt(fan_in)):   max-abs <= CFG5_MAXABS_RANDOM
#     (measured 0.199 on a B200, |out|max 3.79; the dense FP16 block: 2.3e-3).  Random
#     Gaussian 128 x 128 basis blocks M_S have cond ~ 450-5000 and K' = K M_S^-1 carries
#     FP16 rounding amplified by it — a property of BD on random weights,
#     not of the kernel (K'/V' themselves meet the FP16 elementwise bound, cfg2 above);
#   * well-conditioned basis blocks (orthogonal M_S, as trained weights approach — the
#     paper's DSV2-Lite QK NMSE is 2.4e-4):  max-abs <= CFG5_MAXABS_WELL
#     (measured 1.46e-3, |out|max 2.6 — BELOW the dense FP16 block's 1.61e-3).
CFG5_MAXABS_RANDOM = 0.3
CFG5_MAXABS_WELL = 4.0e-3


def _orthogonal_basis_blocks(w: M.MLAWeights, seed: int) -> M.MLAWeights:
    """Replace, per head, the kv_b_proj rows of both candidate bases (latent dims
    [0, 128) and [384, 512)) of its k_nope and v columns by scaled random orthogonal
    matrices: cond(M_S) = 1 whichever tag the prep selects."""
    cfg = w.cfg
    g = torch.Generator().manual_seed(seed)
    wk = w.w_kvb.clone()
    r, dn, dv = cfg.kv_lora_rank, cfg.qk_nope, cfg.v_head
    for h in range(cfg.n_heads):
        c0 = h * (dn + dv)
        for rows in (slice(0, dn), slice(r - dn, r)):
            for cols, width in ((slice(c0, c0 + dn), dn), (slice(c0 + dn, c0 + dn + dv), dv)):
                q, _ = torch.linalg.qr(torch.randn(width, width, generator=g, dtype=torch.float64))
                wk[rows, cols] = q / math.sqrt(r)
    return M.MLAWeights(cfg=cfg, w_q=w.w_q, w_kva=w.w_kva, kva_norm=w.kva_norm, w_kvb=wk,
                        w_o=w.w_o)


_CFG5_REF: dict = {}


def _cfg5_reference(weights: str, cuda):
    """(weights, prepared BD weights, FP64 dense output, FP16 dense error) at 32k tokens,
    computed once per weight set (the FP64 reference is the expensive part)."""
    if weights not in _CFG5_REF:
        w = M.gen_random_mla(5)
        if weights == "well_conditioned":
            w = _orthogonal_basis_blocks(w, 55)
        p = M.mla_prepare(w)
        L = 32768
        g = torch.Generator(device=cuda).manual_seed(6)
        hid64 = torch.randn(L, w.cfg.hidden, generator=g, device=cuda, dtype=torch.float64)
        ref = _dense_block_fp64_chunked(hid64, w.to(cuda))
        hid16 = hid64.half()
        dense16 = M.mla_forward(hid16, w.to(cuda, torch.float16))
        e_dense = float((dense16.double() - ref).abs().max())
        _CFG5_REF[weights] = (w, p, hid16, ref, e_dense)
    return _CFG5_REF[weights]


@pytest.mark.parametrize("attention", ["sdpa", "bd"])
@pytest.mark.parametrize("weights", ["random", "well_conditioned"])
def test_cfg5_block_32k_fp16_max_abs_bound(weights, attention, cuda):
    """N1 row: the stated max-abs bound holds for the BD block with either attention core
    — cuDNN SDPA on the BD kernel's head-major K'/V', or the tcgen05 MLA attention kernel
    reading them in place (attention='bd', csrc/mla_attn.cu)."""
    w, p, hid16, ref, e_dense = _cfg5_reference(weights, cuda)
    got16 = M.bd_mla_forward(hid16, p.to(cuda, torch.float16), attention=attention)
    assert bool(torch.isfinite(got16).all())
    e_bd = float((got16.double() - ref).abs().max())
    peak = float(ref.abs().max())
    print(f"cfg5 32k FP16 ({weights}, attention={attention}) max-abs vs FP64 dense: BD {e_bd:.4g}, "
          f"dense FP16 {e_dense:.4g}, |out|max {peak:.4g}, tags {p.qk_tag.value}/{p.vo_tag.value}")
    bound = CFG5_MAXABS_RANDOM if weights == "random" else CFG5_MAXABS_WELL
    assert e_bd <= bound, (e_bd, e_dense, peak)
    assert e_dense <= bound
