"""DeepSeek-V2-Lite MLA block with the BD-rewritten kv_b_proj (BASELINE config 5).

CPU: the offline prep is algebraically exact — per head, the BD query/key pair
reproduces the dense no-RoPE scores and the BD value/output pair reproduces the dense
value-output product (float64, small geometry).  GPU: the BD block equals the dense
block end to end in float64 (exact kernel), and in FP16 (tensor-core kernel) within a
stated bound; head-sharded shards reassemble the full output.
"""

import numpy as np
import pytest
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import mla as M

SMALL = M.MLAConfig(hidden=96, n_heads=4, kv_lora_rank=48, qk_nope=16, qk_rope=8, v_head=16)


def _np(t):
    return t.detach().double().cpu().numpy()


def test_mla_prep_preserves_scores_and_value_output_products():
    w = M.gen_random_mla(0, SMALL)
    p = M.mla_prepare(w)
    cfg, H = SMALL, SMALL.n_heads
    rng = np.random.default_rng(1)
    hid = rng.standard_normal((7, cfg.hidden))
    ckv = rng.standard_normal((7, cfg.kv_lora_rank))
    wq, wkvb, wo = _np(w.w_q), _np(w.w_kvb), _np(w.w_o)
    wqb, cqk, cvo, bvo = _np(p.w_q), _np(p.c_qk), _np(p.c_vo), _np(p.b_vo)
    dn, dr, dv, r = cfg.qk_nope, cfg.qk_rope, cfg.v_head, cfg.kv_lora_rank
    s_k = slice(0, dn) if p.qk_tag is bd.Tag.FIRST else slice(r - dn, r)
    n_k = slice(dn, r) if p.qk_tag is bd.Tag.FIRST else slice(0, r - dn)
    s_v = slice(0, dv) if p.vo_tag is bd.Tag.FIRST else slice(r - dv, r)
    n_v = slice(dv, r) if p.vo_tag is bd.Tag.FIRST else slice(0, r - dv)
    for h in range(H):
        q0, k0 = h * (dn + dr), h * (dn + dv)
        dense = (hid @ wq[:, q0:q0 + dn]) @ (ckv @ wkvb[:, k0:k0 + dn]).T
        k_bd = ckv[:, s_k] + ckv[:, n_k] @ cqk[:, h * dn:(h + 1) * dn]
        scores = (hid @ wqb[:, q0:q0 + dn]) @ k_bd.T
        np.testing.assert_allclose(scores, dense, rtol=1e-9, atol=1e-9)
        # RoPE channels of the query weight are untouched
        np.testing.assert_array_equal(wqb[:, q0 + dn:q0 + dn + dr], wq[:, q0 + dn:q0 + dn + dr])
        vo_dense = (ckv @ wkvb[:, k0 + dn:k0 + dn + dv]) @ wo[h * dv:(h + 1) * dv]
        v_bd = ckv[:, s_v] + ckv[:, n_v] @ cvo[:, h * dv:(h + 1) * dv]
        np.testing.assert_allclose(v_bd @ bvo[h * dv:(h + 1) * dv], vo_dense, rtol=1e-9, atol=1e-9)
    # 25 % fewer kv_b_proj weights: 2 x 384 x 2048 vs 512 x 4096 at DSV2-Lite
    assert p.kv_param_count == 2 * (r - dn) * H * dn


def test_block_flops_bd_saving_matches_formula():
    cfg = M.DSV2_LITE
    dense = M.block_flops(32768, cfg, bd=False)
    bdf = M.block_flops(32768, cfg, bd=True)
    saved = 2 * 32768 * (128 * 16 * 128 + 128 * 16 * 128)
    assert dense - bdf == saved


@pytest.mark.gpu
def test_bd_mla_block_equals_dense_fp64_and_fp16(cuda):
    w = M.gen_random_mla(3, SMALL)
    p = M.mla_prepare(w)
    hid = torch.randn(40, SMALL.hidden, dtype=torch.float64, generator=torch.Generator().manual_seed(4))
    wd, pd, hd = w.to(cuda), p.to(cuda), hid.to(cuda)
    dense = M.mla_forward(hd, wd)
    got = M.bd_mla_forward(hd, pd)
    assert bd.max_relative_error(got, dense) <= 1e-10


@pytest.mark.gpu
def test_bd_mla_dsv2_lite_fp16_vs_fp64_dense(cuda):
    """Full DeepSeek-V2-Lite geometry, 2048 tokens, FP16 on the tcgen05 kernel.  Bound:
    random-init BD amplifies FP16 rounding by cond(M_S); the measured
    error is printed and bounded loosely; the dense FP16 block is the like-for-like."""
    w = M.gen_random_mla(5)
    p = M.mla_prepare(w)
    g = torch.Generator().manual_seed(6)
    hid = torch.randn(2048, 2048, generator=g, dtype=torch.float64)
    ref = M.mla_forward(hid.to(cuda), w.to(cuda))
    got16 = M.bd_mla_forward(hid.half().to(cuda), p.to(cuda, torch.float16))
    dense16 = M.mla_forward(hid.half().to(cuda), w.to(cuda, torch.float16))
    e_bd = bd.max_relative_error(got16, ref)
    e_dense = bd.max_relative_error(dense16, ref)
    print(f"DSV2-Lite block 2048 tok FP16 max-rel vs FP64 dense: BD {e_bd:.3g}, dense {e_dense:.3g}")
    assert torch.isfinite(got16).all()
    assert e_bd <= 0.1  # measured 2.95e-2 (dense FP16: 6.6e-4), B200 round 1


@pytest.mark.gpu
def test_head_sharded_mla_partials_sum_to_the_full_block(cuda):
    """cfg5's multi-GPU split on one device: each head shard's partial block output
    (its q columns, C columns, B_vo rows; kv_a replicated) sums to the unsharded block —
    what the all_reduce in bd_mla_forward computes across ranks."""
    w = M.gen_random_mla(8, SMALL)
    p = M.mla_prepare(w).to(cuda)
    hid = torch.randn(33, SMALL.hidden, dtype=torch.float64,
                      generator=torch.Generator().manual_seed(9)).to(cuda)
    full = M.bd_mla_forward(hid, p)
    for world in (2, 4):
        parts = [M.bd_mla_forward(hid, M.shard_bd_mla(p, world, r)) for r in range(world)]
        assert bd.max_relative_error(sum(parts), full) <= 1e-12


def _hf_attention(seed=11):
    """A small transformers DeepseekV2Attention (q-LoRA-free, like DSV2-Lite) with every
    parameter random (including the kv_a RMSNorm weight), float64, SDPA causal."""
    pytest.importorskip("transformers")
    from transformers.models.deepseek_v2 import modeling_deepseek_v2 as HF
    from transformers.models.deepseek_v2.configuration_deepseek_v2 import DeepseekV2Config
    hcfg = DeepseekV2Config(hidden_size=96, num_attention_heads=4, num_key_value_heads=4,
                            kv_lora_rank=48, q_lora_rank=None, qk_nope_head_dim=16,
                            qk_rope_head_dim=8, v_head_dim=16, max_position_embeddings=256)
    hcfg._attn_implementation = "sdpa"
    torch.manual_seed(seed)
    att = HF.DeepseekV2Attention(hcfg, 0).double()
    with torch.no_grad():
        for name, prm in att.named_parameters():
            prm.copy_(torch.randn_like(prm) / (prm.shape[-1] ** 0.5 if prm.dim() == 2 else 1.0)
                      + (1.0 if prm.dim() == 1 else 0.0))
    rot = HF.DeepseekV2RotaryEmbedding(hcfg)
    return hcfg, att, rot


def _hf_forward(att, rot, hid):
    pe = rot(hid[None], torch.arange(hid.shape[0])[None])
    with torch.no_grad():
        return att(hid[None], attention_mask=None, position_embeddings=pe)[0][0]


def test_hf_deepseek_v2_attention_equals_mla_forward():
    """The checkpoint importer and the block forward against transformers' own
    DeepseekV2Attention (same weights, float64 except the float32 RoPE / RMSNorm both
    implementations use)."""
    hcfg, att, rot = _hf_attention()
    cfg = M.mla_config_from_hf(hcfg)
    assert cfg == M.MLAConfig(hidden=96, n_heads=4, kv_lora_rank=48, qk_nope=16, qk_rope=8,
                              v_head=16, rope_interleaved=True)
    hid = torch.randn(37, 96, dtype=torch.float64, generator=torch.Generator().manual_seed(2))
    ref = _hf_forward(att, rot, hid)
    got = M.mla_forward(hid, M.mla_from_hf(att.state_dict(), cfg))
    assert bd.max_relative_error(got, ref) <= 1e-6  # measured 3.9e-8 (rotate-half RoPE: 0.29)


def test_rewrite_hf_checkpoint_replaces_attention_and_round_trips():
    hcfg, att, rot = _hf_attention(12)
    cfg = M.mla_config_from_hf(hcfg)
    sd = {f"model.layers.0.self_attn.{k}": v for k, v in att.state_dict().items()}
    sd["model.layers.0.mlp.up_proj.weight"] = torch.randn(8, 96, dtype=torch.float64)
    new = M.rewrite_hf_checkpoint(sd, cfg)
    pre = "model.layers.0.self_attn."
    assert pre + "kv_b_proj.weight" not in new
    assert torch.equal(new["model.layers.0.mlp.up_proj.weight"], sd["model.layers.0.mlp.up_proj.weight"])
    assert new[pre + "kv_b_proj.c_qk"].shape == (48 - 16, 4 * 16)
    # 25 % fewer kv_b weights at d_h = r / 4 (here 2 x 32 x 64 vs 48 x 128)
    n_new = new[pre + "kv_b_proj.c_qk"].numel() + new[pre + "kv_b_proj.c_vo"].numel()
    assert n_new == 2 * 32 * 64 and sd[pre + "kv_b_proj.weight"].numel() == 48 * 128
    back = M.bd_mla_from_state_dict(new, cfg, pre)
    want = M.mla_prepare(M.mla_from_hf(att.state_dict(), cfg))
    for k in ("w_q", "w_kva", "kva_norm", "c_qk", "c_vo", "b_vo"):
        assert torch.equal(getattr(back, k), getattr(want, k)), k
    assert (back.qk_tag, back.vo_tag, back.n_heads) == (want.qk_tag, want.vo_tag, 4)


@pytest.mark.gpu
def test_bd_mla_on_rewritten_hf_checkpoint_matches_hf_attention(cuda):
    """End to end: transformers DeepseekV2Attention → rewritten BD checkpoint → the BD
    block on the GPU (float64: exact kernel) reproduces the HF module's output."""
    hcfg, att, rot = _hf_attention(13)
    cfg = M.mla_config_from_hf(hcfg)
    new = M.rewrite_hf_checkpoint(att.state_dict(), cfg)
    w = M.bd_mla_from_state_dict(new, cfg).to(cuda)
    hid = torch.randn(45, 96, dtype=torch.float64, generator=torch.Generator().manual_seed(3))
    ref = _hf_forward(att, rot, hid)
    got = M.bd_mla_forward(hid.to(cuda), w).cpu()
    assert bd.max_relative_error(got, ref) <= 1e-6


def test_fold_rmsnorm_is_the_exact_algebra():
    """CPU: folding the RMSNorm weight into C reproduces the projection of the normalised
    latent — r * (x[:, ~S] (diag(g) C) + g_S x[:, S]) == K'(x * r * g) in float64."""
    rng = np.random.default_rng(5)
    L, d_h, n = 9, 16, 3
    d = 48
    x = torch.from_numpy(rng.standard_normal((L, d)))
    gamma = torch.from_numpy(0.5 + rng.random(d))
    c = torch.from_numpy(rng.standard_normal((d - d_h, n * d_h)))
    r = torch.rsqrt(x.pow(2).mean(1, keepdim=True) + 1e-6)
    xn = x * r * gamma
    for tag in bd.Tag:
        cg, rg = bd.fold_rmsnorm(c, gamma, d_h, tag)
        mul, rep = bd.tag_offsets(d, d_h, tag)
        K = d - d_h
        want = xn[:, rep:rep + d_h].repeat(1, n) + xn[:, mul:mul + K] @ c
        got = r * (x[:, mul:mul + K] @ cg + (rg.double() * x[:, rep:rep + d_h]).repeat(1, n))
        # rep_gamma is float32 by contract: 1e-7-level relative rounding on the rep term
        np.testing.assert_allclose(got.numpy(), want.numpy(), rtol=1e-5, atol=1e-7)
    assert rg.dtype == torch.float32 and cg.dtype == c.dtype
    with pytest.raises(bd.ShapeError):
        bd.fold_rmsnorm(c, gamma[:-1], d_h, bd.Tag.FIRST)


def test_mla_prepare_attaches_the_norm_fold():
    w = M.gen_random_mla(21, SMALL)
    p = M.mla_prepare(w)
    assert p.norm_fold is not None
    cq, cv, gq, gv = p.norm_fold
    assert cq.shape == p.c_qk.shape and cv.shape == p.c_vo.shape
    assert gq.shape == (SMALL.qk_nope,) and gv.shape == (SMALL.v_head,)
    shard = M.shard_bd_mla(p, 2, 1)
    assert shard.norm_fold[0].shape == (p.c_qk.shape[0], p.c_qk.shape[1] // 2)
