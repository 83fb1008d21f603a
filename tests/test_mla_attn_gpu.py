"""The tcgen05 MLA attention kernel (csrc/mla_attn.cu, C ABI ``bd_mla_attention``) that
consumes the BD projection's outputs in place.

Oracle: the same attention in float64 (torch on the GPU) on the kernel's exact 16-bit
inputs.  Bound: the kernel's max-abs error must stay within 2x the error of torch's own
FP16/BF16 SDPA (cuDNN / flash) on the same inputs, plus a small absolute floor — i.e.
"within 16-bit rounding", measured like for like.  Block level: the BD MLA block with
this attention against the float64 dense block, beside the SDPA-based BD block.
"""

import math

import pytest
import torch

import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import mla as M

pytestmark = pytest.mark.gpu


def _inputs(L, H, dtype, seed, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    q = torch.randn(L, H, 192, device=dev, generator=g).to(dtype)
    k = torch.randn(H, L, 128, device=dev, generator=g).to(dtype)
    kpe = torch.randn(L, 64, device=dev, generator=g).to(dtype)
    v = torch.randn(H, L, 128, device=dev, generator=g).to(dtype)
    return q, k, kpe, v


def _ref64(q, k, kpe, v, scale, causal):
    L, H, _ = q.shape
    qd, kd, pd, vd = (t.double() for t in (q, k, kpe, v))
    out = torch.empty(L, H, 128, dtype=torch.float64, device=q.device)
    for h in range(H):
        s = (qd[:, h, :128] @ kd[h].T + qd[:, h, 128:] @ pd.T) * scale
        if causal:
            s.masked_fill_(torch.ones(L, L, dtype=torch.bool, device=q.device).triu(1), float("-inf"))
        out[:, h] = torch.softmax(s, -1) @ vd[h]
    return out


def _sdpa16(q, k, kpe, v, scale, causal):
    L, H, _ = q.shape
    kk = torch.cat([k, kpe[None].expand(H, L, 64)], -1)
    o = torch.nn.functional.scaled_dot_product_attention(
        q.transpose(0, 1)[None], kk[None], v[None], is_causal=causal, scale=scale)
    return o[0].transpose(0, 1)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("L,H,causal", [(128, 1, True), (300, 3, True), (1000, 2, True),
                                        (257, 2, False), (4096, 2, True)])
def test_mla_attention_matches_fp64(dtype, L, H, causal, cuda):
    q, k, kpe, v = _inputs(L, H, dtype, L + H, cuda)
    scale = 1.0 / math.sqrt(192)
    ours = M.mla_attention(q, k, kpe, v, scale=scale, causal=causal)
    ref = _ref64(q, k, kpe, v, scale, causal)
    lib = _sdpa16(q, k, kpe, v, scale, causal)
    e_ours = float((ours.double() - ref).abs().max())
    e_lib = float((lib.double() - ref).abs().max())
    print(f"L={L} H={H} causal={causal} {dtype}: max-abs ours {e_ours:.3g}, torch SDPA {e_lib:.3g}")
    assert torch.isfinite(ours).all()
    assert e_ours <= 2.0 * e_lib + (2e-3 if dtype == torch.float16 else 1.6e-2)


def test_mla_attention_strided_views_and_out(cuda):
    """q as the q-projection's [L, H*192] output viewed [L, H, 192]; head slices of the
    K'/V' buffers and of the output (the head-group path of bd_mla_forward)."""
    L, H = 515, 4
    q, k, kpe, v = _inputs(L, H, torch.float16, 3, cuda)
    scale = 0.07
    full = M.mla_attention(q, k, kpe, v, scale=scale)
    out = torch.full((L, H, 128), 7.0, dtype=torch.float16, device=cuda)
    for h0 in (0, 2):
        M.mla_attention(q[:, h0:h0 + 2], k[h0:h0 + 2], kpe, v[h0:h0 + 2], scale=scale,
                        out=out[:, h0:h0 + 2])
    torch.testing.assert_close(out, full, rtol=0, atol=0)


def test_mla_attention_validation(cuda):
    q, k, kpe, v = _inputs(64, 2, torch.float16, 1, cuda)
    with pytest.raises(bd.ShapeError):
        M.mla_attention(q[..., :128], k, kpe, v, scale=0.1)
    with pytest.raises(bd.PrecisionError):
        M.mla_attention(q.float(), k.float(), kpe.float(), v.float(), scale=0.1)
    with pytest.raises(ValueError):
        M.mla_attention(q, k, kpe, v, scale=-1.0)


@pytest.mark.parametrize("head_group", [None, 2])
def test_bd_mla_block_with_bd_attention(head_group, cuda):
    """DeepSeek-V2-Lite block, 2048 tokens, FP16: the BD block with the tcgen05 attention
    (whole, or in head groups through the L2 ring) vs the float64 dense block, beside the
    BD block with SDPA — same inputs, same weights."""
    w = M.gen_random_mla(5)
    p = M.mla_prepare(w)
    g = torch.Generator().manual_seed(6)
    hid = torch.randn(2048, 2048, generator=g, dtype=torch.float64)
    ref = M.mla_forward(hid.to(cuda), w.to(cuda))
    p16 = p.to(cuda, torch.float16)
    h16 = hid.half().to(cuda)
    ours = M.bd_mla_forward(h16, p16, attention="bd", head_group=head_group)
    sdpa = M.bd_mla_forward(h16, p16, attention="sdpa")
    e_ours = float((ours.double() - ref).abs().max())
    e_sdpa = float((sdpa.double() - ref).abs().max())
    print(f"block 2048 tok FP16 max-abs vs FP64 dense: bd-attention {e_ours:.4g}, sdpa {e_sdpa:.4g}")
    assert torch.isfinite(ours).all()
    assert e_ours <= 1.5 * e_sdpa + 1e-3
