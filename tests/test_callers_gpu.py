"""GPU parity of the projection's callers: bda_forward / attention_scores (ref
attention.py:298-325), the BD low-rank layer (ref linear.py:101-108) and the plain
product (ref tensor.py:189-213), against the reference's own outputs (tests/golden)
and the CPU oracle.

Tolerances:
  * exact kernel paths (float32/float64 bd_matmul, bd_linear_forward): bit-identical;
  * bda_forward float64 vs the reference mha_forward output: <= 1e-10 (ref verify.py:23);
  * K'/V' inside bda_forward (the projection itself): bit-identical in float32 — the
    north star's "1e-5 relative for FP32" met with margin;
  * bda_forward float32 attention output (cfg1, P64 prep) vs the reference's own
    bda_forward: max-abs <= 1e-5 (|out| <= 0.6), max-rel <= 2.5e-5.  Every product
    runs in the reference's order; the residue is exp/row-sum rounding in softmax
    (numpy SIMD exp + pairwise sum vs CUDA), amplified by cond(M_S) through V' and
    B_vo;
  * float16 BD layer: <= 2e-3 max-rel vs the float64 oracle on the same rounded inputs.
"""

import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import _native as N
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_bda_forward_cfg1_fp32_matches_reference_output(cuda):
    meta = json.loads((GOLDEN / "cfg1.json").read_text())
    g = np.load(GOLDEN / "cfg1.npz")
    w = bd.gen_random_mha(bd.Rng(7), 512, 64, 8, torch.float32)
    p = bd.bda_prepare(w, prepare_in_p64=True).to(cuda)
    x = bd.rand_gaussian(bd.Rng(8), 256, 512, torch.float32, cuda)
    out = bd.bda_forward(x, p)
    ref = torch.from_numpy(g["bda_out"])
    assert float((out.cpu() - ref).abs().max()) <= 1e-5
    assert bd.max_relative_error(out, ref) <= 2.5e-5
    # and against the reference's dense MHA output: the BDA-vs-MHA error the reference
    # itself shows for this model (2.0e-5, cfg1.json) plus float32 rounding
    err = bd.max_relative_error(out, torch.from_numpy(g["mha_out"]))
    assert err <= meta["bda_vs_mha_max_rel"] + 1e-5
    # K' and V' inside bda_forward come from one grouped launch; check them bit-exactly
    k, v = bd.fused_kv_proj_grouped(x, [(p.c_qk, 64, 8, p.qk_tag), (p.c_vo, 64, 8, p.vo_tag)])
    np.testing.assert_array_equal(k.cpu().numpy(), g["k_out"])
    np.testing.assert_array_equal(v.cpu().numpy(), g["v_out"])


@pytest.mark.parametrize("shape", [(32, 8, 4, 10), (48, 12, 3, 7), (24, 4, 5, 1)])
def test_bda_forward_fp64_equivalence(shape, cuda):
    d, d_h, n, L = shape
    s = bd.equivalence_check(bd.Rng(123), d, d_h, n, L, torch.float64, trials=4, device=cuda)
    assert s.ok, s


def test_bda_forward_fp32_equivalence_p32_threshold(cuda):
    s = bd.equivalence_check(bd.Rng(5), 64, 16, 4, 33, torch.float32, trials=3, device=cuda)
    assert s.ok, s


def test_attention_scores_preserved_per_head(cuda):
    w = bd.gen_random_mha(bd.Rng(9), 48, 8, 6, torch.float64, cuda)
    p = bd.bda_prepare(w)
    x = bd.rand_gaussian(bd.Rng(10), 20, 48, torch.float64, cuda)
    for h in range(6):
        a = bd.attention_scores(x, w, h)
        b = bd.attention_scores(x, p, h)
        assert bd.max_relative_error(b, a) <= 1e-10
    with pytest.raises(IndexError):
        bd.attention_scores(x, p, 6)


def test_bda_forward_causal_and_fp16(cuda):
    w = bd.gen_random_mha(bd.Rng(2), 256, 64, 4, torch.float64)
    p = bd.bda_prepare(w)
    x64 = bd.rand_gaussian(bd.Rng(3), 128, 256, torch.float64, cuda)
    ref = bd.mha_forward(x64, w.to(cuda), causal=True)
    got64 = bd.bda_forward(x64, p.to(cuda), causal=True)
    assert bd.max_relative_error(got64, ref) <= 1e-10
    # FP16: BD amplifies rounding by cond(M_S) — bound stated per config
    got16 = bd.bda_forward(x64.half(), p.to(cuda).cast(torch.float16), causal=True)
    err16 = bd.max_relative_error(got16, ref)
    print("fp16 bda vs fp64 mha max-rel", err16)
    assert err16 <= 3e-2  # measured 9.0e-3 (B200, round 1)


def test_input_validation(cuda):
    w = bd.gen_random_mha(bd.Rng(1), 16, 4, 2, torch.float32, cuda)
    p = bd.bda_prepare(w)
    with pytest.raises(bd.ShapeError):
        bd.bda_forward(torch.zeros(3, 15, device=cuda), p)
    with pytest.raises(bd.PrecisionError):
        bd.bda_forward(torch.zeros(3, 16, device=cuda, dtype=torch.float64), p)


# ------------------------------------------------------------------ BD low-rank layer
def test_bd_linear_forward_bit_exact_vs_reference(cuda):
    meta = json.loads((GOLDEN / "linear_small.json").read_text())
    g = np.load(GOLDEN / "linear_small.npz")
    for i, m in enumerate(meta):
        layer = bd.LowRankLayer(u=torch.from_numpy(g[f"u{i}"]), v=torch.from_numpy(g[f"v{i}"]))
        conv = bd.bd_linear_from_lowrank(layer, device=cuda)
        y = bd.bd_linear_forward(torch.from_numpy(g[f"x{i}"]).to(cuda), conv)
        np.testing.assert_array_equal(y.cpu().numpy(), g[f"y{i}"], err_msg=str(m))


def test_bd_linear_fp16_tensor_cores(cuda):
    d_in, d_out, r, L = 512, 768, 128, 300
    rng = bd.Rng(4)
    layer = bd.LowRankLayer(u=bd.rand_gaussian(rng, d_in, r) / 8,
                            v=bd.rand_gaussian(rng, d_out, r) / 8)
    conv = bd.bd_linear_from_lowrank(layer, device=cuda, dtype=torch.float16)
    x = bd.rand_gaussian(rng, L, d_in, torch.float16, cuda)
    y = bd.bd_linear_forward(x, conv, check_finite=True)
    # oracle on identical rounded operands, with h rounded to FP16 like the kernel's
    xb, B, C = (t.cpu().double().numpy() for t in (x, conv.basis, conv.coeff))
    h = (xb @ B).astype(np.float16).astype(np.float64)
    hc = h @ C
    want = np.concatenate([h, hc], 1) if conv.tag is bd.Tag.FIRST else np.concatenate([hc, h], 1)
    assert O.max_relative_error(y.cpu().double().numpy(), want) <= 2e-3
    # against the low-rank layer it replaces: same function, different rounding
    ref = (x.double() @ layer.u.to(cuda)) @ layer.v.to(cuda).T
    assert bd.max_relative_error(y, ref) <= 2e-2


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_matmul_exact_equals_reference_fixed_order(dtype, cuda):
    rng = O.Rng(8)
    a = O.rand_gaussian(rng, 70, 45, dtype)
    b = O.rand_gaussian(rng, 45, 33, dtype)
    got = bd.matmul(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda))
    np.testing.assert_array_equal(got.cpu().numpy(), O.matmul_ref(a, b))


def test_matmul_fp16_and_launch_count(cuda):
    a = torch.randn(1000, 264, device=cuda).half()
    b = torch.randn(264, 200, device=cuda).half()
    before = N.launch_count()
    got = bd.matmul(a, b)
    torch.cuda.synchronize()
    assert N.launch_count() == before + 1
    ref = a.double() @ b.double()
    assert bd.max_relative_error(got, ref) <= 1e-3


def test_bd_linear_cfg4_geometry_fp16(cuda):
    """BASELINE config 4 layer (4096 -> 1024 -> 4096), 256 tokens: both GEMMs stream K
    (4096 and 1024) through the kernel; oracle with h rounded like the kernel."""
    din, r, dout, L = 4096, 1024, 4096, 256
    g = torch.Generator().manual_seed(7)
    basis = (torch.randn(din, r, generator=g) / 64).half()
    coeff = (torch.randn(r, dout - r, generator=g) / 32).half()
    fac = bd.BDFactors(axis=bd.Axis.COLUMN, tag=bd.Tag.LAST, basis=basis.double().numpy(),
                       coeff=coeff.double().numpy(), orig_rows=din, orig_cols=dout, rank=r,
                       residual=0.0, rank_deficient=False)
    layer = bd.BDLinearLayer(fac, basis.to(cuda), coeff.to(cuda))
    x = torch.randn(L, din, generator=g).half().to(cuda)
    y = bd.bd_linear_forward(x, layer, check_finite=True)
    h = (x.double() @ basis.to(cuda).double()).half().double()
    want = torch.cat([h @ coeff.to(cuda).double(), h], dim=1)  # LAST: [h C, h]
    assert bd.max_relative_error(y, want) <= 2e-3


def test_head_sharded_bda_partials_sum_to_the_full_block(cuda):
    """parallel.sharded_bda_forward on one device: the shards' partial outputs (no
    process group -> no all_reduce) sum to the unsharded bda_forward."""
    from paper_2510_01718_b200 import parallel as P
    w = bd.gen_random_mha(bd.Rng(12), 48, 8, 6, torch.float64)
    prepared = bd.bda_prepare(w).to(cuda)
    x = bd.rand_gaussian(bd.Rng(13), 25, 48, torch.float64, cuda)
    full = bd.bda_forward(x, prepared, causal=True)
    for world in (2, 3, 6):
        parts = [P.sharded_bda_forward(x, P.shard_bda_weights(prepared, world, r), causal=True)
                 for r in range(world)]
        assert bd.max_relative_error(sum(parts), full) <= 1e-12
