"""GPU parity of the BD K/V projection against the reference (golden vectors) and the
CPU oracle.  All calls go through the C-ABI library (libbd_kvproj.so).

Tolerances:
  * float32 / float64 (exact kernel): bit-identical to the reference.
  * float16 (tensor cores): max_relative_error <= 1e-3 against the FP64 oracle on the
    same rounded inputs, plus the elementwise bound
    |out - ref| <= 2 u16 |ref| + 2 K u32 sum_k |x||c| + u16 * |x_rep|.
  * bfloat16: max_relative_error <= 8e-3 and the same elementwise bound with u_bf16.
"""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import _native as N
from oracle import oracle as O

pytestmark = pytest.mark.gpu

U16 = {torch.float16: 2.0 ** -11, torch.bfloat16: 2.0 ** -8}
MAXREL = {torch.float16: 1e-3, torch.bfloat16: 8e-3}
U32 = 2.0 ** -24


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def to_np64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def assert_tc_close(got: torch.Tensor, x: torch.Tensor, c: torch.Tensor, d_h, n, tag, rows=None):
    """Compare a 16-bit kernel output with the FP64 oracle on identical rounded inputs."""
    xs = x if rows is None else x[rows]
    g = got if rows is None else got[rows]
    x64, c64 = to_np64(xs), to_np64(c)
    ref = O.fused_kv_proj_ref(x64, c64, d_h, n, tag.value, threads=O.default_threads())
    mul_base, rep_base = bd.tag_offsets(x64.shape[1], d_h, tag)
    K = x64.shape[1] - d_h
    absprod = O.fused_kv_proj_ref(np.abs(x64), np.abs(c64), d_h, n, tag.value,
                                  threads=O.default_threads())  # sum|x||c| + |x_rep|
    g64 = to_np64(g)
    u = U16[got.dtype]
    bound = 2 * u * np.abs(ref) + 2 * K * U32 * absprod + 1e-30
    err = np.abs(g64 - ref)
    worst = float((err / bound).max())
    assert worst <= 1.0, f"elementwise bound exceeded by {worst:.3g}x"
    assert O.max_relative_error(g64, ref) <= MAXREL[got.dtype]


# ------------------------------------------------------------------ exact path
@pytest.fixture(scope="module")
def small():
    meta = json.loads((GOLDEN / "fused_small.json").read_text())
    return meta, np.load(GOLDEN / "fused_small.npz")


def test_exact_kernel_bit_identical_on_every_reference_case(small, cuda):
    meta, arrs = small
    for i, m in enumerate(meta):
        x = torch.from_numpy(arrs[f"x{i}"]).to(cuda)
        c = torch.from_numpy(arrs[f"c{i}"]).to(cuda)
        out = bd.fused_kv_proj(x, c, m["d_h"], m["n_heads"], bd.Tag(m["tag"]))
        np.testing.assert_array_equal(out.cpu().numpy(), arrs[f"out{i}"], err_msg=m["source"])


def test_exact_cfg1_k_and_v_match_reference_hashes(cuda):
    meta = json.loads((GOLDEN / "cfg1.json").read_text())
    g = np.load(GOLDEN / "cfg1.npz")
    x = torch.from_numpy(O.rand_gaussian(O.Rng(8), 256, 512, np.float32)).to(cuda)
    k = bd.fused_kv_proj(x, torch.from_numpy(g["c_qk"]).to(cuda), 64, 8, bd.Tag(meta["qk_tag"]))
    v = bd.fused_kv_proj(x, torch.from_numpy(g["c_vo"]).to(cuda), 64, 8, bd.Tag(meta["vo_tag"]))
    assert sha(k.cpu().numpy()) == meta["k_out_sha256"]
    assert sha(v.cpu().numpy()) == meta["v_out_sha256"]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", [(1, 9, 3, 2), (300, 200, 40, 3), (129, 77, 13, 5),
                                   (1000, 520, 136, 4)])
def test_exact_kernel_matches_oracle_random_shapes(dtype, shape, cuda):
    L, d, d_h, n = shape
    rng = O.Rng(sum(shape))
    x = O.rand_gaussian(rng, L, d, dtype)
    c = O.rand_gaussian(rng, d - d_h, n * d_h, dtype)
    for tag in bd.Tag:
        out = bd.fused_kv_proj(torch.from_numpy(x).to(cuda), torch.from_numpy(c).to(cuda), d_h, n,
                               tag)
        np.testing.assert_array_equal(out.cpu().numpy(),
                                      O.fused_kv_proj_ref(x, c, d_h, n, tag.value, threads=8))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("layout", ["token", "head"])
@pytest.mark.parametrize("shape", [(4000, 374, 73, 9), (6000, 103, 100, 6)])
def test_exact_large_tile_path_ragged(dtype, layout, shape, cuda):
    """Outputs big enough for the 128 x 128 exact tiles (>= 2 tiles per SM), every edge
    ragged (L, N and K = d - d_h not multiples of the tile or the k-slab; K = 3 is all
    tail): grouped K'+V', bit-identical to the C restatement of the reference kernel."""
    L, d, d_h, n = shape
    rng = O.Rng(sum(shape))
    x = O.rand_gaussian(rng, L, d, dtype)
    cs = [O.rand_gaussian(rng, d - d_h, n * d_h, dtype) for _ in range(2)]
    xt = torch.from_numpy(x).to(cuda)
    specs = [(torch.from_numpy(c).to(cuda), d_h, n, t) for c, t in zip(cs, bd.Tag)]
    outs = bd.fused_kv_proj_grouped(xt, specs, out_layout=layout)
    for c, t, o in zip(cs, bd.Tag, outs):
        got = o.cpu().numpy()
        if layout == "head":
            got = got.transpose(1, 0, 2).reshape(L, n * d_h)
        np.testing.assert_array_equal(got, O.fused_kv_proj_ref(x, c, d_h, n, t.value,
                                                                threads=O.max_threads()))


def test_exact_grouped_launch_equals_separate(cuda):
    rng = O.Rng(11)
    x = torch.from_numpy(O.rand_gaussian(rng, 70, 48, np.float32)).to(cuda)
    ck = torch.from_numpy(O.rand_gaussian(rng, 40, 24, np.float32)).to(cuda)
    cv = torch.from_numpy(O.rand_gaussian(rng, 40, 24, np.float32)).to(cuda)
    k, v = bd.fused_kv_proj_grouped(x, [(ck, 8, 3, bd.Tag.FIRST), (cv, 8, 3, bd.Tag.LAST)])
    torch.testing.assert_close(k, bd.fused_kv_proj(x, ck, 8, 3, bd.Tag.FIRST), rtol=0, atol=0)
    torch.testing.assert_close(v, bd.fused_kv_proj(x, cv, 8, 3, bd.Tag.LAST), rtol=0, atol=0)


def test_non_finite_result_raises(cuda):
    x = torch.ones(4, 10, device=cuda)
    x[1, 5] = float("inf")
    c = torch.ones(7, 9, device=cuda)
    with pytest.raises(ValueError, match="non-finite"):
        bd.fused_kv_proj(x, c, 3, 3)
    xh = x.half()
    with pytest.raises(ValueError, match="non-finite"):
        bd.fused_kv_proj(torch.nn.functional.pad(xh, (0, 6)), torch.ones(8, 16, device=cuda).half(),
                         8, 2)


def test_host_entry_point_bit_exact(cuda):
    rng = O.Rng(21)
    x = O.rand_gaussian(rng, 33, 50, np.float32)
    c = O.rand_gaussian(rng, 40, 30, np.float32)
    np.testing.assert_array_equal(bd.fused_kv_proj_host(x, c, 10, 3, bd.Tag.LAST),
                                  O.fused_kv_proj_ref(x, c, 10, 3, "last"))


# ------------------------------------------------------------------ tensor-core path
TC_SHAPES = [
    # L, d, d_h, n_heads
    (256, 512, 64, 8),      # cfg1 geometry
    (1000, 512, 128, 16),   # DSV2-Lite kv_b_proj half, ragged L
    (128, 328, 64, 3),      # K=264 (not a multiple of 64), N=192 (< one 256 tile)
    (77, 136, 8, 5),        # tiny d_h, N=40
    (300, 1024, 128, 7),    # N = 896: last tile partial
    (200, 1024, 256, 3),    # d_h = 256: rep not staged (per-element gather path), K = 768
    (130, 200, 24, 5),      # d_h = 24, N = 120: odd head width, one partial sub-chunk
]


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("shape", TC_SHAPES)
def test_tc_kernel_matches_fp64_oracle(dtype, shape, cuda):
    L, d, d_h, n = shape
    g = torch.Generator().manual_seed(L * 7 + d)
    x = torch.randn(L, d, generator=g).to(dtype).to(cuda)
    c = (torch.randn(d - d_h, n * d_h, generator=g) / 4).to(dtype).to(cuda)
    for tag in bd.Tag:
        out = bd.fused_kv_proj(x, c, d_h, n, tag)
        assert out.dtype == dtype
        assert_tc_close(out, x, c, d_h, n, tag)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_tc_cfg2_full_size_sampled_rows(dtype, cuda):
    """DSV2-Lite kv_b_proj, 8192 tokens, K and V in one launch (BASELINE config 2)."""
    L, d, d_h, n = 8192, 512, 128, 16
    g = torch.Generator().manual_seed(2)
    x = torch.randn(L, d, generator=g).to(dtype).to(cuda)
    ck = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    cv = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    k, v = bd.fused_kv_proj_grouped(x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)],
                                    check_finite=True)
    rows = torch.randperm(L, generator=g)[:96].sort().values
    rows = torch.cat([rows, torch.tensor([0, 127, 128, L - 1])])
    assert_tc_close(k, x, ck, d_h, n, bd.Tag.FIRST, rows=rows.to(cuda))
    assert_tc_close(v, x, cv, d_h, n, bd.Tag.LAST, rows=rows.to(cuda))
    # size-independent properties over the FULL output:
    # (1) zero coefficients -> exact repeat of the basis slice
    z = bd.fused_kv_proj(x, torch.zeros_like(ck), d_h, n, bd.Tag.FIRST)
    torch.testing.assert_close(z, x[:, :d_h].repeat(1, n), rtol=0, atol=0)
    # (2) scaling x by 2 is exact in binary floating point -> output doubles exactly
    #     (wherever the result is a normal number: subnormal outputs round on an absolute
    #     grid, so round(2v) and 2 round(v) may differ there)
    k2 = bd.fused_kv_proj(x * 2, ck, d_h, n, bd.Tag.FIRST)
    normal = k.float().abs() >= torch.finfo(dtype).tiny * 2
    assert int(normal.sum()) > 0.99 * k.numel()
    torch.testing.assert_close(k2[normal], (k * 2)[normal], rtol=0, atol=0)
    # (3) grouped launch == separate launches, bit for bit
    torch.testing.assert_close(bd.fused_kv_proj(x, cv, d_h, n, bd.Tag.LAST), v, rtol=0, atol=0)


def test_tc_matches_cublas_dense_with_rewritten_weight(cuda):
    """Kernel vs cuBLAS X @ W' where W' = [I; C] per head (the BD-rewritten dense weight):
    same math, different summation -> within FP16 rounding."""
    L, d, d_h, n = 2048, 512, 128, 16
    g = torch.Generator().manual_seed(5)
    x = torch.randn(L, d, generator=g).half().to(cuda)
    c = (torch.randn(d - d_h, n * d_h, generator=g) / 8).half().to(cuda)
    eye = torch.eye(d_h, dtype=torch.float16, device=cuda).repeat(1, n)
    w_dense = torch.cat([eye, c], dim=0)  # FIRST tag: identity rows at S = [0, d_h)
    dense = x @ w_dense
    ours = bd.fused_kv_proj(x, c, d_h, n, bd.Tag.FIRST)
    rel = (ours.float() - dense.float()).abs().max() / dense.float().abs().max()
    assert float(rel) < 2e-3


def test_tc_head_shards_are_bit_identical(cuda):
    """Column (head) shards of c give bit-identical columns: the multi-GPU invariant."""
    L, d, d_h, n = 512, 512, 128, 16
    g = torch.Generator().manual_seed(9)
    x = torch.randn(L, d, generator=g).half().to(cuda)
    c = (torch.randn(d - d_h, n * d_h, generator=g) / 8).half().to(cuda)
    full = bd.fused_kv_proj(x, c, d_h, n, bd.Tag.LAST)
    for world in (2, 4, 8):
        per = n // world
        for r in range(world):
            cs = c[:, r * per * d_h:(r + 1) * per * d_h].contiguous()
            part = bd.fused_kv_proj(x, cs, d_h, per, bd.Tag.LAST)
            torch.testing.assert_close(part, full[:, r * per * d_h:(r + 1) * per * d_h],
                                       rtol=0, atol=0)


@pytest.mark.parametrize("L", [200, 40])  # persistent and small-L kernels
def test_tc_strided_views(L, cuda):
    """Row-strided x/out views (e.g. a slice of a larger activation buffer) are honoured."""
    d, d_h, n = 256, 64, 4
    g = torch.Generator().manual_seed(3)
    big = torch.randn(L, d + 64, generator=g).half().to(cuda)
    x = big[:, 32:32 + d]
    c = (torch.randn(d - d_h, n * d_h, generator=g) / 4).half().to(cuda)
    obuf = torch.full((L, n * d_h + 16), 7.0, dtype=torch.float16, device=cuda)
    out = obuf[:, 8:8 + n * d_h]
    bd.fused_kv_proj(x, c, d_h, n, bd.Tag.FIRST, out=out)
    assert_tc_close(out, x, c, d_h, n, bd.Tag.FIRST)
    assert bool((obuf[:, :8] == 7).all()) and bool((obuf[:, 8 + n * d_h:] == 7).all())


def test_tc_host_entry_point(cuda):
    rng = O.Rng(4)
    x = O.rand_gaussian(rng, 300, 256, np.float16)
    c = (O.rand_gaussian(rng, 192, 256, np.float32) / 4).astype(np.float16)
    out = bd.fused_kv_proj_host(x, c, 64, 4, bd.Tag.FIRST)
    assert_tc_close(torch.from_numpy(out), torch.from_numpy(x), torch.from_numpy(c), 64, 4,
                    bd.Tag.FIRST)


def test_launch_counter_counts_our_kernels(cuda):
    x = torch.randn(64, 64, device=cuda).half()
    c = torch.randn(32, 64, device=cuda).half()
    before = N.launch_count()
    bd.fused_kv_proj(x, c, 32, 2, check_finite=False)
    torch.cuda.synchronize()
    assert N.launch_count() == before + 1


def test_compat_shim_is_bit_exact_on_every_reference_case(small, cuda):
    """INTEGRATION.md's drop-in for numba's _fused_kernel (numpy in, out overwritten)."""
    from paper_2510_01718_b200 import compat
    meta, arrs = small
    for i, m in enumerate(meta):
        x, c = arrs[f"x{i}"], arrs[f"c{i}"]
        mul_base, rep_base = O.tag_offsets(x.shape[1], m["d_h"], m["tag"])
        out = np.zeros((x.shape[0], m["n_heads"] * m["d_h"]), dtype=x.dtype)  # ref pre-zeroes
        compat._fused_kernel(x, c, m["d_h"], m["n_heads"], mul_base, rep_base, out)
        np.testing.assert_array_equal(out, arrs[f"out{i}"], err_msg=m["source"])


def test_tc_cfg3_llama_shape_streaming_k(cuda):
    """BASELINE config 3 geometry (d=4096, 32 heads x 128, BF16): K = 3968 streams A
    through the slot ring.  512 tokens, sampled rows vs the FP64 oracle."""
    L, d, d_h, n = 512, 4096, 128, 32
    g = torch.Generator().manual_seed(33)
    x = torch.randn(L, d, generator=g).bfloat16().to(cuda)
    ck = (torch.randn(d - d_h, n * d_h, generator=g) / 64).bfloat16().to(cuda)
    cv = (torch.randn(d - d_h, n * d_h, generator=g) / 64).bfloat16().to(cuda)
    k, v = bd.fused_kv_proj_grouped(x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)],
                                    check_finite=True)
    rows = torch.tensor([0, 1, 127, 128, 255, 256, 300, 511], device=cuda)
    assert_tc_close(k, x, ck, d_h, n, bd.Tag.FIRST, rows=rows)
    assert_tc_close(v, x, cv, d_h, n, bd.Tag.LAST, rows=rows)


def test_tc_grouped_four_problems_mixed_shapes(cuda):
    """Up to BD_MAX_GROUP problems in one launch, different N / d_h / tags and one
    resident-A (K <= 384) next to one streaming-A (K > 384) problem."""
    g = torch.Generator().manual_seed(44)
    L = 300
    x1 = torch.randn(L, 512, generator=g).half().to(cuda)
    c1 = (torch.randn(384, 2048, generator=g) / 8).half().to(cuda)
    c2 = (torch.randn(448, 512, generator=g) / 8).half().to(cuda)
    c3 = (torch.randn(384, 256, generator=g) / 8).half().to(cuda)
    c4 = (torch.randn(504, 64, generator=g) / 8).half().to(cuda)
    outs = bd.fused_kv_proj_grouped(x1, [(c1, 128, 16, bd.Tag.FIRST), (c2, 64, 8, bd.Tag.LAST),
                                         (c3, 128, 2, bd.Tag.LAST), (c4, 8, 8, bd.Tag.FIRST)])
    for o, (c, d_h, n, tag) in zip(outs, [(c1, 128, 16, bd.Tag.FIRST), (c2, 64, 8, bd.Tag.LAST),
                                          (c3, 128, 2, bd.Tag.LAST), (c4, 8, 8, bd.Tag.FIRST)]):
        assert_tc_close(o, x1, c, d_h, n, tag)
        torch.testing.assert_close(o, bd.fused_kv_proj(x1, c, d_h, n, tag), rtol=0, atol=0)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16, torch.float32])
@pytest.mark.parametrize("shape", [(300, 512, 128, 16), (77, 256, 64, 3), (8192, 512, 128, 16)])
def test_head_major_output_equals_token_major(dtype, shape, cuda):
    """out_layout='head' writes [n, L, d_h] (per-head TMA boxes clipped at each head's
    L rows): bit-identical to the token-major result rearranged."""
    L, d, d_h, n = shape
    g = torch.Generator().manual_seed(L + d_h)
    x = torch.randn(L, d, generator=g).to(dtype).to(cuda)
    ck = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    cv = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    specs = [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)]
    tok = bd.fused_kv_proj_grouped(x, specs)
    head = bd.fused_kv_proj_grouped(x, specs, out_layout="head")
    for t, h in zip(tok, head):
        assert h.shape == (n, L, d_h)
        torch.testing.assert_close(h, t.view(L, n, d_h).permute(1, 0, 2), rtol=0, atol=0)
    single = bd.fused_kv_proj(x, cv, d_h, n, bd.Tag.LAST, out_layout="head")
    torch.testing.assert_close(single, head[1], rtol=0, atol=0)


def test_head_major_tc_needs_d_h_multiple_of_64(cuda):
    x = torch.randn(64, 72, device=cuda).half()
    c = torch.randn(64, 16, device=cuda).half()
    with pytest.raises(bd.ShapeError):
        bd.fused_kv_proj(x, c, 8, 2, out_layout="head")


@pytest.mark.parametrize("dtype,L", [(torch.float16, 700), (torch.bfloat16, 700),
                                     (torch.float32, 700), (torch.float32, 3000)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_fused_allgather_single_device_ranks(dtype, L, world, cuda):
    """The all-gather fused into the epilogue, every 'rank' on one device: after each
    rank's launch with its head shard, EVERY rank's gathered buffer holds the full
    head-major K'/V' — bit-identical to the unsharded head-major projection (the
    multi-GPU version differs only in the buffers being peer memory).  FP32 at L = 3000
    takes the exact kernel's 128 x 128 tiles for world <= 2, its 64 x 64 tiles beyond."""
    from paper_2510_01718_b200 import parallel as P
    d, d_h, n = 512, 128, 16
    g = torch.Generator().manual_seed(world)
    x = torch.randn(L, d, generator=g).to(dtype).to(cuda)
    ck = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    cv = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    full = bd.fused_kv_proj_grouped(x, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)],
                                    out_layout="head")
    gathered = [[torch.full((n, L, d_h), 3.0, dtype=dtype, device=cuda) for _ in range(world)]
                for _ in range(2)]
    for r in range(world):
        specs = [(P.shard_columns(ck, d_h, n, world, r), d_h, n // world, bd.Tag.FIRST),
                 (P.shard_columns(cv, d_h, n, world, r), d_h, n // world, bd.Tag.LAST)]
        P.fused_allgather_kv_proj(x, specs, gathered, r)
    for p_ in range(2):
        for r in range(world):
            torch.testing.assert_close(gathered[p_][r], full[p_], rtol=0, atol=0)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("L", [1, 7, 64, 128, 129, 200, 256, 300, 384, 500, 640])
def test_small_l_kernel_bit_identical_to_persistent_kernel(dtype, L, cuda):
    """L <= 640 at this width runs the small-L (decode) kernel (32 / 64 / 128 / 160-column
    blocks by L); its rows equal, bit for bit, the same rows computed by the
    persistent kernel inside a longer batch (same FP32 tensor-core accumulation, same
    FHADD + rounding), for both tags, grouped, and head-major."""
    d, d_h, n = 512, 128, 16
    g = torch.Generator().manual_seed(L)
    x_long = torch.randn(1500, d, generator=g).to(dtype).to(cuda)
    ck = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    cv = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    specs = [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)]
    k_long, v_long = bd.fused_kv_proj_grouped(x_long, specs)
    x = x_long[:L].clone()
    k, v = bd.fused_kv_proj_grouped(x, specs, check_finite=True)
    torch.testing.assert_close(k, k_long[:L], rtol=0, atol=0)
    torch.testing.assert_close(v, v_long[:L], rtol=0, atol=0)
    kh, vh = bd.fused_kv_proj_grouped(x, specs, out_layout="head")
    torch.testing.assert_close(kh, k.view(L, n, d_h).transpose(0, 1), rtol=0, atol=0)
    torch.testing.assert_close(vh, v.view(L, n, d_h).transpose(0, 1), rtol=0, atol=0)


def test_launch_parameter_cache_follows_buffers(cuda):
    """The C library caches encoded launch parameters per buffer signature: alternating
    calls over different buffers (same shapes), strides, layouts, tags and flag pointers
    must each compute their own result (no stale tensor maps or flag pointers)."""
    L, d, d_h, n = 700, 512, 128, 16
    g = torch.Generator().manual_seed(21)
    xs = [torch.randn(L, d, generator=g).half().to(cuda) for _ in range(3)]
    cs = [(torch.randn(d - d_h, n * d_h, generator=g) / 8).half().to(cuda) for _ in range(2)]
    ref = {(i, j, t): bd.fused_kv_proj(xs[i], cs[j], d_h, n, t, check_finite=False)
           for i in range(3) for j in range(2) for t in bd.Tag}
    for rnd in range(3):  # > cache size distinct signatures, revisited
        for (i, j, t), want in ref.items():
            out = torch.empty(L, n * d_h + 64, dtype=torch.half, device=cuda)[:, :n * d_h] \
                if (i + j + rnd) % 2 else None
            got = bd.fused_kv_proj(xs[i], cs[j], d_h, n, t, out=out, check_finite=(rnd == 1))
            torch.testing.assert_close(got, want, rtol=0, atol=0)
    # the non-finite flag of a cached signature still reaches the kernel
    bad = xs[0].clone()
    bad[5, 300] = float("inf")
    with pytest.raises(ValueError):
        bd.fused_kv_proj(bad, cs[0], d_h, n, bd.Tag.FIRST, check_finite=True)
    with pytest.raises(ValueError):
        bd.fused_kv_proj(bad, cs[0], d_h, n, bd.Tag.FIRST, check_finite=True)


def _rmsnorm_bd_ref(x, cs, gamma, eps, d_h, n):
    """float64 reference of the fused path on the kernel's exact inputs: the 16-bit x, the
    folded (rounded) c_g and float32 rep_gamma — r * (x[:, mul] c_g + rep_gamma x[:, rep])."""
    xd = x.double()
    r = torch.rsqrt(xd.pow(2).mean(1, keepdim=True) + eps)
    outs = []
    for c_g, rg, tag in cs:
        mul, rep = bd.tag_offsets(x.shape[1], d_h, tag)
        K = c_g.shape[0]
        rep_term = (rg.double()[None, :] * xd[:, rep:rep + d_h]).repeat(1, n)
        outs.append(r * (xd[:, mul:mul + K] @ c_g.double() + rep_term))
    return outs


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("L", [100, 256, 300, 8192])
def test_fused_rmsnorm_projection(dtype, L, cuda):
    """RMSNorm fused into the K'/V' projection (DeepSeek kv_a_layernorm + kv_b_proj):
    against a float64 evaluation on the same (rounded) operands, and against the unfused
    path (RMSNorm -> round to dtype -> projection).  L = 256 gives pairs a single tile of a
    row-block (the A slots' release then waits for the norm's reads)."""
    d, d_h, n, eps = 512, 128, 16, 1e-6
    g = torch.Generator().manual_seed(L + 3)
    x = (torch.randn(L, d, generator=g) * (0.5 + torch.rand(L, 1, generator=g) * 3)).to(dtype).to(cuda)
    gamma = (0.5 + torch.rand(d, generator=g)).to(cuda)
    ck = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    cv = (torch.randn(d - d_h, n * d_h, generator=g) / 8).to(dtype).to(cuda)
    folded = [bd.fold_rmsnorm(ck, gamma, d_h, bd.Tag.FIRST) + (bd.Tag.FIRST,),
              bd.fold_rmsnorm(cv, gamma, d_h, bd.Tag.LAST) + (bd.Tag.LAST,)]
    specs = [(cg, rg, d_h, n, t) for cg, rg, t in folded]
    k, v = bd.fused_rmsnorm_kv_proj_grouped(x, specs, eps, check_finite=True)
    kr, vr = _rmsnorm_bd_ref(x, folded, gamma, eps, d_h, n)
    tol = {torch.float16: 2e-3, torch.bfloat16: 1.6e-2, torch.float32: 2e-6,
           torch.float64: 1e-13}[dtype]
    for got, ref in ((k, kr), (v, vr)):
        err = float((got.double() - ref).abs().max() / ref.abs().max())
        assert err <= tol, err
    # the unfused composition: normalise, round to dtype, project
    xn = (x.double() * torch.rsqrt(x.double().pow(2).mean(1, keepdim=True) + eps)
          * gamma.double()).to(dtype)
    ku, vu = bd.fused_kv_proj_grouped(xn, [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)])
    loose = {torch.float16: 8e-3, torch.bfloat16: 6e-2, torch.float32: 2e-5, torch.float64: 1e-12}[dtype]
    for got, ref in ((k, ku), (v, vu)):
        err = float((got.double() - ref.double()).abs().max() / ref.double().abs().max())
        assert err <= loose, err
    # head-major output of the same launch
    kh, vh = bd.fused_rmsnorm_kv_proj_grouped(x, specs, eps, out_layout="head")
    torch.testing.assert_close(kh, k.view(L, n, d_h).transpose(0, 1), rtol=0, atol=0)
    torch.testing.assert_close(vh, v.view(L, n, d_h).transpose(0, 1), rtol=0, atol=0)


def test_fused_rmsnorm_rejects_unsupported_shapes(cuda):
    x = torch.randn(64, 200, device=cuda).half()
    c = torch.randn(176, 24 * 5, device=cuda).half()
    cg, rg = bd.fold_rmsnorm(c, torch.ones(200, device=cuda), 24, bd.Tag.FIRST)
    with pytest.raises(bd.ShapeError):
        bd.fused_rmsnorm_kv_proj_grouped(x, [(cg, rg, 24, 5, bd.Tag.FIRST)], 1e-6)


def test_tc_random_shapes_fuzz(cuda):
    """Randomised sweep across the tensor-core kernels' dispatch space — small-L single
    CTAs, small-L pairs, the persistent kernel with contiguous or round-robin schedules —
    with random legal shapes, tags, dtypes, layouts, strides and grouping: every output
    against the FP64 oracle's elementwise bound, grouped == separate bit for bit."""
    rng = np.random.default_rng(int(os.environ.get("BD_FUZZ_SEED", "2026")))
    for case in range(int(os.environ.get("BD_FUZZ_CASES", "60"))):
        dtype = [torch.float16, torch.bfloat16][case % 2]
        d_h = int(rng.choice([8, 24, 64, 128, 192]))
        K = int(rng.choice([8, 56, 200, 384, 448, 904]))
        d = K + d_h
        # the second problem may use another head width (same x, so K differs too);
        # head-major output needs d_h % 64 == 0 for every problem of the launch
        d_h2 = d_h if rng.random() < 0.5 else int(rng.choice([8, 24, 64, 128]))
        d_h2 = d_h2 if d_h2 < d else d_h
        n = int(rng.integers(1, 12))
        L = int(rng.choice([1, 5, 64, 127, 129, 200, 256, 257, 700]))
        layout = "head" if d_h % 64 == 0 and d_h2 % 64 == 0 and rng.random() < 0.4 else "token"
        pad = int(rng.choice([0, 8, 24]))
        g = torch.Generator().manual_seed(case)
        big = torch.randn(L, d + pad, generator=g).to(dtype).to(cuda)
        x = big[:, pad:pad + d] if pad else big
        dhs = [d_h, d_h2]
        cs = [(torch.randn(d - dh, n * dh, generator=g) / 8).to(dtype).to(cuda) for dh in dhs]
        tags = [bd.Tag.FIRST, bd.Tag.LAST][:: 1 if rng.random() < 0.5 else -1]
        specs = [(c, dh, n, t) for c, dh, t in zip(cs, dhs, tags)]
        outs = bd.fused_kv_proj_grouped(x, specs, out_layout=layout, check_finite=True)
        for (c, dh, _, t), o in zip(specs, outs):
            tok = o.transpose(0, 1).reshape(L, n * dh) if layout == "head" else o
            assert_tc_close(tok, x, c, dh, n, t)
            single = bd.fused_kv_proj(x, c, dh, n, t, out_layout=layout, check_finite=False)
            torch.testing.assert_close(single, o, rtol=0, atol=0)


def test_exact_random_shapes_fuzz(cuda):
    """The exact kernel over random shapes (any d_h, odd sizes), both tags, grouped and
    head-major: bit-identical to the C restatement of the reference kernel."""
    rng = np.random.default_rng(int(os.environ.get("BD_FUZZ_SEED", "7")))
    for case in range(int(os.environ.get("BD_FUZZ_CASES", "30"))):
        npdt = [np.float32, np.float64][case % 2]
        d_h = int(rng.integers(1, 40))
        d = d_h + int(rng.integers(1, 120))
        n = int(rng.integers(1, 6))
        L = int(rng.integers(1, 150))
        x = rng.standard_normal((L, d)).astype(npdt)
        cs = [(rng.standard_normal((d - d_h, n * d_h)) / 4).astype(npdt) for _ in range(2)]
        xt = torch.from_numpy(x).to(cuda)
        specs = [(torch.from_numpy(c).to(cuda), d_h, n, t) for c, t in zip(cs, bd.Tag)]
        layout = "head" if case % 3 == 0 else "token"
        outs = bd.fused_kv_proj_grouped(xt, specs, out_layout=layout)
        for c, t, o in zip(cs, bd.Tag, outs):
            want = O.fused_kv_proj_ref(x, c, d_h, n, t.value)
            got = o.cpu().numpy()
            if layout == "head":
                got = got.transpose(1, 0, 2).reshape(L, n * d_h)
            np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("order", [(96, 128), (128, 96), (8, 64, 128, 24)])
def test_grouped_mixed_d_h_rep_staging_order(order, cuda):
    """Grouped launch where a problem whose rep tile is NOT staged (d_h not in {64, 128})
    precedes one whose rep tile is (the look-ahead that stages the next
    row-block's rep must skip non-staged row-blocks, or the pair whose range crosses
    into the staged problem waits forever).  L > 256 so pairs span both problems."""
    L, d = 700, 480
    g = torch.Generator().manual_seed(sum(order))
    x = torch.randn(L, d, generator=g).half().to(cuda)
    specs = []
    for i, d_h in enumerate(order):
        n = max(1, 512 // d_h)
        c = (torch.randn(d - d_h, n * d_h, generator=g) / 8).half().to(cuda)
        specs.append((c, d_h, n, [bd.Tag.FIRST, bd.Tag.LAST][i % 2]))
    outs = bd.fused_kv_proj_grouped(x, specs, check_finite=True)
    torch.cuda.synchronize()
    for o, (c, d_h, n, t) in zip(outs, specs):
        assert_tc_close(o, x, c, d_h, n, t)
        torch.testing.assert_close(o, bd.fused_kv_proj(x, c, d_h, n, t), rtol=0, atol=0)


def test_fused_rmsnorm_eps_zero_ragged_l_is_finite(cuda):
    """eps = 0 with L not a multiple of 256: rows past L (TMA zero-fill) must not trip
    the non-finite check (rsqrt(0) * 0 = NaN in padding rows)."""
    L, d, d_h, n = 300, 512, 128, 16
    g = torch.Generator().manual_seed(17)
    x = torch.randn(L, d, generator=g).half().to(cuda)
    gamma = (0.5 + torch.rand(d, generator=g)).to(cuda)
    ck = (torch.randn(d - d_h, n * d_h, generator=g) / 8).half().to(cuda)
    cv = (torch.randn(d - d_h, n * d_h, generator=g) / 8).half().to(cuda)
    folded = [bd.fold_rmsnorm(ck, gamma, d_h, bd.Tag.FIRST) + (bd.Tag.FIRST,),
              bd.fold_rmsnorm(cv, gamma, d_h, bd.Tag.LAST) + (bd.Tag.LAST,)]
    specs = [(cg, rg, d_h, n, t) for cg, rg, t in folded]
    k, v = bd.fused_rmsnorm_kv_proj_grouped(x, specs, 0.0, check_finite=True)
    kr, vr = _rmsnorm_bd_ref(x, folded, gamma, 0.0, d_h, n)
    for got, ref in ((k, kr), (v, vr)):
        assert float((got.double() - ref).abs().max() / ref.abs().max()) <= 2e-3


def test_check_finite_is_the_default_like_the_reference(cuda):
    """ref tensor.py:112-113 raises on any non-finite result: the grouped call and
    bda_forward do too unless asked not to."""
    x = torch.randn(64, 96, device=cuda).half()
    x[3, 50] = float("inf")
    c = torch.randn(64, 64, device=cuda).half()
    with pytest.raises(ValueError, match="non-finite"):
        bd.fused_kv_proj_grouped(x, [(c, 32, 2, bd.Tag.FIRST)])
    out = bd.fused_kv_proj_grouped(x, [(c, 32, 2, bd.Tag.FIRST)], check_finite=False)
    assert not bool(torch.isfinite(out[0]).all())


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_mirror_schedule_narrow_shards(dtype, cuda):
    """2 + 2 heads (one 256-wide column tile per problem) at 20480 tokens: the launch takes
    the mirror schedule (coefficient tile resident, x streamed, tiles column-tile major).
    Its outputs equal, bit for bit, the same heads' columns of a 16-head launch (the
    row-block-major schedule), and one row of every 256-row block meets the FP64 oracle's
    elementwise bound — the per-rank shape of head-sharded weak scaling at 8 GPUs."""
    L, d, d_h, n_full, h0, n = 20480, 512, 128, 16, 6, 2
    g = torch.Generator().manual_seed(88)
    x = torch.randn(L, d, generator=g).to(dtype).to(cuda)
    ck = (torch.randn(d - d_h, n_full * d_h, generator=g) / 8).to(dtype).to(cuda)
    cv = (torch.randn(d - d_h, n_full * d_h, generator=g) / 8).to(dtype).to(cuda)
    k_full, v_full = bd.fused_kv_proj_grouped(
        x, [(ck, d_h, n_full, bd.Tag.FIRST), (cv, d_h, n_full, bd.Tag.LAST)], check_finite=False)
    cols = slice(h0 * d_h, (h0 + n) * d_h)
    cks, cvs = ck[:, cols].contiguous(), cv[:, cols].contiguous()
    k, v = bd.fused_kv_proj_grouped(x, [(cks, d_h, n, bd.Tag.FIRST), (cvs, d_h, n, bd.Tag.LAST)],
                                    check_finite=True)
    torch.testing.assert_close(k, k_full[:, cols], rtol=0, atol=0)
    torch.testing.assert_close(v, v_full[:, cols], rtol=0, atol=0)
    rows = torch.tensor(sorted({min(L - 1, b * 256 + (37 * b) % 256) for b in range(L // 256)}))
    assert_tc_close(k, x, cks, d_h, n, bd.Tag.FIRST, rows=rows.to(cuda))
    assert_tc_close(v, x, cvs, d_h, n, bd.Tag.LAST, rows=rows.to(cuda))


@pytest.mark.parametrize("layout", ["token", "head"])
def test_mirror_schedule_k_tail_and_layouts(layout, cuda):
    """The mirror schedule with a K that is not a multiple of 64 (d = 328, d_h = 64:
    K = 264, the last coefficient / x k-block zero-filled by TMA), 4 heads of 64 (one
    256-wide tile) at 20480 tokens, token- and head-major output: equal to the same heads'
    columns of a 12-head launch (row-block-major) and within the oracle bound."""
    L, d, d_h, n_full, h0, n = 20480, 328, 64, 12, 4, 4
    g = torch.Generator().manual_seed(99)
    x = torch.randn(L, d, generator=g).half().to(cuda)
    ck = (torch.randn(d - d_h, n_full * d_h, generator=g) / 8).half().to(cuda)
    cv = (torch.randn(d - d_h, n_full * d_h, generator=g) / 8).half().to(cuda)
    cols = slice(h0 * d_h, (h0 + n) * d_h)
    k_full, v_full = bd.fused_kv_proj_grouped(
        x, [(ck, d_h, n_full, bd.Tag.FIRST), (cv, d_h, n_full, bd.Tag.LAST)], check_finite=False)
    cks, cvs = ck[:, cols].contiguous(), cv[:, cols].contiguous()
    k, v = bd.fused_kv_proj_grouped(x, [(cks, d_h, n, bd.Tag.FIRST), (cvs, d_h, n, bd.Tag.LAST)],
                                    out_layout=layout, check_finite=True)
    if layout == "head":
        k = k.transpose(0, 1).reshape(L, n * d_h)
        v = v.transpose(0, 1).reshape(L, n * d_h)
    torch.testing.assert_close(k, k_full[:, cols], rtol=0, atol=0)
    torch.testing.assert_close(v, v_full[:, cols], rtol=0, atol=0)
    rows = torch.tensor(sorted({min(L - 1, b * 256 + (53 * b) % 256) for b in range(L // 256)}))
    assert_tc_close(k, x, cks, d_h, n, bd.Tag.FIRST, rows=rows.to(cuda))
    assert_tc_close(v, x, cvs, d_h, n, bd.Tag.LAST, rows=rows.to(cuda))


@pytest.mark.parametrize("L", [1, 300, 1000, 8192])
@pytest.mark.parametrize("chunks", [1, 4])
def test_host_pipeline_equals_device_path(L, chunks, cuda):
    """fused_kv_proj_grouped_host (the end-to-end path: pinned host x in, K'/V' out,
    row blocks pipelined over copy-in / kernel / copy-out streams) returns exactly the
    device path's K'/V' for ragged L and any chunking."""
    d, d_h, n = 512, 128, 16
    g = torch.Generator().manual_seed(L + chunks)
    xh = torch.randn(L, d, generator=g).half().pin_memory()
    ck = (torch.randn(d - d_h, n * d_h, generator=g) / 8).half().to(cuda)
    cv = (torch.randn(d - d_h, n * d_h, generator=g) / 8).half().to(cuda)
    specs = [(ck, d_h, n, bd.Tag.FIRST), (cv, d_h, n, bd.Tag.LAST)]
    k, v = bd.fused_kv_proj_grouped_host(xh, specs, chunks=chunks)
    assert not k.is_cuda and not v.is_cuda
    kd, vd = bd.fused_kv_proj_grouped(xh.to(cuda), specs)
    torch.testing.assert_close(k, kd.cpu(), rtol=0, atol=0)
    torch.testing.assert_close(v, vd.cpu(), rtol=0, atol=0)


def test_host_pipeline_raises_on_non_finite(cuda):
    xh = torch.ones(700, 512).half()
    xh[650, 300] = float("inf")
    c = (torch.ones(384, 256) / 8).half().to(cuda)
    with pytest.raises(ValueError, match="non-finite"):
        bd.fused_kv_proj_grouped_host(xh.pin_memory(), [(c, 128, 2, bd.Tag.FIRST)])
    # the flag is reset per call: a finite input right after passes
    ok = bd.fused_kv_proj_grouped_host(torch.ones(700, 512).half().pin_memory(),
                                       [(c, 128, 2, bd.Tag.FIRST)])
    assert torch.isfinite(ok[0].float()).all()
