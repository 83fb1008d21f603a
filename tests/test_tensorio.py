"""BDT1 / manifest interchange with the reference's prepared bundles (ref
tensorio.py): a bundle written by bdattn itself (tests/golden/bundle, made by
make_golden.py) loads here bit-exactly, our prep of the same model matches it, and
what we write is byte-identical to what the reference wrote.  CPU; the GPU test loads
straight onto the device in FP32 and runs the exact kernel."""

import filecmp

import numpy as np
import pytest
import torch

from conftest import GOLDEN
import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import tensorio as tio

BUNDLE = GOLDEN / "bundle"


def test_reference_bundle_loads_and_matches_our_prep():
    w_ref = tio.load_mha_manifest(BUNDLE / "model.mha")
    p_ref = tio.load_bda_manifest(BUNDLE / "model.bda")
    w = bd.gen_random_mha(bd.Rng(21), 24, 4, 5, torch.float32)
    for r in tio.MHA_ROLES:
        torch.testing.assert_close(getattr(w_ref, r), getattr(w, r), rtol=0, atol=0)
    p = bd.bda_prepare(w, prepare_in_p64=True)
    assert (p.qk_tag, p.vo_tag) == (p_ref.qk_tag, p_ref.vo_tag)
    assert p.qk_candidate_residuals == p_ref.qk_candidate_residuals
    for r in tio.BDA_ROLES:
        torch.testing.assert_close(getattr(p_ref, r), getattr(p, r), rtol=0, atol=0)
    assert tio.manifest_kind(BUNDLE / "model.bda") == "bda"


def test_our_bundle_is_byte_identical_to_the_reference(tmp_path):
    p = bd.bda_prepare(bd.gen_random_mha(bd.Rng(21), 24, 4, 5, torch.float32),
                       prepare_in_p64=True)
    tio.save_bda_manifest(tmp_path / "model.bda", p)
    for f in ["model.bda"] + [f"model.{r}.bdt" for r in tio.BDA_ROLES]:
        assert filecmp.cmp(tmp_path / f, BUNDLE / f, shallow=False), f


def test_bad_files_raise(tmp_path):
    (tmp_path / "x.bdt").write_bytes(b"BDT0" + bytes(18))
    with pytest.raises(tio.TensorFileError):
        tio.load_tensor(tmp_path / "x.bdt")
    tio.save_tensor(tmp_path / "y.bdt", torch.ones(2, 3))
    raw = (tmp_path / "y.bdt").read_bytes()
    (tmp_path / "z.bdt").write_bytes(raw[:-4])
    with pytest.raises(tio.TensorFileError):
        tio.load_tensor(tmp_path / "z.bdt")
    (tmp_path / "m.bda").write_text("bda-manifest v2\n")
    with pytest.raises(tio.ManifestError):
        tio.load_bda_manifest(tmp_path / "m.bda")
    with pytest.raises(tio.TensorFileError):
        tio.save_tensor(tmp_path / "h.bdt", torch.ones(2, 2, dtype=torch.float16))


@pytest.mark.gpu
def test_bundle_to_gpu_fp32_projection(cuda):
    """A reference-written bundle loaded straight onto the GPU drives the exact FP32
    kernel: bit-identical to the C restatement of the reference kernel (the bundle's
    d_h = 4 is below the tensor-core path's multiple-of-8 granularity)."""
    from oracle import oracle as O
    p = tio.load_bda_manifest(BUNDLE / "model.bda", device=cuda)
    assert p.c_qk.dtype == torch.float32
    x = bd.rand_gaussian(bd.Rng(5), 16, 24, torch.float32, cuda)
    k = bd.fused_kv_proj(x, p.c_qk, p.d_h, p.n_heads, p.qk_tag)
    want = O.fused_kv_proj_ref(x.cpu().numpy(), p.c_qk.cpu().numpy(), p.d_h, p.n_heads,
                               p.qk_tag.value)
    np.testing.assert_array_equal(k.cpu().numpy(), want)
