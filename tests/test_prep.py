"""The offline preparation (decompose.py, attention.bda_prepare, linear prep) and the
input generators reproduce the reference bit for bit — tags (the basis S), candidate
residuals, prepared matrices — against tests/golden (made by running the reference,
tests/golden/make_golden.py).  CPU only: prep is offline NumPy/SciPy by design."""

import hashlib
import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import decompose as D


def sha(t) -> str:
    a = t.numpy() if isinstance(t, torch.Tensor) else t
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


DT = {"p64": torch.float64, "p32": torch.float32}


@pytest.fixture(scope="module")
def prep_cases():
    return json.loads((GOLDEN / "prep_tags.json").read_text())


def test_prep_tags_residuals_and_matrices_match_reference(prep_cases):
    assert len(prep_cases) == 32
    for c in prep_cases:
        w = bd.gen_random_mha(bd.Rng(c["seed"]), c["d"], c["d_h"], c["n_heads"], DT[c["precision"]])
        p = bd.bda_prepare(w, prepare_in_p64=c["prepare_in_p64"])
        where = f"case {c}"
        # the basis S: bit-exact
        assert p.qk_tag.value == c["qk_tag"], where
        assert p.vo_tag.value == c["vo_tag"], where
        # the mean residuals that decided it: bit-exact (same operation sequence)
        assert [repr(v) for v in p.qk_candidate_residuals] == c["qk_candidate_residuals"], where
        assert [repr(v) for v in p.vo_candidate_residuals] == c["vo_candidate_residuals"], where
        for name in ("c_qk", "c_vo", "b_qk", "b_vo"):
            assert sha(getattr(p, name)) == c[f"{name}_sha256"], (name, where)


def test_cfg1_prep_matches_reference_arrays():
    meta = json.loads((GOLDEN / "cfg1.json").read_text())
    g = np.load(GOLDEN / "cfg1.npz")
    w = bd.gen_random_mha(bd.Rng(7), 512, 64, 8, torch.float32)
    assert sha(w.w_k) == meta["w_k_sha256"]
    p = bd.bda_prepare(w, prepare_in_p64=True)
    assert p.qk_tag.value == meta["qk_tag"] and p.vo_tag.value == meta["vo_tag"]
    assert [repr(v) for v in p.qk_candidate_residuals] == meta["qk_candidate_residuals"]
    for name in ("b_qk", "c_qk", "c_vo", "b_vo"):
        np.testing.assert_array_equal(getattr(p, name).numpy(), g[name], err_msg=name)


def test_rand_gaussian_reproduces_reference_draw():
    meta = json.loads((GOLDEN / "cfg1.json").read_text())
    x = bd.rand_gaussian(bd.Rng(8), 256, 512, torch.float32)
    assert sha(x) == meta["x_sha256"]
    # derive() child streams are schedule-independent (ref tensor.py:394-396)
    a = bd.rand_gaussian(bd.Rng(3).derive(5), 4, 4)
    b = bd.rand_gaussian(bd.Rng(3).derive(5), 4, 4)
    torch.testing.assert_close(a, b, rtol=0, atol=0)


def test_linear_prep_matches_reference():
    meta = json.loads((GOLDEN / "linear_small.json").read_text())
    g = np.load(GOLDEN / "linear_small.npz")
    for i, m in enumerate(meta):
        layer = bd.LowRankLayer(u=torch.from_numpy(g[f"u{i}"]), v=torch.from_numpy(g[f"v{i}"]))
        conv = bd.bd_linear_from_lowrank(layer)
        assert conv.tag.value == m["tag"], m
        assert repr(conv.factors.residual) == m["residual"], m
        np.testing.assert_array_equal(conv.factors.basis, g[f"basis{i}"])
        np.testing.assert_array_equal(conv.factors.coeff, g[f"coeff{i}"])


def test_ordered_matmul_is_the_reference_rounding_sequence():
    rng = bd.Rng(3)
    a = bd.rand_gaussian(rng, 9, 6, torch.float32).numpy()
    b = bd.rand_gaussian(rng, 6, 11, torch.float32).numpy()
    want = np.zeros((9, 11), np.float32)
    for i in range(9):
        for j in range(11):
            acc = np.float32(0)
            for k in range(6):
                acc = np.float32(acc + np.float32(a[i, k] * b[k, j]))
            want[i, j] = acc
    np.testing.assert_array_equal(D.ordered_matmul(a, b), want)


def test_decompose_round_trip_and_cost_report():
    # ref test_decompose.py: rank-r products rebuild exactly (to tolerance) from BD factors
    rng = bd.Rng(11)
    u = bd.rand_gaussian(rng, 12, 3).numpy()
    v = bd.rand_gaussian(rng, 3, 10).numpy()
    w = u @ v
    for axis in bd.Axis:
        f = bd.bd_decompose(w, 3, axis)
        np.testing.assert_allclose(bd.bd_reconstruct(f), w, rtol=0, atol=1e-12)
        assert f.param_count == 3 * (12 + 10 - 3)
    r = bd.cost_report(12, 10, 3)
    assert (r.full_params, r.lowrank_params, r.bd_params) == (120, 66, 57)
    assert (r.lowrank_recon_flops, r.bd_recon_flops) == (720, 540)
    with pytest.raises(ValueError):
        bd.cost_report(4, 4, 4)


def test_select_tag_ties_go_first_and_force_first():
    w = bd.gen_random_mha(bd.Rng(1), 24, 4, 5)
    p = bd.bda_prepare(w, force_first=True)
    assert p.qk_tag is bd.Tag.FIRST and p.vo_tag is bd.Tag.FIRST
    assert p.param_count == 2 * 20 * 24 + 2 * 20 * 20


def test_weight_carriers_validate_like_the_reference():
    w = bd.gen_random_mha(bd.Rng(1), 16, 4, 2)
    with pytest.raises(bd.ShapeError):
        bd.MHAWeights(16, 2, 4, w.w_q[:, :4], w.w_k, w.w_v, w.w_o)
    with pytest.raises(ValueError):
        bd.MHAWeights(4, 1, 4, w.w_q, w.w_k, w.w_v, w.w_o)
    with pytest.raises(bd.PrecisionError):
        bd.MHAWeights(16, 2, 4, w.w_q.float(), w.w_k, w.w_v, w.w_o)
    assert w.param_count == 4 * 16 * 8


def test_reconstruction_error_report_matches_reference():
    """verify.reconstruction_error_report (ref verify.py:127-155) on the reference's own
    prepared factors: per-head MSE/NMSE and max-rel, both targets, P64 and P32 prep."""
    from paper_2510_01718_b200.verify import Target, reconstruction_error_report
    cases = json.loads((GOLDEN / "recon_report.json").read_text())
    assert len(cases) == 32
    for c in cases:
        w = bd.gen_random_mha(bd.Rng(c["seed"]), c["d"], c["d_h"], c["n_heads"], DT[c["precision"]])
        p = bd.bda_prepare(w, prepare_in_p64=c["prepare_in_p64"])
        r = reconstruction_error_report(w, p, Target(c["target"]))
        where = f"case {c['seed']} {c['d']}/{c['d_h']}/{c['n_heads']} {c['precision']} {c['target']}"
        assert r.precision == p.precision, where
        # same per-head products in the layer precision (platform BLAS, one thread) and
        # the same FP64 reductions: the report reproduces the reference bit for bit
        assert repr(r.mse) == c["mse"] and repr(r.nmse) == c["nmse"], where
        assert repr(r.max_rel) == c["max_rel"], where
        assert [[repr(a), repr(b)] for a, b in r.per_head] == c["per_head"], where
