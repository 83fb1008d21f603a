"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports bdattn 0.1.0 from /root/reference/pkg/src without writing into it
 and records, for the hot path:

  fused_small.npz  inputs + outputs of the reference fused op on the cases its own
                   tests use: the hand example and zero-C case (test_attention.py:175-185),
                   the 40 bit-identity trials (test_attention.py:187-203) and criterion 7's
                   100 random shapes (test_acceptance.py:175-196).
  cfg1.npz         BASELINE config 1: gen_random_mha(Rng(7), 512, 64, 8, P32) prepared with
                   bda_prepare(prepare_in_p64=True), x = rand_gaussian(Rng(8), 256, 512, P32):
                   the prepared matrices, tags, K'/V' outputs (as SHA-256 of their bytes +
                   the arrays), bda_forward and mha_forward outputs.
  prep_tags.json   tags and candidate mean residuals (repr of the floats) of bda_prepare on
                   small seeded models, so a port of the prep can be checked bit-exactly
                   for the selected basis S.
  linear_small.npz bd_linear_forward / lowrank_forward on small seeded layers.
  recon_report.json reconstruction_error_report (verify.py:127-155) of bda_prepare on
                   small seeded models, both targets, P64 and P32 (floats as repr).

The GPU box never reads /root/reference; tests read only these committed files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import bdattn as bd  # noqa: E402
from bdattn import Precision, Rng, Tag  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fused_small() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta = []

    def add(x, c, d_h, n, tag, source):
        out = bd.fused_kv_proj(x, c, d_h, n, tag)
        i = len(meta)
        arrays[f"x{i}"] = x.data
        arrays[f"c{i}"] = c.data
        arrays[f"out{i}"] = out.data
        meta.append({"d_h": d_h, "n_heads": n, "tag": tag.value, "dtype": str(x.data.dtype),
                     "source": source})

    # hand example (test_attention.py:182-185) and zero coefficients (:175-180)
    add(bd.Tensor2D([[2.0, 5.0]]), bd.Tensor2D([[3.0]]), 1, 1, Tag.FIRST, "hand_example")
    add(bd.rand_gaussian(Rng(13), 4, 10), bd.zeros(7, 9), 3, 3, Tag.FIRST, "zero_c")
    # bit-identity trials (test_attention.py:187-203)
    for tag in (Tag.FIRST, Tag.LAST):
        for precision in (Precision.P64, Precision.P32):
            rng = Rng(14)
            for trial in range(10):
                r = rng.derive(trial)
                d, d_h, n = 13, 4, 3
                x = bd.rand_gaussian(r, 6, d, precision)
                c = bd.rand_gaussian(r, d - d_h, n * d_h, precision)
                add(x, c, d_h, n, tag, f"bit_identity/{tag.value}/{precision.value}/{trial}")
    # criterion 7 (test_acceptance.py:175-196)
    for trial in range(100):
        rng = Rng(77).derive(trial)
        d_h = 2 + trial % 5
        n_heads = 1 + trial % 4
        d = d_h + 1 + trial % 9
        seq_len = 1 + trial % 8
        tag = Tag.FIRST if trial % 2 == 0 else Tag.LAST
        precision = Precision.P64 if trial % 3 else Precision.P32
        x = bd.rand_gaussian(rng, seq_len, d, precision)
        c = bd.rand_gaussian(rng, d - d_h, n_heads * d_h, precision)
        add(x, c, d_h, n_heads, tag, f"criterion07/{trial}")
    np.savez(OUT / "fused_small.npz", **arrays)
    (OUT / "fused_small.json").write_text(json.dumps(meta, indent=0) + "\n")
    print(f"fused_small: {len(meta)} cases")


def cfg1() -> None:
    w = bd.gen_random_mha(Rng(7), 512, 64, 8, Precision.P32)
    p = bd.bda_prepare(w, prepare_in_p64=True)
    x = bd.rand_gaussian(Rng(8), 256, 512, Precision.P32)
    k = bd.fused_kv_proj(x, p.c_qk, p.d_h, p.n_heads, p.qk_tag)
    v = bd.fused_kv_proj(x, p.c_vo, p.d_h, p.n_heads, p.vo_tag)
    bda = bd.bda_forward(x, p)
    mha = bd.mha_forward(x, w)
    np.savez(
        OUT / "cfg1.npz",
        b_qk=p.b_qk.data, c_qk=p.c_qk.data, c_vo=p.c_vo.data, b_vo=p.b_vo.data,
        k_out=k.data, v_out=v.data, bda_out=bda.data, mha_out=mha.data,
    )
    meta = {
        "model": "gen_random_mha(Rng(7), 512, 64, 8, P32); bda_prepare(prepare_in_p64=True)",
        "x": "rand_gaussian(Rng(8), 256, 512, P32)",
        "x_sha256": sha(x.data),
        "w_k_sha256": sha(w.w_k.data),
        "qk_tag": p.qk_tag.value, "vo_tag": p.vo_tag.value,
        "qk_candidate_residuals": [repr(v_) for v_ in p.qk_candidate_residuals],
        "vo_candidate_residuals": [repr(v_) for v_ in p.vo_candidate_residuals],
        "k_out_sha256": sha(k.data), "v_out_sha256": sha(v.data),
        "bda_vs_mha_max_rel": bd.max_relative_error(bda, mha),
    }
    (OUT / "cfg1.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("cfg1:", meta["qk_tag"], meta["vo_tag"], meta["bda_vs_mha_max_rel"])


def prep_tags() -> None:
    cases = []
    for seed in range(8):
        for (d, d_h, n) in ((64, 16, 4), (24, 4, 5)):
            for precision, p64 in ((Precision.P64, False), (Precision.P32, True)):
                w = bd.gen_random_mha(Rng(seed), d, d_h, n, precision)
                p = bd.bda_prepare(w, prepare_in_p64=p64)
                cases.append({
                    "seed": seed, "d": d, "d_h": d_h, "n_heads": n,
                    "precision": precision.value, "prepare_in_p64": p64,
                    "qk_tag": p.qk_tag.value, "vo_tag": p.vo_tag.value,
                    "qk_candidate_residuals": [repr(v) for v in p.qk_candidate_residuals],
                    "vo_candidate_residuals": [repr(v) for v in p.vo_candidate_residuals],
                    "c_qk_sha256": sha(p.c_qk.data), "c_vo_sha256": sha(p.c_vo.data),
                    "b_qk_sha256": sha(p.b_qk.data), "b_vo_sha256": sha(p.b_vo.data),
                })
    (OUT / "prep_tags.json").write_text(json.dumps(cases, indent=0) + "\n")
    print(f"prep_tags: {len(cases)} cases")


def linear_small() -> None:
    arrays = {}
    meta = []
    for i, (d_in, d_out, r, seed) in enumerate(((8, 12, 3, 1000), (64, 16, 7, 2), (16, 64, 8, 3),
                                                 (32, 32, 16, 4))):
        rng = Rng(seed)
        layer = bd.LowRankLayer(u=bd.rand_gaussian(rng, d_in, r), v=bd.rand_gaussian(rng, d_out, r))
        conv = bd.bd_linear_from_lowrank(layer)
        x = bd.rand_gaussian(rng, 6, d_in)
        arrays[f"u{i}"] = layer.u.data
        arrays[f"v{i}"] = layer.v.data
        arrays[f"basis{i}"] = conv.factors.basis.data
        arrays[f"coeff{i}"] = conv.factors.coeff.data
        arrays[f"x{i}"] = x.data
        arrays[f"y{i}"] = bd.bd_linear_forward(x, conv).data
        arrays[f"ylr{i}"] = bd.lowrank_forward(x, layer).data
        meta.append({"d_in": d_in, "d_out": d_out, "rank": r, "seed": seed,
                     "tag": conv.tag.value, "residual": repr(conv.factors.residual)})
    np.savez(OUT / "linear_small.npz", **arrays)
    (OUT / "linear_small.json").write_text(json.dumps(meta, indent=0) + "\n")
    print(f"linear_small: {len(meta)} cases")


def recon_report() -> None:
    from bdattn.verify import Target, reconstruction_error_report
    cases = []
    for seed in range(4):
        for (d, d_h, n) in ((64, 16, 4), (24, 4, 5)):
            for precision, p64 in ((Precision.P64, False), (Precision.P32, True)):
                w = bd.gen_random_mha(Rng(100 + seed), d, d_h, n, precision)
                p = bd.bda_prepare(w, prepare_in_p64=p64)
                for target in (Target.QK, Target.VO):
                    r = reconstruction_error_report(w, p, target)
                    cases.append({
                        "seed": 100 + seed, "d": d, "d_h": d_h, "n_heads": n,
                        "precision": precision.value, "prepare_in_p64": p64,
                        "target": target.value, "mse": repr(r.mse), "nmse": repr(r.nmse),
                        "max_rel": repr(r.max_rel),
                        "per_head": [[repr(a), repr(b)] for a, b in r.per_head],
                    })
    (OUT / "recon_report.json").write_text(json.dumps(cases, indent=0) + "\n")
    print(f"recon_report: {len(cases)} cases")


def bundle() -> None:
    """A prepared bundle written by the reference's own tensorio (`bdattn prepare`
    output format): MHA and BDA manifests + BDT1 files for a small seeded model."""
    from bdattn import tensorio
    out = OUT / "bundle"
    out.mkdir(exist_ok=True)
    w = bd.gen_random_mha(Rng(21), 24, 4, 5, Precision.P32)
    p = bd.bda_prepare(w, prepare_in_p64=True)
    tensorio.save_mha_manifest(out / "model.mha", w)
    tensorio.save_bda_manifest(out / "model.bda", p)
    print("bundle:", sorted(f.name for f in out.iterdir()))


if __name__ == "__main__":
    import sys as _sys
    todo = _sys.argv[1:] or ["fused_small", "cfg1", "prep_tags", "linear_small", "recon_report",
                             "bundle"]
    for name in todo:
        globals()[name]()
