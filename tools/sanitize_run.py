"""Small invocations of every kernel variant, for compute-sanitizer (memcheck,
synccheck, racecheck, initcheck) — tools/gpu_sanitize.sh runs each tool over it.

Variants: exact kernel (FP32/FP64), persistent CTA-pair tcgen05 kernel (contiguous
and round-robin schedules, token- and head-major output, non-finite check), small-L
kernel (single CTA and CTA pair), fused-RMSNorm (kNorm) variant, fused all-gather
epilogue (single-device ranks), BD low-rank layer.  Each result is checked against a
float64 torch evaluation so a sanitizer run is also a correctness run.
"""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2510_01718_b200 as bd  # noqa: E402
from paper_2510_01718_b200 import parallel as P  # noqa: E402


def ref(x, c, d_h, n, tag):
    mul, rep = bd.tag_offsets(x.shape[1], d_h, tag)
    K = c.shape[0]
    xd = x.double()
    return xd[:, mul:mul + K] @ c.double() + xd[:, rep:rep + d_h].repeat(1, n)


def check(got, want, tol):
    err = float((got.double() - want).abs().max() / want.abs().max())
    assert err <= tol, err


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(0)
    for dt, tol in ((torch.float32, 1e-6), (torch.float64, 1e-13)):   # exact kernel
        x = torch.randn(70, 100, generator=g).to(dt).to(dev)
        c = torch.randn(76, 72, generator=g).to(dt).to(dev)
        check(bd.fused_kv_proj(x, c, 24, 3, bd.Tag.LAST), ref(x, c, 24, 3, bd.Tag.LAST), tol)
        # the 64 x 64 (L = 600) and 128 x 128 (L = 2400: >= 2 tiles per SM) tile kernels,
        # ragged edges (K = 125, N = 2040)
        for L in (600, 2400):
            x = torch.randn(L, 133, generator=g).to(dt).to(dev)
            c = torch.randn(125, 2040, generator=g).to(dt).to(dev)
            check(bd.fused_kv_proj(x, c, 8, 255, bd.Tag.FIRST), ref(x, c, 8, 255, bd.Tag.FIRST),
                  tol)
    for dt in (torch.float16, torch.bfloat16):
        tol = 2e-3 if dt == torch.float16 else 1.6e-2
        # persistent pair kernel, contiguous schedule, 2 problems, check on
        x = torch.randn(600, 512, generator=g).to(dt).to(dev)
        ck = (torch.randn(384, 1024, generator=g) / 8).to(dt).to(dev)
        cv = (torch.randn(384, 1024, generator=g) / 8).to(dt).to(dev)
        k, v = bd.fused_kv_proj_grouped(x, [(ck, 128, 8, bd.Tag.FIRST), (cv, 128, 8, bd.Tag.LAST)])
        check(k, ref(x, ck, 128, 8, bd.Tag.FIRST), tol)
        check(v, ref(x, cv, 128, 8, bd.Tag.LAST), tol)
        kh, = bd.fused_kv_proj_grouped(x, [(ck, 128, 8, bd.Tag.FIRST)], out_layout="head")
        assert torch.equal(kh, k.view(600, 8, 128).transpose(0, 1))
        # round-robin schedule (K > 384 streams A), mixed d_h
        x2 = torch.randn(300, 480, generator=g).to(dt).to(dev)
        c8 = (torch.randn(472, 64, generator=g) / 8).to(dt).to(dev)
        c128 = (torch.randn(352, 512, generator=g) / 8).to(dt).to(dev)
        a, b = bd.fused_kv_proj_grouped(x2, [(c8, 8, 8, bd.Tag.FIRST), (c128, 128, 4, bd.Tag.LAST)])
        check(a, ref(x2, c8, 8, 8, bd.Tag.FIRST), tol)
        check(b, ref(x2, c128, 128, 4, bd.Tag.LAST), tol)
        # small-L kernel: one row block (L <= 128) and two 128-row blocks (L = 200)
        for L in (40, 200):
            k, v = bd.fused_kv_proj_grouped(x[:L].contiguous(), [(ck, 128, 8, bd.Tag.FIRST),
                                                                 (cv, 128, 8, bd.Tag.LAST)])
            check(k, ref(x[:L], ck, 128, 8, bd.Tag.FIRST), tol)
        # small-L kernel, 32- and 160-column blocks (4096 columns: L = 100 and L = 600)
        cw = (torch.randn(384, 2048, generator=g) / 8).to(dt).to(dev)
        for L in (100, 600):
            k, v = bd.fused_kv_proj_grouped(x[:L].contiguous(), [(cw, 128, 16, bd.Tag.FIRST),
                                                                 (cw, 128, 16, bd.Tag.LAST)])
            check(v, ref(x[:L], cw, 128, 16, bd.Tag.LAST), tol)
        # fused RMSNorm variant
        gamma = (0.5 + torch.rand(512, generator=g)).to(dev)
        fk = bd.fold_rmsnorm(ck, gamma, 128, bd.Tag.FIRST)
        fv = bd.fold_rmsnorm(cv, gamma, 128, bd.Tag.LAST)
        k, v = bd.fused_rmsnorm_kv_proj_grouped(
            x, [(fk[0], fk[1], 128, 8, bd.Tag.FIRST), (fv[0], fv[1], 128, 8, bd.Tag.LAST)], 1e-6)
        assert bool(torch.isfinite(k).all())
        # fused all-gather epilogue, two "ranks" on one device
        full = bd.fused_kv_proj_grouped(x, [(ck, 128, 8, bd.Tag.FIRST)], out_layout="head")[0]
        bufs = [[torch.zeros(8, 600, 128, dtype=dt, device=dev) for _ in range(2)]]
        for r in range(2):
            P.fused_allgather_kv_proj(x, [(P.shard_columns(ck, 128, 8, 2, r), 128, 4,
                                           bd.Tag.FIRST)], bufs, r)
        assert torch.equal(bufs[0][0], full) and torch.equal(bufs[0][1], full)
    # BD low-rank layer (two plain-GEMM launches)
    basis = (torch.randn(256, 64, generator=g) / 16).half().to(dev)
    coeff = (torch.randn(64, 192, generator=g) / 8).half().to(dev)
    fac = bd.BDFactors(axis=bd.Axis.COLUMN, tag=bd.Tag.FIRST, basis=basis.double().cpu().numpy(),
                       coeff=coeff.double().cpu().numpy(), orig_rows=256, orig_cols=256, rank=64,
                       residual=0.0, rank_deficient=False)
    y = bd.bd_linear_forward(torch.randn(300, 256, generator=g).half().to(dev),
                             bd.BDLinearLayer(fac, basis, coeff))
    assert bool(torch.isfinite(y).all())
    # tcgen05 MLA prefill attention (csrc/mla_attn.cu): causal with a ragged last tile,
    # non-causal, a strided q view; FP16 and BF16, vs float64
    from paper_2510_01718_b200 import mla as M
    for dt in (torch.float16, torch.bfloat16):
        for L, H, causal in ((300, 2, True), (200, 3, False)):
            q = torch.randn(L, H, 192, generator=g).to(dt).to(dev)
            kn = torch.randn(H, L, 128, generator=g).to(dt).to(dev)
            kpe = torch.randn(L, 64, generator=g).to(dt).to(dev)
            vv = torch.randn(H, L, 128, generator=g).to(dt).to(dev)
            sc = 1.0 / 192 ** 0.5
            o = M.mla_attention(q, kn, kpe, vv, scale=sc, causal=causal)
            qd, kd, pd, vd = (t.double() for t in (q, kn, kpe, vv))
            for h in range(H):
                sm = (qd[:, h, :128] @ kd[h].T + qd[:, h, 128:] @ pd.T) * sc
                if causal:
                    sm.masked_fill_(torch.ones(L, L, dtype=torch.bool, device=dev).triu(1),
                                    float("-inf"))
                err = float((o[:, h].double() - torch.softmax(sm, -1) @ vd[h]).abs().max())
                assert err < (2e-2 if dt == torch.bfloat16 else 3e-3), (dt, L, H, h, err)
        wide = torch.randn(256, 4, 256, generator=g).to(dt).to(dev)[..., :192]
        o = M.mla_attention(wide, torch.randn(4, 256, 128, generator=g).to(dt).to(dev),
                            torch.randn(256, 64, generator=g).to(dt).to(dev),
                            torch.randn(4, 256, 128, generator=g).to(dt).to(dev), scale=0.07)
        assert bool(torch.isfinite(o).all())
    torch.cuda.synchronize()
    print("sanitize_run: all variants ok")


if __name__ == "__main__":
    main()
