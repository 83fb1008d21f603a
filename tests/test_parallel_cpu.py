"""Head-sharded projection and block over torch.distributed — world size 2, gloo, CPU.

The compute is injected (``parallel.Ops``) from the CPU oracle so the host-side
sharding, the head-major all-gather and the all-reduce are exercised without a GPU;
on the GPU box the same functions run with the default CUDA ops (bench.py, NCCL).
Invariants: gathered shards are bit-identical to the unsharded oracle output (and to
the reference's cfg1 K'/V' hashes); the sharded block equals the unsharded block.
"""

import hashlib
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
import torch.nn.functional as F

from conftest import GOLDEN, ROOT
import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import parallel as P


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def cpu_ops():
    """Oracle-backed CPU compute for the tests (never the product default)."""
    import sys
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O

    def kv(x, specs, out_layout="token"):
        outs = []
        for c, d_h, n, tag in specs:
            o = torch.from_numpy(O.fused_kv_proj_ref(x.numpy(), c.numpy(), d_h, n, tag.value))
            if out_layout == "head":
                o = o.view(-1, n, d_h).permute(1, 0, 2).contiguous()
            outs.append(o)
        return outs

    def proj(x, w):
        return x @ w

    def attend(q, k, v, n, d_h, causal=False):
        L = q.shape[0]
        qh, kh, vh = (t.view(L, n, d_h).transpose(0, 1) for t in (q, k, v))
        o = F.scaled_dot_product_attention(qh, kh, vh, is_causal=causal, scale=d_h ** -0.5)
        return o.transpose(0, 1).reshape(L, n * d_h)

    return P.Ops(kv_proj_grouped=kv, proj=proj, attend=attend)


def test_head_range_and_shards():
    assert [P.head_range(16, 4, r) for r in range(4)] == [(0, 4), (4, 8), (8, 12), (12, 16)]
    with pytest.raises(ValueError):
        P.head_range(16, 3, 0)
    c = torch.arange(3 * 8.0).view(3, 8)
    torch.testing.assert_close(P.shard_columns(c, 2, 4, 2, 1), c[:, 4:8])
    assert P.weak_scaling_tokens(8192, 8) == 65536
    assert P.flops_per_rank(8192, 512, 128, 16, 8) == 2 * 2 * 8192 * 384 * 2 * 128


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
        r, w, _ = P.init_from_env("gloo")
        ops = cpu_ops()
        # --- projection: cfg1 prepared model (reference goldens), heads sharded
        g = np.load(GOLDEN / "cfg1.npz")
        meta = json.loads((GOLDEN / "cfg1.json").read_text())
        x = bd.rand_gaussian(bd.Rng(8), 256, 512, torch.float32)
        res = {}
        for name, tag in (("c_qk", meta["qk_tag"]), ("c_vo", meta["vo_tag"])):
            c = torch.from_numpy(g[name])
            local = P.sharded_kv_proj(x, P.shard_columns(c, 64, 8, w, r), 64, bd.Tag(tag), ops=ops)
            assert local.shape == (256, 8 // w * 64)
            full = P.all_gather_heads(local, 64)
            res[name] = hashlib.sha256(full.numpy().tobytes()).hexdigest()
            # head-major straight from the kernel: gathered with no staging copy
            hm = P.sharded_kv_proj(x, P.shard_columns(c, 64, 8, w, r), 64, bd.Tag(tag), ops=ops,
                                   head_major=True)
            fh = P.all_gather_heads(hm, 64)
            assert fh.shape == (8, 256, 64)
            assert torch.equal(fh.permute(1, 0, 2).reshape(256, 512), full)
        # --- block: global prep, then shard; compare with the unsharded block
        mha = bd.gen_random_mha(bd.Rng(3), 48, 8, 4, torch.float64)
        prepared = bd.bda_prepare(mha)
        xb = bd.rand_gaussian(bd.Rng(4), 12, 48, torch.float64)
        part = P.sharded_bda_forward(xb, P.shard_bda_weights(prepared, w, r), causal=True, ops=ops)
        res["block"] = part.numpy()
        res["k_ok"] = res["c_qk"] == meta["k_out_sha256"]
        res["v_ok"] = res["c_vo"] == meta["v_out_sha256"]
        q.put((rank, res))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_two_rank_gloo_sharded_projection_and_block():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(results[r], dict), results[r]
        assert results[r]["k_ok"] and results[r]["v_ok"], "gathered K'/V' differ from reference"
    # the all-reduced block is identical on both ranks and equals the unsharded block
    np.testing.assert_array_equal(results[0]["block"], results[1]["block"])
    mha = bd.gen_random_mha(bd.Rng(3), 48, 8, 4, torch.float64)
    prepared = bd.bda_prepare(mha)
    xb = bd.rand_gaussian(bd.Rng(4), 12, 48, torch.float64)
    single = P.sharded_bda_forward(xb, prepared, causal=True, ops=cpu_ops())
    np.testing.assert_allclose(results[0]["block"], single.numpy(), rtol=0, atol=1e-12)
    # and the block is the attention it replaces (BD is exact in FP64)
    ops = cpu_ops()
    q_, k_, v_ = xb @ mha.w_q, xb @ mha.w_k, xb @ mha.w_v
    dense = ops.attend(q_, k_, v_, 4, 8, True) @ mha.w_o
    assert bd.max_relative_error(torch.from_numpy(results[0]["block"]), dense) <= 1e-10


# ----------------------------------------------------------------------------- MLA block
def _bd_mla_block_cpu(hidden, w, fused):
    """The BD MLA block's math on the CPU in float64 (the GPU path is mla.bd_mla_forward):
    K'/V' from the latent through the BD projection — with kv_a_layernorm folded into the
    coefficients (``fused``, w.norm_fold) or applied first — and explicit causal softmax
    attention; returns this (possibly head-sharded) block's partial output."""
    from paper_2510_01718_b200 import mla as M
    cfg, H = w.cfg, w.n_heads
    L = hidden.shape[0]
    r, dn, dv, dr = cfg.kv_lora_rank, cfg.qk_nope, cfg.v_head, cfg.qk_rope
    rope = lambda t: M._rope(t, cfg.rope_theta, cfg.rope_interleaved)  # noqa: E731
    q = (hidden @ w.w_q).view(L, H, dn + dr)
    q_nope, q_pe = q[..., :dn], rope(q[..., dn:])
    kv = hidden @ w.w_kva
    x, k_pe = kv[:, :r], rope(kv[:, r:])

    def proj(c, d_h, tag, gamma_rep=None):
        mul, rep = bd.tag_offsets(r, d_h, tag)
        K = r - d_h
        outs = []
        for h in range(H):
            ch = c[:, h * d_h:(h + 1) * d_h]
            if fused:  # r_i * (x[:, mul] c_g + gamma_rep * x[:, rep])
                rr = torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + cfg.rms_eps)
                outs.append(rr * (x[:, mul:mul + K] @ ch + gamma_rep.double() * x[:, rep:rep + d_h]))
            else:
                xn = M._rms_norm(x, w.kva_norm, cfg.rms_eps)
                outs.append(xn[:, rep:rep + d_h] + xn[:, mul:mul + K] @ ch)
        return torch.stack(outs, 1)  # [L, H, d_h]

    if fused:
        cq, cv, gq, gv = w.norm_fold
        k_nope, v = proj(cq, dn, w.qk_tag, gq), proj(cv, dv, w.vo_tag, gv)
    else:
        k_nope, v = proj(w.c_qk, dn, w.qk_tag), proj(w.c_vo, dv, w.vo_tag)
    scale = 1.0 / (dn + dr) ** 0.5
    mask = torch.ones(L, L, dtype=torch.bool).triu(1)
    o = []
    for h in range(H):
        s = (q_nope[:, h] @ k_nope[:, h].T + q_pe[:, h] @ k_pe.T) * scale
        o.append(torch.softmax(s.masked_fill(mask, float("-inf")), -1) @ v[:, h])
    return torch.cat(o, 1) @ w.b_vo


def _dense_mla_block_cpu(hidden, w):
    """The dense block it replaces (original kv_b_proj), float64, same attention code."""
    from paper_2510_01718_b200 import mla as M
    cfg, H = w.cfg, w.cfg.n_heads
    L = hidden.shape[0]
    r, dn, dv, dr = cfg.kv_lora_rank, cfg.qk_nope, cfg.v_head, cfg.qk_rope
    rope = lambda t: M._rope(t, cfg.rope_theta, cfg.rope_interleaved)  # noqa: E731
    q = (hidden @ w.w_q).view(L, H, dn + dr)
    kv = hidden @ w.w_kva
    c_kv = M._rms_norm(kv[:, :r], w.kva_norm, cfg.rms_eps)
    kvb = (c_kv @ w.w_kvb).view(L, H, dn + dv)
    k_pe = rope(kv[:, r:])
    scale = 1.0 / (dn + dr) ** 0.5
    mask = torch.ones(L, L, dtype=torch.bool).triu(1)
    o = []
    for h in range(H):
        s = (q[:, h, :dn] @ kvb[:, h, :dn].T + rope(q[:, h:h + 1, dn:])[:, 0] @ k_pe.T) * scale
        o.append(torch.softmax(s.masked_fill(mask, float("-inf")), -1) @ kvb[:, h, dn:])
    return torch.cat(o, 1) @ w.w_o


def _mla_setup():
    from paper_2510_01718_b200 import mla as M
    cfg = M.MLAConfig(hidden=64, n_heads=4, kv_lora_rank=64, qk_nope=16, qk_rope=8, v_head=16)
    w = M.gen_random_mla(7, cfg)
    g = torch.Generator().manual_seed(8)
    from dataclasses import replace
    w = replace(w, kva_norm=1 + 0.2 * torch.randn(cfg.kv_lora_rank, generator=g, dtype=torch.float64))
    hidden = torch.randn(12, cfg.hidden, generator=g, dtype=torch.float64)
    return w, M.mla_prepare(w), hidden


def _mla_worker(rank, world, port, q):
    try:
        from paper_2510_01718_b200 import mla as M
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
        r, w_, _ = P.init_from_env("gloo")
        _, p, hidden = _mla_setup()
        local = M.shard_bd_mla(p, w_, r)
        res = {"n_heads": local.n_heads}
        for fused in (True, False):
            part = _bd_mla_block_cpu(hidden, local, fused)
            dist.all_reduce(part)
            res[f"block_{fused}"] = part.numpy()
        q.put((rank, res))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_two_rank_gloo_sharded_bd_mla_block():
    """shard_bd_mla (q columns, C_qk / C_vo columns, the folded-norm coefficients, B_vo
    rows) over a world-size-2 gloo group: the all-reduced partial blocks are identical on
    both ranks, equal the unsharded BD block (to float64 summation order) and the dense
    block it replaces — with kv_a_layernorm folded into the coefficients and applied
    first."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mla_worker, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p_ in procs:
        p_.join(timeout=60)
    for r in range(world):
        assert isinstance(results[r], dict), results[r]
        assert results[r]["n_heads"] == 2
    w, p, hidden = _mla_setup()
    dense = _dense_mla_block_cpu(hidden, w)
    for fused in (True, False):
        np.testing.assert_array_equal(results[0][f"block_{fused}"], results[1][f"block_{fused}"])
        single = _bd_mla_block_cpu(hidden, p, fused).numpy()
        np.testing.assert_allclose(results[0][f"block_{fused}"], single, rtol=0, atol=1e-12)
        # float64 BD vs dense: 2.1e-8 (fused norm) / 7.0e-9 measured — the random 16 x 16
        # basis blocks' condition number amplifies float64 rounding
        err = bd.max_relative_error(torch.from_numpy(single), dense)
        assert err <= 1e-7, (fused, err)
