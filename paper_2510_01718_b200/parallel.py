"""Head-parallel sharding of the BD projection and the BDA block (one process per GPU).

The projection shards naturally: output column j depends only on column j of C, and
the per-element reduction order does not depend on how N is split (the reference
tests exactly this invariance, ref test_tensor.py:113-119; our kernels keep it — see
tests/test_kv_proj_gpu.py::test_tc_head_shards_are_bit_identical).  So rank r of g
owns heads [r n/g, (r+1) n/g): the contiguous column slice of c_qk / c_vo in the
reference layout, of b_qk's columns and of b_vo's rows.  x is replicated.

* Head-parallel consumers (per-head attention) need NO collective: ``sharded_kv_proj``
  returns the local heads only.
* When a full-width K'/V' is required, ``all_gather_heads`` runs ONE NCCL
  ``all_gather_into_tensor`` on the head-major layout [n_local, L, d_h] (contiguous per
  rank) and returns the token-major [L, n d_h] view.
* The block (``sharded_bda_forward``) computes its heads' attention and its rows of
  the output projection, then ONE ``all_reduce`` sums the partial outputs.

The tag (the basis S) must be chosen over ALL heads before sharding: the reference's
``_select_tag`` averages residuals across heads (ref attention.py:181-189), so
``shard_bda_weights`` slices an already-prepared ``BDAWeights``.

Compute goes through ``ops`` (default: the CUDA kernels).  The CPU multi-process tests
(gloo, world size 2) inject CPU ops so the host-side sharding logic is covered without
a GPU; the product default never runs on the CPU.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

import ctypes

from . import _native as N
from .attention import BDAWeights, _attend, _proj
from .decompose import Tag
from .kv_proj import (_DTYPES, _MODES, _check, _on_device, _problem, _rowmajor,
                      fused_kv_proj_grouped)


def head_range(n_heads: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous heads of `rank`; every rank gets n_heads / world (must divide)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if n_heads % world:
        raise ValueError(f"{n_heads} heads do not shard evenly over {world} ranks")
    per = n_heads // world
    return rank * per, (rank + 1) * per


def shard_columns(c: torch.Tensor, d_h: int, n_heads: int, world: int, rank: int) -> torch.Tensor:
    """Column slice of a (rows x n_heads d_h) matrix for `rank`'s heads (contiguous copy)."""
    h0, h1 = head_range(n_heads, world, rank)
    return c[:, h0 * d_h:h1 * d_h].contiguous()


def shard_bda_weights(w: BDAWeights, world: int, rank: int) -> BDAWeights:
    """The rank's slice of a prepared BDA model (tags are global, chosen before)."""
    h0, h1 = head_range(w.n_heads, world, rank)
    lo, hi = h0 * w.d_h, h1 * w.d_h
    return BDAWeights(
        d=w.d, n_heads=h1 - h0, d_h=w.d_h,
        b_qk=w.b_qk[:, lo:hi].contiguous(), c_qk=w.c_qk[:, lo:hi].contiguous(),
        c_vo=w.c_vo[:, lo:hi].contiguous(), b_vo=w.b_vo[lo:hi, :].contiguous(),
        qk_tag=w.qk_tag, vo_tag=w.vo_tag,
        qk_candidate_residuals=w.qk_candidate_residuals,
        vo_candidate_residuals=w.vo_candidate_residuals,
        qk_deficient_heads=tuple(h - h0 for h in w.qk_deficient_heads if h0 <= h < h1),
        vo_deficient_heads=tuple(h - h0 for h in w.vo_deficient_heads if h0 <= h < h1))


@dataclass
class Ops:
    """The compute the sharded paths call.  Default = the CUDA kernels."""

    kv_proj_grouped: Callable = fused_kv_proj_grouped
    proj: Callable = _proj
    attend: Callable = _attend


GPU_OPS = Ops()


def sharded_kv_proj(x: torch.Tensor, c_local: torch.Tensor, d_h: int, tag: Tag,
                    *, ops: Ops = GPU_OPS, head_major: bool = False) -> torch.Tensor:
    """This rank's heads of K'; no collective.  Token-major [L, n_local d_h], or with
    ``head_major`` the kernel writes [n_local, L, d_h] directly (per-head contiguous:
    what head-parallel attention and ``all_gather_heads`` consume without a copy)."""
    n_local = c_local.shape[1] // d_h
    if head_major:
        return ops.kv_proj_grouped(x, [(c_local, d_h, n_local, tag)], out_layout="head")[0]
    return ops.kv_proj_grouped(x, [(c_local, d_h, n_local, tag)])[0]


def all_gather_heads(local: torch.Tensor, d_h: int, group=None) -> torch.Tensor:
    """Full width from every rank's heads, heads in rank order.

    One ``all_gather_into_tensor`` over the head-major layout: each rank contributes a
    contiguous [n_local, L, d_h] block, so the collective is a single flat gather.  A
    head-major local (3-D, straight from the kernel) gathers without any copy and
    returns [n, L, d_h]; a token-major local is staged and [L, n d_h] returned.
    """
    world = dist.get_world_size(group)
    if local.dim() == 3:  # already head-major from the kernel: gather in place, no copy
        n_local, L, _ = local.shape
        full = torch.empty((world * n_local, L, d_h), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(full, local, group=group)
        return full
    L, w = local.shape
    n_local = w // d_h
    head_major = local.view(L, n_local, d_h).permute(1, 0, 2).contiguous()
    full = torch.empty((world * n_local, L, d_h), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(full, head_major, group=group)
    return full.permute(1, 0, 2).reshape(L, world * n_local * d_h)


def fused_allgather_kv_proj(x: torch.Tensor,
                            specs: list[tuple[torch.Tensor, int, int, Tag]],
                            gathered: list[list[torch.Tensor]], rank: int, *,
                            mode: str = "auto") -> None:
    """Head-parallel projection with the all-gather fused into the kernel's epilogue.

    ``specs`` are this rank's (c_local, d_h, n_local, tag) problems; ``gathered[p][r]`` is
    rank r's full-width head-major buffer [world * n_local, L, d_h] for problem p — peer
    memory (``SymmetricGather`` below) on a multi-GPU node, any device tensors for a
    single-device check.  The kernel writes this rank's heads into planes
    [rank * n_local, (rank + 1) * n_local) of EVERY buffer over NVLink as it produces
    them (TMA stores to peer addresses), so the transfer overlaps the math tile by tile
    and no NCCL collective follows.  Readers must synchronise with all ranks afterwards
    (``SymmetricGather.barrier``).
    """
    world = len(gathered[0])
    if not 1 <= world <= N.BD_MAX_PEERS or not 0 <= rank < world:
        raise ValueError(f"world must be in [1, {N.BD_MAX_PEERS}] and 0 <= rank < world")
    x = _rowmajor(x)
    L = int(x.shape[0])
    probs = (N.KvProblem * len(specs))()
    ptrs = (ctypes.c_void_p * (len(specs) * world))()
    for i, (c, d_h, n, tag) in enumerate(specs):
        _check(x, c, d_h, n)
        c = _rowmajor(c)
        for r, g in enumerate(gathered[i]):
            if tuple(g.shape) != (world * n, L, d_h) or g.dtype != x.dtype or not g.is_contiguous():
                raise ValueError(f"gathered[{i}][{r}] must be a contiguous {(world * n, L, d_h)} "
                                 f"{x.dtype} tensor")
            ptrs[i * world + r] = g.data_ptr()
        probs[i] = _problem(x, c, gathered[i][rank][rank * n:(rank + 1) * n], d_h, n, tag)
    st = _on_device(x.device, N.load().bd_kv_proj_grouped_allgather, probs, len(specs),
                    _DTYPES[x.dtype], _MODES[mode], world, rank, ptrs, None)
    N.check(st, "bd_kv_proj_grouped_allgather")


class SymmetricGather:
    """Per-problem full-width gather buffers in torch symmetric memory (one allocation
    per rank, peer-mapped over NVLink) for ``fused_allgather_kv_proj``."""

    def __init__(self, shapes: list[tuple[int, int, int]], dtype, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        self.group = group if group is not None else dist.group.WORLD
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.local, self.handles, self.peers = [], [], []
        for shape in shapes:
            buf = symm_mem.empty(shape, dtype=dtype, device=dev)
            hdl = symm_mem.rendezvous(buf, self.group)
            self.local.append(buf)
            self.handles.append(hdl)
            self.peers.append([hdl.get_buffer(r, shape, dtype) for r in range(self.world)])

    def barrier(self) -> None:
        """Every rank's writes into every buffer are complete and visible."""
        self.handles[0].barrier()


def sharded_bda_forward(x: torch.Tensor, w_local: BDAWeights, *, causal: bool = False,
                        group=None, ops: Ops = GPU_OPS) -> torch.Tensor:
    """BDA block with heads sharded over the group: local Q', K', V' (K' and V' in one
    launch), local attention, local rows of B_vo, then one all_reduce of the partial
    outputs (ref attention.py:298-307 computes the unsharded block)."""
    q = ops.proj(x, w_local.b_qk)
    k, v = ops.kv_proj_grouped(x, [(w_local.c_qk, w_local.d_h, w_local.n_heads, w_local.qk_tag),
                                   (w_local.c_vo, w_local.d_h, w_local.n_heads, w_local.vo_tag)])
    partial = ops.proj(ops.attend(q, k, v, w_local.n_heads, w_local.d_h, causal), w_local.b_vo)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial, group=group)
    return partial


def init_from_env(backend: str | None = None) -> tuple[int, int, int]:
    """(rank, world, local_rank) from torchrun's env; initialises the process group
    (NCCL on GPUs, gloo otherwise) when world > 1."""
    import os
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend, **kw)
    return rank, world, local


def weak_scaling_tokens(tokens_per_gpu: int, world: int) -> int:
    """Head-sharded weak scaling keeps per-GPU work fixed: every rank projects all
    tokens for n/g heads, so total tokens grow with g (work per GPU = L n/g)."""
    return int(tokens_per_gpu) * int(world)


def flops_per_rank(L: int, d: int, d_h: int, n_heads: int, world: int) -> int:
    """Multiply-FLOPs of K' + V' on one rank of a head-sharded group."""
    return 2 * 2 * L * (d - d_h) * (n_heads // world) * d_h


__all__ = ["head_range", "shard_columns", "shard_bda_weights", "Ops", "GPU_OPS",
           "sharded_kv_proj", "all_gather_heads", "fused_allgather_kv_proj", "SymmetricGather",
           "sharded_bda_forward", "init_from_env", "weak_scaling_tokens", "flops_per_rank"]
