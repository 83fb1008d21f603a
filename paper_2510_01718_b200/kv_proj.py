"""The BD K/V projection operator — the drop-in for ``bdattn.fused_kv_proj``.

    K'_h = X[:, S] + X[:, ~S] @ C_h          (ref: pkg/src/bdattn/attention.py:273-295)

``fused_kv_proj`` keeps the reference's name, argument meaning, tag semantics and
check order (PrecisionError, then ShapeError for c's rows, then for c's cols;
attention.py:283-288) and raises ``ValueError`` on a non-finite result like the
reference's ``Tensor2D._wrap`` (tensor.py:112-113).  Tensors are torch CUDA tensors;
the arithmetic runs in the C-ABI library (libbd_kvproj.so):

* float32 / float64 -> the exact SIMT kernel, bit-identical to the reference;
* float16 / bfloat16 -> the sm_100a tcgen05 kernel (FP32 accumulate, fused
  gather-add, one output rounding).

There is no CPU fallback: CPU tensors raise.  ``fused_kv_proj_host`` is the
synchronous host-buffer entry (numpy in, numpy out) that mirrors the reference's
numba call boundary exactly.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .decompose import Tag
from .errors import NativeLibraryError, PrecisionError, ShapeError


_DTYPES = {
    torch.float32: N.BD_F32,
    torch.float64: N.BD_F64,
    torch.float16: N.BD_F16,
    torch.bfloat16: N.BD_BF16,
}
_NP_DTYPES = {np.dtype(np.float32): N.BD_F32, np.dtype(np.float64): N.BD_F64,
              np.dtype(np.float16): N.BD_F16}
_MODES = {"auto": N.BD_MODE_AUTO, "exact": N.BD_MODE_EXACT, "tc": N.BD_MODE_TC}


def tag_offsets(d: int, d_h: int, tag: Tag) -> tuple[int, int]:
    """(mul_base, rep_base) for a tag (ref: attention.py:289-292)."""
    if tag is Tag.FIRST:
        return d_h, 0
    if tag is Tag.LAST:
        return 0, d - d_h
    raise ValueError(f"unknown tag {tag!r}")


def _rows_cols(t) -> tuple[int, int]:
    if t.dim() != 2:
        raise ShapeError(f"expected a 2-D tensor, got {t.dim()}-D")
    return int(t.shape[0]), int(t.shape[1])


def _check(x: torch.Tensor, c: torch.Tensor, d_h: int, n_heads: int) -> None:
    # Same order as the reference (attention.py:283-288).
    if x.dtype != c.dtype:
        raise PrecisionError("x and c must share precision")
    _, xcols = _rows_cols(x)
    crows, ccols = _rows_cols(c)
    if crows != xcols - d_h:
        raise ShapeError(f"c has {crows} rows, expected d - d_h = {xcols - d_h}")
    if ccols != n_heads * d_h:
        raise ShapeError(f"c has {ccols} cols, expected n_heads * d_h = {n_heads * d_h}")
    if x.dtype not in _DTYPES:
        raise PrecisionError(f"unsupported dtype {x.dtype}; expected float32/64, float16, bfloat16")
    if not (x.is_cuda and c.is_cuda):
        raise NativeLibraryError(
            "fused_kv_proj needs CUDA tensors (no CPU fallback); "
            "use fused_kv_proj_host for host buffers")
    if x.device != c.device:
        raise ValueError(f"x on {x.device} but c on {c.device}")


def _rowmajor(t: torch.Tensor) -> torch.Tensor:
    return t if (t.stride(1) == 1 and t.stride(0) >= t.shape[1]) else t.contiguous()


_LAYOUTS = {"token": N.BD_OUT_TOKEN_MAJOR, "head": N.BD_OUT_HEAD_MAJOR}


def _out_tensor(x, d_h, n_heads, layout, out=None):
    """Allocate or validate the output: token-major (L, n d_h) like the reference, or
    head-major (n, L, d_h) — per-head contiguous, what attention and a flat head
    all-gather consume."""
    L = int(x.shape[0])
    if layout not in _LAYOUTS:
        raise ValueError(f"unknown out_layout {layout!r}")
    shape = (L, n_heads * d_h) if layout == "token" else (n_heads, L, d_h)
    if out is None:
        return torch.empty(shape, dtype=x.dtype, device=x.device)
    ok = tuple(out.shape) == shape and out.dtype == x.dtype and out.stride(-1) == 1
    if layout == "head":
        ok = ok and out.stride(0) == L * out.stride(1)
    if not ok:
        raise ShapeError(f"out must be a {layout}-major {shape} tensor of x's dtype")
    return out


def _problem(x, c, out, d_h, n_heads, tag) -> N.KvProblem:
    L, d = int(x.shape[0]), int(x.shape[1])
    mul_base, rep_base = tag_offsets(d, d_h, tag)
    ldo = out.stride(0) if out.dim() == 2 else out.stride(1)
    return N.KvProblem(x.data_ptr(), c.data_ptr(), out.data_ptr(), x.stride(0), c.stride(0),
                       ldo, L, d, d_h, n_heads, mul_base, rep_base)


_raw_stream_fn = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _on_device(dev: torch.device, fn, *args):
    """Call a C-ABI entry point with the device's current stream appended, making the
    device current only when it is not already (the context manager costs microseconds
    per call on an eager serving path)."""
    cur = torch.cuda.current_device()
    idx = cur if dev.index is None else dev.index
    if idx == cur:
        stream = (_raw_stream_fn(idx) if _raw_stream_fn is not None
                  else torch.cuda.current_stream(idx).cuda_stream)
        return fn(*args, stream)
    with torch.cuda.device(idx):
        return fn(*args, torch.cuda.current_stream(idx).cuda_stream)


def _finish(flag: torch.Tensor | None) -> None:
    if flag is not None and int(flag.item()) != 0:
        raise ValueError("operation produced non-finite values")


def fused_kv_proj(x: torch.Tensor, c: torch.Tensor, d_h: int, n_heads: int,
                  tag: Tag = Tag.FIRST, *, out: torch.Tensor | None = None,
                  check_finite: bool = True, mode: str = "auto",
                  out_layout: str = "token") -> torch.Tensor:
    """Merged key/value projection in one pass over the output.

    Equivalent to tiling one d_h-wide slice of x n_heads times and adding the
    product of the complementary slice with c (FIRST repeats the leading slice,
    LAST the trailing one), without materialising the repeat or the slice.
    Enqueued on the current CUDA stream; ``check_finite`` synchronises once to
    read the kernel's non-finite flag (pass False on latency-critical paths).
    """
    _check(x, c, d_h, n_heads)
    x = _rowmajor(x)
    c = _rowmajor(c)
    out = _out_tensor(x, d_h, n_heads, out_layout, out)
    flag = torch.zeros(1, dtype=torch.int32, device=x.device) if check_finite else None
    prob = _problem(x, c, out, d_h, n_heads, tag)
    st = _on_device(x.device, N.load().bd_kv_proj_grouped_ex, ctypes.byref(prob), 1,
                    _DTYPES[x.dtype], _MODES[mode], _LAYOUTS[out_layout],
                    flag.data_ptr() if flag is not None else None)
    N.check(st, "bd_kv_proj")
    _finish(flag)
    return out


def fused_kv_proj_grouped(x: torch.Tensor,
                          specs: Sequence[tuple[torch.Tensor, int, int, Tag]],
                          *, outs: Sequence[torch.Tensor] | None = None,
                          check_finite: bool = True, mode: str = "auto",
                          flag: torch.Tensor | None = None,
                          out_layout: str = "token") -> list[torch.Tensor]:
    """Several projections of the same x in ONE kernel launch.

    ``specs`` is a list of (c, d_h, n_heads, tag) — e.g. K' and V' of
    ``bda_forward`` (ref attention.py:305-306), whose tags may differ.

    Like the reference (tensor.py:112-113) a non-finite result raises ``ValueError``
    by default, which costs one synchronisation to read the kernel's flag.  Pass
    ``check_finite=False`` for the unchecked fast path (no sync: CUDA-graph capturable),
    or a device int32 ``flag`` the kernel ORs into, to check later yourself.
    """
    if not 1 <= len(specs) <= N.BD_MAX_GROUP:
        raise ValueError(f"between 1 and {N.BD_MAX_GROUP} projections per launch")
    x = _rowmajor(x)
    probs = (N.KvProblem * len(specs))()
    results = []
    for i, (c, d_h, n_heads, tag) in enumerate(specs):
        _check(x, c, d_h, n_heads)
        c = _rowmajor(c)
        o = _out_tensor(x, d_h, n_heads, out_layout, outs[i] if outs is not None else None)
        probs[i] = _problem(x, c, o, d_h, n_heads, tag)
        results.append(o)
    own_flag = flag is None and check_finite
    if own_flag:
        flag = torch.zeros(1, dtype=torch.int32, device=x.device)
    st = _on_device(x.device, N.load().bd_kv_proj_grouped_ex, probs, len(specs),
                    _DTYPES[x.dtype], _MODES[mode], _LAYOUTS[out_layout],
                    flag.data_ptr() if flag is not None else None)
    N.check(st, "bd_kv_proj_grouped")
    if own_flag:
        _finish(flag)
    return results


def fold_rmsnorm(c: torch.Tensor, gamma: torch.Tensor, d_h: int,
                 tag: Tag) -> tuple[torch.Tensor, torch.Tensor]:
    """Offline fold of an RMSNorm weight into a BD coefficient matrix.

    For x_n = RMSNorm(x) * gamma the projection's multiplied term is
    x_n[:, mul] @ c = r * x[:, mul] @ (diag(gamma[mul]) c): returns (c_g, rep_gamma) with
    c_g = diag(gamma[mul_base : mul_base + K]) c (rounded once to c's dtype) and
    rep_gamma = gamma[rep_base : rep_base + d_h] in float32, the arguments of
    ``fused_rmsnorm_kv_proj_grouped``.
    """
    K = int(c.shape[0])
    d = K + d_h
    if gamma.dim() != 1 or int(gamma.shape[0]) != d:
        raise ShapeError(f"gamma must have d = {d} entries")
    mul_base, rep_base = tag_offsets(d, d_h, tag)
    g = gamma.to(device=c.device, dtype=torch.float64)
    c_g = (g[mul_base:mul_base + K, None] * c.to(torch.float64)).to(c.dtype).contiguous()
    return c_g, g[rep_base:rep_base + d_h].to(torch.float32).contiguous()


def fused_rmsnorm_kv_proj_grouped(x: torch.Tensor,
                                  specs: Sequence[tuple[torch.Tensor, torch.Tensor, int, int, Tag]],
                                  eps: float, *, outs: Sequence[torch.Tensor] | None = None,
                                  check_finite: bool = True, mode: str = "auto",
                                  out_layout: str = "token") -> list[torch.Tensor]:
    """K'/V' of the RMS-normalised latent in ONE launch, the norm fused (one read of x).

    ``x`` is the raw latent (e.g. DeepSeek-V2's compressed kv before kv_a_layernorm);
    ``specs`` are (c_g, rep_gamma, d_h, n_heads, tag) with (c_g, rep_gamma) from
    ``fold_rmsnorm``.  Equals ``fused_kv_proj_grouped(rms_norm(x) * gamma, ...)`` up to
    rounding (the normalised x is never rounded to 16 bit).  ``check_finite`` as in
    ``fused_kv_proj_grouped``.
    """
    if not 1 <= len(specs) <= N.BD_MAX_GROUP:
        raise ValueError(f"between 1 and {N.BD_MAX_GROUP} projections per launch")
    x = _rowmajor(x)
    probs = (N.KvProblem * len(specs))()
    gam = (ctypes.c_void_p * len(specs))()
    results = []
    for i, (c, rg, d_h, n_heads, tag) in enumerate(specs):
        _check(x, c, d_h, n_heads)
        if rg.dtype != torch.float32 or rg.numel() != d_h or not rg.is_contiguous() or \
                rg.device != x.device:
            raise ShapeError(f"rep_gamma must be a contiguous float32 ({d_h},) tensor on x's device")
        c = _rowmajor(c)
        o = _out_tensor(x, d_h, n_heads, out_layout, outs[i] if outs is not None else None)
        probs[i] = _problem(x, c, o, d_h, n_heads, tag)
        gam[i] = rg.data_ptr()
        results.append(o)
    flag = torch.zeros(1, dtype=torch.int32, device=x.device) if check_finite else None
    st = _on_device(x.device, N.load().bd_kv_proj_grouped_rmsnorm, probs, len(specs),
                    _DTYPES[x.dtype], _MODES[mode], _LAYOUTS[out_layout], gam, float(eps),
                    flag.data_ptr() if flag is not None else None)
    N.check(st, "bd_kv_proj_grouped_rmsnorm")
    _finish(flag)
    return results


class _HostPipeline:
    """Per-device streams, events and staging buffers of the chunked host path."""

    def __init__(self, dev):
        self.h2d = torch.cuda.Stream(dev)
        self.comp = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.bufs: dict = {}

    def host_flag(self):
        f = self.bufs.get("flag_host")
        if f is None:
            f = self.bufs["flag_host"] = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        return f

    def buf(self, tag, shape, dtype, dev):
        key = (tag, tuple(shape), dtype)
        b = self.bufs.get(key)
        if b is None:
            b = self.bufs[key] = torch.empty(shape, dtype=dtype, device=dev)
        return b


_pipes: dict = {}


def fused_kv_proj_grouped_host(x_host: torch.Tensor,
                               specs: Sequence[tuple[torch.Tensor, int, int, Tag]],
                               *, outs: Sequence[torch.Tensor] | None = None,
                               mode: str = "auto", chunks: int = 4) -> list[torch.Tensor]:
    """Grouped projection of a HOST activation tensor against device-resident C's.

    The end-to-end path of a caller whose activations live on the host: copies x in,
    runs the grouped kernel, copies every projection out (into ``outs``, pinned host
    tensors, or new pinned ones) and returns once they are ready.  The tokens are split
    into ``chunks`` row blocks pipelined over three streams — H2D of block i+1, the
    kernel on block i and D2H of block i-1 overlap — so the step costs about the
    PCIe transfer of its outputs (the kernel itself is ~1/40 of that at cfg2).
    """
    if x_host.is_cuda:
        raise ValueError("x_host must be a host tensor; use fused_kv_proj_grouped")
    dev = specs[0][0].device
    pipe = _pipes.get(dev)
    if pipe is None:
        pipe = _pipes[dev] = _HostPipeline(dev)
    L = int(x_host.shape[0])
    xd = pipe.buf("x", x_host.shape, x_host.dtype, dev)
    dev_outs = [pipe.buf(("o", i), (L, n * d_h), x_host.dtype, dev)
                for i, (_, d_h, n, _) in enumerate(specs)]
    if outs is None:
        outs = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in dev_outs]
    caller = torch.cuda.current_stream(dev)
    # one non-finite flag for every chunk, read once after the last copy-out (the
    # reference raises on a non-finite result, tensor.py:112-113)
    flag = pipe.buf("flag", (1,), torch.int32, dev)
    pipe.h2d.wait_stream(caller)
    with torch.cuda.stream(pipe.h2d):
        flag.zero_()  # device buffers are free once the caller's work is
    done = None
    for r0, r1 in _chunk_bounds(L, chunks):
        with torch.cuda.stream(pipe.h2d):
            xd[r0:r1].copy_(x_host[r0:r1], non_blocking=True)
        pipe.comp.wait_stream(pipe.h2d)
        with torch.cuda.stream(pipe.comp):
            fused_kv_proj_grouped(xd[r0:r1], specs, outs=[o[r0:r1] for o in dev_outs], mode=mode,
                                  flag=flag)
        pipe.d2h.wait_stream(pipe.comp)
        with torch.cuda.stream(pipe.d2h):
            for o, r in zip(outs, dev_outs):
                o[r0:r1].copy_(r[r0:r1], non_blocking=True)
    # the flag rides the copy-out stream into pinned memory: no extra synchronising read
    flag_host = pipe.host_flag()
    with torch.cuda.stream(pipe.d2h):
        flag_host.copy_(flag, non_blocking=True)
        done = torch.cuda.Event()
        done.record(pipe.d2h)
    done.synchronize()
    caller.wait_stream(pipe.d2h)
    if int(flag_host[0]) != 0:
        raise ValueError("operation produced non-finite values")
    return list(outs)


def _chunk_bounds(L: int, chunks: int) -> list[tuple[int, int]]:
    """Row blocks of the host pipeline: ``chunks`` equal blocks of whole 256-row tiles.
    (A short first block, to start the first copy-out earlier, measured slower at cfg2:
    1.39 vs 1.35 ms per step, tools/e2e_ab.py.)"""
    if L <= 0:
        return []
    step = max(1, -(-L // max(1, chunks)))
    step = -(-step // 256) * 256  # whole 256-row CTA-pair tiles per block
    return [(r0, min(L, r0 + step)) for r0 in range(0, L, step)]


def fused_kv_proj_host(x: np.ndarray, c: np.ndarray, d_h: int, n_heads: int,
                       tag: Tag = Tag.FIRST, *, mode: str = "auto") -> np.ndarray:
    """Synchronous host-buffer projection through ``bd_kv_proj_host``.

    Takes and returns C-contiguous numpy arrays (float32/float64/float16), exactly
    the boundary of the reference's numba kernel call (attention.py:293-295):
    copies in, runs on the GPU, copies out.
    """
    if x.dtype != c.dtype:
        raise PrecisionError("x and c must share precision")
    if x.ndim != 2 or c.ndim != 2:
        raise ShapeError("expected 2-D arrays")
    if c.shape[0] != x.shape[1] - d_h:
        raise ShapeError(f"c has {c.shape[0]} rows, expected d - d_h = {x.shape[1] - d_h}")
    if c.shape[1] != n_heads * d_h:
        raise ShapeError(f"c has {c.shape[1]} cols, expected n_heads * d_h = {n_heads * d_h}")
    if x.dtype not in _NP_DTYPES:
        raise PrecisionError(f"unsupported dtype {x.dtype}")
    x = np.ascontiguousarray(x)
    c = np.ascontiguousarray(c)
    L, d = x.shape
    mul_base, rep_base = tag_offsets(d, d_h, tag)
    out = np.empty((L, n_heads * d_h), dtype=x.dtype)
    bad = ctypes.c_int(0)
    st = N.load().bd_kv_proj_host(x.ctypes.data, c.ctypes.data, out.ctypes.data, L, d, d_h,
                                  n_heads, mul_base, rep_base, _NP_DTYPES[x.dtype], _MODES[mode],
                                  ctypes.byref(bad))
    N.check(st, "bd_kv_proj_host")
    if bad.value:
        raise ValueError("operation produced non-finite values")
    return out


def kv_flops(L: int, d: int, d_h: int, n_heads: int) -> int:
    """Multiply-FLOPs of one BD projection: 2 L (d - d_h) N (ref bench.py:158 ratio)."""
    return 2 * L * (d - d_h) * n_heads * d_h


def flop_ratio(d: int, d_h: int) -> float:
    """Dense / BD FLOP ratio d / (d - d_h) (ref: bench.py:266)."""
    return d / (d - d_h)
