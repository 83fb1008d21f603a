"""BD replacement of a low-rank linear layer (ref: pkg/src/bdattn/linear.py).

    W = U V^T (d_in x d_out, rank r)  --column BD-->  B = W[:, S] (d_in x r), C (r x (d_out-r))
    forward:  h = x B;   y = [h, h C]  (tag FIRST)   or   [h C, h]  (tag LAST)

The forward is ONE C-ABI call (``bd_linear_forward``) that issues two GEMMs on the
current stream: the first writes h straight into its final columns of y, the second
reads it back from there as its A operand and writes h C beside it — the reference's
``concat_cols`` (linear.py:107-108) costs nothing.  float32/float64 use the exact
kernel without the repeated-slice add, i.e. the reference's fixed-order matmul, so the
result is bit-identical to ``bdattn.bd_linear_forward``; float16/bfloat16 use the
tcgen05 tensor-core kernel.  Prep (``bd_linear_from_lowrank``) is offline NumPy.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .decompose import Axis, BDFactors, Tag, bd_decompose, ordered_matmul
from .errors import NativeLibraryError, PrecisionError, ShapeError
from .kv_proj import _DTYPES, _MODES, _on_device, _rowmajor


@dataclass(frozen=True)
class LowRankLayer:
    """Two-factor layer: u is d_in x r, v is d_out x r (ref linear.py:19-52)."""

    u: torch.Tensor
    v: torch.Tensor

    def __post_init__(self):
        if self.u.shape[1] != self.v.shape[1]:
            raise ShapeError(f"factor ranks differ: {self.u.shape[1]} vs {self.v.shape[1]}")
        if self.u.dtype != self.v.dtype:
            raise ShapeError("factors must share precision")
        if not self.u.shape[1] < min(self.u.shape[0], self.v.shape[0]):
            raise ValueError(f"rank {self.u.shape[1]} must be < min(d_in={self.u.shape[0]}, "
                             f"d_out={self.v.shape[0]})")

    @property
    def d_in(self) -> int:
        return int(self.u.shape[0])

    @property
    def d_out(self) -> int:
        return int(self.v.shape[0])

    @property
    def rank(self) -> int:
        return int(self.u.shape[1])

    @property
    def param_count(self) -> int:
        return self.rank * (self.d_in + self.d_out)


@dataclass(frozen=True)
class BDLinearLayer:
    """Column-axis BD factors of U V^T, plus the device copies the kernel reads
    (ref linear.py:55-88)."""

    factors: BDFactors
    basis: torch.Tensor   # d_in x r
    coeff: torch.Tensor   # r x (d_out - r)

    def __post_init__(self):
        if self.factors.axis is not Axis.COLUMN:
            raise ValueError("BDLinearLayer needs column-axis factors")

    @property
    def d_in(self) -> int:
        return self.factors.orig_rows

    @property
    def d_out(self) -> int:
        return self.factors.orig_cols

    @property
    def rank(self) -> int:
        return self.factors.rank

    @property
    def tag(self) -> Tag:
        return self.factors.tag

    @property
    def param_count(self) -> int:
        return self.factors.param_count

    def to(self, device=None, dtype=None) -> "BDLinearLayer":
        return BDLinearLayer(self.factors, self.basis.to(device=device, dtype=dtype),
                             self.coeff.to(device=device, dtype=dtype))


def lowrank_forward(x: torch.Tensor, layer: LowRankLayer) -> torch.Tensor:
    """(x U) V^T with cuBLAS — the baseline the BD layer replaces (ref linear.py:84-88)."""
    if x.shape[-1] != layer.d_in:
        raise ShapeError(f"input has {x.shape[-1]} cols, layer expects {layer.d_in}")
    return (x @ layer.u) @ layer.v.T


def bd_linear_from_lowrank(layer: LowRankLayer, *, prepare_in_p64: bool = False,
                           device=None, dtype: torch.dtype | None = None) -> BDLinearLayer:
    """Decompose U V^T column-wise at the layer's rank (ref linear.py:91-98).

    Like the reference the product is formed with the fixed-order matmul in the layer's
    precision; ``prepare_in_p64`` (or a 16-bit layer) runs it in float64 instead and
    rounds the factors (P32 prep costs 4e-3 max-rel at cfg4).
    """
    p32 = layer.u.dtype == torch.float32 and not prepare_in_p64
    work = np.float32 if p32 else np.float64
    u = np.ascontiguousarray(layer.u.detach().to("cpu", torch.float64).numpy().astype(work))
    vt = np.ascontiguousarray(layer.v.detach().to("cpu", torch.float64).numpy().astype(work).T)
    f = bd_decompose(ordered_matmul(u, vt), layer.rank, Axis.COLUMN)
    out_dtype = dtype or layer.u.dtype
    dev = device if device is not None else layer.u.device
    return BDLinearLayer(f, torch.from_numpy(f.basis).to(dev, out_dtype),
                         torch.from_numpy(f.coeff).to(dev, out_dtype))


def bd_linear_forward(x: torch.Tensor, layer: BDLinearLayer, *, out: torch.Tensor | None = None,
                      check_finite: bool = True, mode: str = "auto") -> torch.Tensor:
    """Two-step forward h = x B; y = [h, h C] / [h C, h] (ref linear.py:101-108).

    A non-finite result raises ``ValueError`` like the reference (tensor.py:112-113);
    ``check_finite=False`` skips the flag read (no synchronisation)."""
    if x.dim() != 2 or x.shape[1] != layer.d_in:
        raise ShapeError(f"input has {x.shape[-1]} cols, layer expects {layer.d_in}")
    if x.dtype != layer.basis.dtype or x.dtype != layer.coeff.dtype:
        raise PrecisionError("input and layer must share precision")
    if x.dtype not in _DTYPES:
        raise PrecisionError(f"unsupported dtype {x.dtype}")
    if not (x.is_cuda and layer.basis.is_cuda and layer.coeff.is_cuda):
        raise NativeLibraryError("bd_linear_forward needs CUDA tensors (no CPU fallback)")
    x = _rowmajor(x)
    basis, coeff = _rowmajor(layer.basis), _rowmajor(layer.coeff)
    L = int(x.shape[0])
    if out is None:
        out = torch.empty((L, layer.d_out), dtype=x.dtype, device=x.device)
    elif tuple(out.shape) != (L, layer.d_out) or out.dtype != x.dtype or out.stride(1) != 1:
        raise ShapeError("out must be a row-major (L, d_out) tensor of x's dtype")
    flag = torch.zeros(1, dtype=torch.int32, device=x.device) if check_finite else None
    tag = N.BD_TAG_FIRST if layer.tag is Tag.FIRST else N.BD_TAG_LAST
    st = _on_device(x.device, N.load().bd_linear_forward,
                    x.data_ptr(), x.stride(0), basis.data_ptr(), basis.stride(0),
                    coeff.data_ptr(), coeff.stride(0), out.data_ptr(), out.stride(0), L,
                    layer.d_in, layer.rank, layer.d_out, tag, _DTYPES[x.dtype], _MODES[mode],
                    flag.data_ptr() if flag is not None else None)
    N.check(st, "bd_linear_forward")
    if flag is not None and int(flag.item()) != 0:
        raise ValueError("operation produced non-finite values")
    return out


def matmul(a: torch.Tensor, b: torch.Tensor, *, mode: str = "auto") -> torch.Tensor:
    """a @ b through ``bd_matmul``: float32/float64 bit-identical to the reference's
    fixed-order matmul (ref tensor.py:189-213), 16-bit on tensor cores."""
    if a.dtype != b.dtype:
        raise PrecisionError("matmul operands must share precision")
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0]:
        raise ShapeError(f"matmul: inner dims differ ({tuple(a.shape)} vs {tuple(b.shape)})")
    if not (a.is_cuda and b.is_cuda):
        raise NativeLibraryError("matmul needs CUDA tensors (no CPU fallback)")
    a, b = _rowmajor(a), _rowmajor(b)
    out = torch.empty((a.shape[0], b.shape[1]), dtype=a.dtype, device=a.device)
    st = _on_device(a.device, N.load().bd_matmul, a.data_ptr(), a.stride(0), b.data_ptr(),
                    b.stride(0), out.data_ptr(), out.stride(0), a.shape[0], a.shape[1],
                    b.shape[1], _DTYPES[a.dtype], _MODES[mode], None)
    N.check(st, "bd_matmul")
    return out
