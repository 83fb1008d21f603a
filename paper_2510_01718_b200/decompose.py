"""Offline basis decomposition (BD) — the preparation side of the hot path.

A rank-r matrix is stored as r of its own contiguous rows (or columns) plus the
coefficients that rebuild the others.  The first-r and last-r candidates are both
formed; the smaller Frobenius reconstruction residual wins, ties to FIRST
(ref: pkg/src/bdattn/decompose.py:1-8, 117-171).

This stays on the CPU in NumPy/SciPy, as the north star asks ("the offline BD
preparation ... stay in Python"), and it deliberately issues the SAME sequence of
floating-point operations as the reference so the selected basis S (the tag) is
bit-identical to the reference's, not merely close:

* the per-head weight products use ``ordered_matmul``: one accumulator per element,
  k ascending, one rounded multiply and one rounded add per step, starting from +0
  (the reference's numba ``_matmul_kernel`` contract, ref tensor.py:189-213);
* coefficients come from ``numpy.linalg.qr`` + ``scipy.linalg.solve_triangular`` on
  contiguous copies, with the min-norm ``lstsq`` route when the triangular factor's
  diagonal ratio is below 1e-10 (ref tensor.py:325-374);
* residuals use BLAS products pinned to one thread (ref tensor.py:35, 216-226) and a
  64-bit dot product of the flattened error (ref tensor.py:306-309).

Nothing here runs on the inference path; the GPU projection consumes the merged
coefficients (see attention.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import NamedTuple

import numpy as np

# ref: tensor.py:44
RANK_DEFICIENCY_TOL = 1e-10


class Axis(Enum):
    """Whether the basis is a set of rows or of columns (ref decompose.py:20-24)."""

    ROW = "row"
    COLUMN = "column"


class Tag(Enum):
    """Which contiguous block serves as the basis (ref decompose.py:27-31)."""

    FIRST = "first"
    LAST = "last"


class Side(Enum):
    """Side of the basis the unknown coefficients sit on (ref tensor.py:312-316)."""

    SOLVE_LEFT = "left"    # C @ basis ~= targets
    SOLVE_RIGHT = "right"  # basis @ C ~= targets


class LstsqResult(NamedTuple):
    coeff: np.ndarray
    rank_deficient: bool
    diag_ratio: float


def _blas_one_thread():
    """Context pinning BLAS to one thread, as the reference does at import
    (tensor.py:35) — BLAS results can depend on the thread split."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1, user_api="blas")
    except Exception:  # pragma: no cover - threadpoolctl is in the image
        import contextlib
        return contextlib.nullcontext()


def _c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a)


def ordered_matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """a @ b with the reference's per-element rounding sequence.

    out[i, j] = fl(... fl(fl(0 + fl(a[i,0] b[0,j])) + fl(a[i,1] b[1,j])) ...): k ascending,
    separate rounded multiply and add (NumPy never contracts to FMA).  Bit-identical to
    ``bdattn.matmul`` (ref tensor.py:189-213); vectorised over (i, j), sequential in k.
    """
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        from .errors import ShapeError
        raise ShapeError(f"matmul: inner dims differ ({a.shape} vs {b.shape})")
    if a.dtype != b.dtype:
        from .errors import PrecisionError
        raise PrecisionError("matmul operands must share precision")
    out = np.zeros((a.shape[0], b.shape[1]), dtype=a.dtype)
    for k in range(a.shape[1]):
        out += a[:, k:k + 1] * b[k:k + 1, :]
    return out


def blas_matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Platform-BLAS product for tolerance-bound steps (ref tensor.py:216-226)."""
    with _blas_one_thread():
        return _c(a) @ _c(b)


def frobenius_norm(a: np.ndarray) -> float:
    """sqrt of the sum of squares accumulated in 64-bit (ref tensor.py:306-309)."""
    flat = _c(a).ravel().astype(np.float64, copy=False)
    with _blas_one_thread():
        return float(math.sqrt(np.dot(flat, flat)))


def lstsq(basis: np.ndarray, targets: np.ndarray, side: Side) -> LstsqResult:
    """Least-squares coefficients against a basis via QR (ref tensor.py:325-374)."""
    from scipy.linalg import solve_triangular

    from .errors import PrecisionError, ShapeError

    if basis.dtype != targets.dtype:
        raise PrecisionError("lstsq operands must share precision")
    if side is Side.SOLVE_LEFT:
        if basis.shape[1] != targets.shape[1]:
            raise ShapeError(f"lstsq left: basis has {basis.shape[1]} cols, "
                             f"targets {targets.shape[1]}")
        if basis.shape[1] < basis.shape[0]:
            raise ShapeError(f"lstsq left: underdetermined basis {basis.shape}")
        system, rhs = _c(basis.T), _c(targets.T)
    else:
        if basis.shape[0] != targets.shape[0]:
            raise ShapeError(f"lstsq right: basis has {basis.shape[0]} rows, "
                             f"targets {targets.shape[0]}")
        if basis.shape[0] < basis.shape[1]:
            raise ShapeError(f"lstsq right: underdetermined basis {basis.shape}")
        system, rhs = basis, targets
    with _blas_one_thread():
        q, r = np.linalg.qr(system, mode="reduced")
        diag = np.abs(np.diagonal(r))
        largest = float(diag.max())
        ratio = float(diag.min() / largest) if largest > 0.0 else 0.0
        deficient = ratio < RANK_DEFICIENCY_TOL
        if deficient:
            sol = np.linalg.lstsq(system, rhs, rcond=None)[0]
        else:
            sol = solve_triangular(r, q.T @ rhs, lower=False)
    if side is Side.SOLVE_LEFT:
        sol = _c(sol.T)
    return LstsqResult(np.ascontiguousarray(sol, dtype=basis.dtype), deficient, ratio)


@dataclass(frozen=True)
class BDFactors:
    """One BD candidate (ref decompose.py:34-71).

    ROW: ``basis`` r x n, ``coeff`` (m-r) x r, non-basis rows = coeff @ basis.
    COLUMN: ``basis`` m x r, ``coeff`` r x (n-r), non-basis cols = basis @ coeff.
    """

    axis: Axis
    tag: Tag
    basis: np.ndarray
    coeff: np.ndarray
    orig_rows: int
    orig_cols: int
    rank: int
    residual: float
    rank_deficient: bool

    def __post_init__(self):
        m, n, r = self.orig_rows, self.orig_cols, self.rank
        _check_rank(m, n, r, self.axis)
        if self.axis is Axis.ROW:
            eb, ec = (r, n), (m - r, r)
        else:
            eb, ec = (m, r), (r, n - r)
        if tuple(self.basis.shape) != eb:
            raise ValueError(f"basis shape {tuple(self.basis.shape)}, expected {eb}")
        if tuple(self.coeff.shape) != ec:
            raise ValueError(f"coeff shape {tuple(self.coeff.shape)}, expected {ec}")
        if self.residual < 0.0:
            raise ValueError("residual must be non-negative")

    @property
    def param_count(self) -> int:
        """Stored elements r (m + n - r)."""
        return int(self.basis.size + self.coeff.size)


@dataclass(frozen=True)
class CostReport:
    full_params: int
    lowrank_params: int
    bd_params: int
    lowrank_recon_flops: int
    bd_recon_flops: int


def cost_report(m: int, n: int, rank: int) -> CostReport:
    """Closed-form storage / rebuild-FLOP counts (ref decompose.py:84-102)."""
    if not 1 <= rank < min(m, n):
        raise ValueError(
            f"rank must satisfy 1 <= rank < min(m, n); got rank={rank} for {m}x{n}")
    r = rank
    return CostReport(full_params=m * n, lowrank_params=r * (m + n), bd_params=r * (m + n - r),
                      lowrank_recon_flops=2 * r * m * n, bd_recon_flops=2 * r * (m - r) * n)


def _check_rank(m: int, n: int, rank: int, axis: Axis) -> None:
    ok = (1 <= rank < m and rank <= n) if axis is Axis.ROW else (1 <= rank < n and rank <= m)
    if not ok:
        raise ValueError(f"rank {rank} out of range for a {m}x{n} {axis.value} decomposition")


def _rebuild(axis: Axis, tag: Tag, basis: np.ndarray, coeff: np.ndarray) -> np.ndarray:
    if axis is Axis.ROW:
        rebuilt = blas_matmul(coeff, basis)
        parts = [basis, rebuilt] if tag is Tag.FIRST else [rebuilt, basis]
        return np.concatenate(parts, axis=0)
    rebuilt = blas_matmul(basis, coeff)
    parts = [basis, rebuilt] if tag is Tag.FIRST else [rebuilt, basis]
    return np.concatenate(parts, axis=1)


def _candidate(w: np.ndarray, rank: int, axis: Axis, tag: Tag) -> BDFactors:
    """ref decompose.py:127-152."""
    m, n = w.shape
    if axis is Axis.ROW:
        if tag is Tag.FIRST:
            basis, rest = _c(w[:rank]), _c(w[rank:])
        else:
            basis, rest = _c(w[m - rank:]), _c(w[:m - rank])
        coeff, deficient, _ = lstsq(basis, rest, Side.SOLVE_LEFT)
    else:
        if tag is Tag.FIRST:
            basis, rest = _c(w[:, :rank]), _c(w[:, rank:])
        else:
            basis, rest = _c(w[:, n - rank:]), _c(w[:, :n - rank])
        coeff, deficient, _ = lstsq(basis, rest, Side.SOLVE_RIGHT)
    residual = frobenius_norm(w - _rebuild(axis, tag, basis, coeff))
    return BDFactors(axis=axis, tag=tag, basis=basis, coeff=coeff, orig_rows=m, orig_cols=n,
                     rank=rank, residual=residual, rank_deficient=bool(deficient))


def bd_decompose_both(w: np.ndarray, rank: int, axis: Axis) -> tuple[BDFactors, BDFactors]:
    """(FIRST, LAST) candidates with their residuals (ref decompose.py:155-160)."""
    w = _c(np.asarray(w))
    _check_rank(w.shape[0], w.shape[1], rank, axis)
    return _candidate(w, rank, axis, Tag.FIRST), _candidate(w, rank, axis, Tag.LAST)


def bd_decompose(w: np.ndarray, rank: int, axis: Axis) -> BDFactors:
    """Smaller-residual candidate, ties to FIRST (ref decompose.py:163-171)."""
    first, last = bd_decompose_both(w, rank, axis)
    return first if first.residual <= last.residual else last


def bd_reconstruct(f: BDFactors) -> np.ndarray:
    """Rebuild the original matrix from its factors (ref decompose.py:174-180)."""
    return _rebuild(f.axis, f.tag, f.basis, f.coeff)
