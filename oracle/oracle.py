"""Python face of the CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* ``fused_kv_proj_ref`` — the reference's fused K/V projection
  (ref: pkg/src/bdattn/attention.py:249-295) restated in C (oracle/bd_oracle.c),
  bit-identical to the reference for float32/float64 (pinned by tests/golden).
* ``matmul_ref`` — the reference's fixed-order matmul (ref: tensor.py:189-213).
* ``Rng`` / ``rand_gaussian`` / ``gen_random_mha`` — the reference's seeded input
  generators (ref: tensor.py:377-419, verify.py:83-99) restated on numpy's PCG64 +
  SeedSequence, so the same seed gives the same inputs here, on the GPU box and in
  the reference itself.
* ``max_relative_error`` — the reference's parity metric (ref: verify.py:74-80).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libbd_oracle.so"
_lib = None

# ref: tensor.py:186
ROW_BLOCK = 8


def build() -> Path:
    """Compile the C oracle (make in oracle/). Returns the .so path."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        build()
    lib = ctypes.CDLL(str(_LIB_PATH))
    i64 = ctypes.c_int64
    for name in ("bd_oracle_fused_f32", "bd_oracle_fused_f64"):
        fn = getattr(lib, name)
        fn.argtypes = [ctypes.c_void_p] * 3 + [i64] * 6 + [ctypes.c_int]
        fn.restype = None
    for name in ("bd_oracle_matmul_f32", "bd_oracle_matmul_f64"):
        fn = getattr(lib, name)
        fn.argtypes = [ctypes.c_void_p] * 3 + [i64] * 3 + [ctypes.c_int]
        fn.restype = None
    lib.bd_oracle_max_threads.restype = ctypes.c_int
    _lib = lib
    return lib


def max_threads() -> int:
    return int(_load().bd_oracle_max_threads())


def tag_offsets(d: int, d_h: int, tag: str) -> tuple[int, int]:
    """(mul_base, rep_base) for a tag, ref: attention.py:289-292."""
    if tag == "first":
        return d_h, 0
    if tag == "last":
        return 0, d - d_h
    raise ValueError(f"unknown tag {tag!r}")


def fused_kv_proj_ref(x: np.ndarray, c: np.ndarray, d_h: int, n_heads: int, tag: str = "first",
                      threads: int = 1, out: np.ndarray | None = None) -> np.ndarray:
    """Reference fused projection on float32/float64 host arrays (exact sequence)."""
    if x.dtype != c.dtype or x.dtype not in (np.float32, np.float64):
        raise ValueError("x and c must share dtype float32 or float64")
    x = np.ascontiguousarray(x)
    c = np.ascontiguousarray(c)
    L, d = x.shape
    if c.shape != (d - d_h, n_heads * d_h):
        raise ValueError(f"c has shape {c.shape}, expected {(d - d_h, n_heads * d_h)}")
    mul_base, rep_base = tag_offsets(d, d_h, tag)
    if out is None:
        out = np.empty((L, n_heads * d_h), dtype=x.dtype)
    fn = _load().bd_oracle_fused_f32 if x.dtype == np.float32 else _load().bd_oracle_fused_f64
    fn(x.ctypes.data, c.ctypes.data, out.ctypes.data, L, d, d_h, n_heads, mul_base, rep_base,
       int(threads))
    return out


def matmul_ref(a: np.ndarray, b: np.ndarray, threads: int = 1) -> np.ndarray:
    """Reference fixed-order matmul (k ascending, one rounding per step)."""
    if a.dtype != b.dtype or a.dtype not in (np.float32, np.float64):
        raise ValueError("a and b must share dtype float32 or float64")
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    m, kk = a.shape
    if b.shape[0] != kk:
        raise ValueError("inner dims differ")
    out = np.empty((m, b.shape[1]), dtype=a.dtype)
    fn = _load().bd_oracle_matmul_f32 if a.dtype == np.float32 else _load().bd_oracle_matmul_f64
    fn(a.ctypes.data, b.ctypes.data, out.ctypes.data, m, kk, b.shape[1], int(threads))
    return out


def fused_unfused_naive(x: np.ndarray, c: np.ndarray, d_h: int, n_heads: int,
                        tag: str = "first") -> np.ndarray:
    """Pure-Python restatement of the reference's *unfused* composition
    ``add(repeat_cols(slice), matmul(slice, c))`` (ref test_attention.py:197-203),
    element by element with the scalar rounding sequence.  Small shapes only."""
    L, d = x.shape
    mul_base, rep_base = tag_offsets(d, d_h, tag)
    kk = d - d_h
    t = x.dtype.type
    out = np.zeros((L, n_heads * d_h), dtype=x.dtype)
    for i in range(L):
        for j in range(n_heads * d_h):
            acc = t(0.0)
            for k in range(kk):
                acc = t(acc + t(x[i, mul_base + k] * c[k, j]))
            out[i, j] = t(acc + x[i, rep_base + j % d_h])
    return out


def fused_ref_f64(x, c, d_h: int, n_heads: int, tag: str = "first", threads: int = 1) -> np.ndarray:
    """FP64 oracle on (already rounded) 16-bit inputs: the values are exactly
    representable in float64, so this is the reference computed at P64 on the same
    inputs the tensor-core kernel sees."""
    return fused_kv_proj_ref(np.asarray(x, dtype=np.float64), np.asarray(c, dtype=np.float64),
                             d_h, n_heads, tag, threads)


# ----------------------------------------------------------------------------- inputs
class Rng:
    """Restates bdattn.Rng (ref: tensor.py:377-405): PCG64 keyed by
    SeedSequence(seed, spawn_key); derive(i) appends i to the spawn key."""

    def __init__(self, seed: int, _spawn_key: tuple[int, ...] = ()):
        self.seed = int(seed)
        self.spawn_key = tuple(int(k) for k in _spawn_key)
        ss = np.random.SeedSequence(self.seed, spawn_key=self.spawn_key)
        self._gen = np.random.Generator(np.random.PCG64(ss))

    def derive(self, index: int) -> "Rng":
        return Rng(self.seed, self.spawn_key + (int(index),))

    def standard_normal(self, rows: int, cols: int) -> np.ndarray:
        return self._gen.standard_normal((rows, cols))


def rand_gaussian(rng: Rng, rows: int, cols: int, dtype=np.float64) -> np.ndarray:
    """ref: tensor.py:408-419 — drawn in float64, then rounded."""
    return np.ascontiguousarray(rng.standard_normal(rows, cols).astype(dtype, copy=False))


def scale(a: np.ndarray, factor: float) -> np.ndarray:
    """ref: tensor.py:292-295 — factor rounded to the operand precision first."""
    return a * a.dtype.type(factor)


def gen_random_mha(rng: Rng, d: int, d_h: int, n_heads: int, dtype=np.float64) -> dict:
    """ref: verify.py:83-99 — Gaussian weights at scale 1/sqrt(d)."""
    s = 1.0 / math.sqrt(d)
    width = n_heads * d_h
    return {
        "d": d, "n_heads": n_heads, "d_h": d_h,
        "w_q": scale(rand_gaussian(rng, d, width, dtype), s),
        "w_k": scale(rand_gaussian(rng, d, width, dtype), s),
        "w_v": scale(rand_gaussian(rng, d, width, dtype), s),
        "w_o": scale(rand_gaussian(rng, width, d, dtype), s),
    }


def max_relative_error(result, reference) -> float:
    """ref: verify.py:74-80."""
    r = np.asarray(result, dtype=np.float64)
    ref = np.asarray(reference, dtype=np.float64)
    diff = np.abs(r - ref)
    denom = float(np.abs(ref).max()) if ref.size else 0.0
    if denom == 0.0:
        return float(diff.max()) if diff.size else 0.0
    return float(diff.max()) / denom


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
