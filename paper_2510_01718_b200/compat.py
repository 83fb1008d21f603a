"""Drop-in replacement of the reference's native entry point.

``_fused_kernel(x, c, d_h, n_heads, mul_base, rep_base, out)`` has the numba kernel's
exact signature and contract (ref: pkg/src/bdattn/attention.py:249-270, called at
:294): C-contiguous float32/float64 (or float16) host arrays, ``out`` overwritten in
place.  It routes through the synchronous C-ABI entry ``bd_kv_proj_host`` — copy in,
run the GPU kernel (the exact kernel for float32/float64, bit-identical to numba's
output), copy out.  ``install(bdattn.attention)`` rebinds the reference module's
symbol so ``fused_kv_proj``, ``bda_forward`` and the reference's own tests run on the
B200 unchanged.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N

_DT = {np.dtype(np.float32): N.BD_F32, np.dtype(np.float64): N.BD_F64,
       np.dtype(np.float16): N.BD_F16}


def _fused_kernel(x, c, d_h, n_heads, mul_base, rep_base, out) -> None:
    x = np.ascontiguousarray(x)
    c = np.ascontiguousarray(c)
    if x.dtype not in _DT or c.dtype != x.dtype or out.dtype != x.dtype:
        raise ValueError(f"unsupported dtypes {x.dtype}/{c.dtype}/{out.dtype}")
    if not out.flags.c_contiguous or out.shape != (x.shape[0], n_heads * d_h):
        raise ValueError("out must be a C-contiguous (L, n_heads * d_h) array")
    bad = ctypes.c_int(0)
    st = N.load().bd_kv_proj_host(x.ctypes.data, c.ctypes.data, out.ctypes.data, x.shape[0],
                                  x.shape[1], int(d_h), int(n_heads), int(mul_base),
                                  int(rep_base), _DT[x.dtype], N.BD_MODE_AUTO, ctypes.byref(bad))
    N.check(st, "bd_kv_proj_host")


def install(attention_module) -> None:
    """Rebind ``attention_module._fused_kernel`` (e.g. ``bdattn.attention``)."""
    attention_module._fused_kernel = _fused_kernel
