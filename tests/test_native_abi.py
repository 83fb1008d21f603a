"""The C-ABI library loads, exports every symbol include/*.h declares, and rejects
bad arguments before touching the GPU; the Python op keeps the reference's check
order and error types.  CPU only (no kernel is launched here)."""

import ctypes
import re

import numpy as np
import pytest
import torch

from conftest import ROOT
import paper_2510_01718_b200 as bd
from paper_2510_01718_b200 import _native as N
from paper_2510_01718_b200.build import build


@pytest.fixture(scope="module")
def lib():
    build()
    return N.load()


def declared_functions():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = h.read_text()
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(bd_\w+)\s*\(", text, re.M):
            names.add(m.group(1))
    return names


def test_every_declared_symbol_is_exported(lib):
    declared = declared_functions()
    assert declared == set(N.EXPORTED_SYMBOLS), declared
    for name in declared:
        assert hasattr(lib, name), name


def test_abi_version_and_empty_error(lib):
    assert lib.bd_abi_version() == N.ABI_VERSION
    assert isinstance(N.last_error(), str)


def call(lib, **kw):
    a = dict(x=1 << 20, ldx=16, c=1 << 21, ldc=16, out=1 << 22, ldo=16, L=4, d=16, d_h=8,
             n_heads=2, mul_base=8, rep_base=0, dtype=N.BD_F16, mode=N.BD_MODE_AUTO)
    a.update(kw)
    return lib.bd_kv_proj(a["x"], a["ldx"], a["c"], a["ldc"], a["out"], a["ldo"], a["L"], a["d"],
                          a["d_h"], a["n_heads"], a["mul_base"], a["rep_base"], a["dtype"],
                          a["mode"], None, None)


def test_abi_rejects_bad_arguments_without_launching(lib):
    before = lib.bd_launch_count()
    assert call(lib, x=None) == N.BD_ERR_ARG
    assert call(lib, d_h=16) == N.BD_ERR_SHAPE           # d_h >= d
    assert call(lib, L=0) == N.BD_ERR_SHAPE
    assert call(lib, ldc=8) == N.BD_ERR_SHAPE            # ldc < N
    assert call(lib, mul_base=9) == N.BD_ERR_SHAPE       # mul slice past d
    assert call(lib, dtype=7) == N.BD_ERR_DTYPE
    assert call(lib, dtype=N.BD_F32, mode=N.BD_MODE_TC) == N.BD_ERR_DTYPE
    assert call(lib, dtype=N.BD_F16, mode=N.BD_MODE_EXACT) == N.BD_ERR_DTYPE
    assert call(lib, mode=9) == N.BD_ERR_ARG
    assert call(lib, x=(1 << 20) + 2) == N.BD_ERR_ALIGN   # TMA needs 16-B alignment
    assert call(lib, ldx=20, d=16) == N.BD_ERR_ALIGN
    assert "multiples of 8" in N.last_error()
    assert lib.bd_launch_count() == before


def test_grouped_count_bounds(lib):
    probs = (N.KvProblem * 5)()
    assert lib.bd_kv_proj_grouped(probs, 0, N.BD_F16, 0, None, None) == N.BD_ERR_ARG
    assert lib.bd_kv_proj_grouped(probs, 5, N.BD_F16, 0, None, None) == N.BD_ERR_ARG


def test_status_maps_to_reference_exceptions(lib):
    with pytest.raises(bd.ShapeError):
        N.check(N.BD_ERR_SHAPE, "x")
    with pytest.raises(bd.PrecisionError):
        N.check(N.BD_ERR_DTYPE, "x")
    with pytest.raises(bd.NativeLibraryError):
        N.check(N.BD_ERR_CUDA, "x")
    assert issubclass(bd.ShapeError, ValueError) and issubclass(bd.PrecisionError, ValueError)


class TestOperatorValidation:
    """Mirrors ref test_attention.py:205-210 and the check order of attention.py:283-288."""

    def test_precision_checked_first(self):
        x = torch.zeros(2, 8, dtype=torch.float32)
        c = torch.zeros(5, 7, dtype=torch.float64)  # also wrong shape: precision wins
        with pytest.raises(bd.PrecisionError):
            bd.fused_kv_proj(x, c, d_h=2, n_heads=3)

    def test_shape_validation(self):
        x = torch.zeros(2, 8)
        with pytest.raises(bd.ShapeError):
            bd.fused_kv_proj(x, torch.zeros(5, 6), d_h=2, n_heads=3)
        with pytest.raises(bd.ShapeError):
            bd.fused_kv_proj(x, torch.zeros(6, 7), d_h=2, n_heads=3)

    def test_no_cpu_fallback(self):
        x = torch.zeros(2, 8)
        with pytest.raises(bd.NativeLibraryError):
            bd.fused_kv_proj(x, torch.zeros(6, 6), d_h=2, n_heads=3)

    def test_host_entry_validates_like_reference(self):
        x = np.zeros((2, 8), np.float32)
        with pytest.raises(bd.PrecisionError):
            bd.fused_kv_proj_host(x, np.zeros((6, 6), np.float64), 2, 3)
        with pytest.raises(bd.ShapeError):
            bd.fused_kv_proj_host(x, np.zeros((5, 6), np.float32), 2, 3)
        with pytest.raises(bd.ShapeError):
            bd.fused_kv_proj_host(x, np.zeros((6, 7), np.float32), 2, 3)


def test_flop_accounting_matches_reference_bench():
    # ref bench.py:266 flop_ratio = d / (d - d_h); CSV prints 1.3333 (test_acceptance.py:217)
    assert f"{bd.flop_ratio(512, 128):.4f}" == "1.3333"
    assert bd.flop_ratio(32, 8) == pytest.approx(32 / 24)
    assert bd.kv_flops(8192, 512, 128, 16) * 4 == 3 * 2 * 8192 * 512 * 2048


def test_rmsnorm_and_allgather_entries_reject_bad_arguments(lib):
    """The fused-norm and fused-all-gather entry points validate before launching."""
    before = lib.bd_launch_count()
    p = (N.KvProblem * 1)()
    p[0] = N.KvProblem(1 << 20, 1 << 21, 1 << 22, 16, 16, 16, 4, 16, 8, 2, 8, 0)  # tag FIRST
    g = (ctypes.c_void_p * 1)(1 << 23)
    lay = N.BD_OUT_TOKEN_MAJOR
    assert lib.bd_kv_proj_grouped_rmsnorm(p, 1, N.BD_F16, 0, lay, None, 1e-6, None, None) == N.BD_ERR_ARG
    assert lib.bd_kv_proj_grouped_rmsnorm(p, 1, N.BD_F16, 0, lay, g, -1.0, None, None) == N.BD_ERR_ARG
    nul = (ctypes.c_void_p * 1)(None)
    assert lib.bd_kv_proj_grouped_rmsnorm(p, 1, N.BD_F16, 0, lay, nul, 1e-6, None, None) == N.BD_ERR_ARG
    p[0].mul_base, p[0].rep_base = 0, 0  # slices overlap: not a FIRST / LAST partition
    assert lib.bd_kv_proj_grouped_rmsnorm(p, 1, N.BD_F16, 0, lay, g, 1e-6, None, None) == N.BD_ERR_SHAPE
    bufs = (ctypes.c_void_p * 2)(1 << 24, 1 << 25)
    assert lib.bd_kv_proj_grouped_allgather(p, 1, N.BD_F16, 0, 0, 0, bufs, None, None) == N.BD_ERR_ARG
    assert lib.bd_kv_proj_grouped_allgather(p, 1, N.BD_F16, 0, 2, 2, bufs, None, None) == N.BD_ERR_ARG
    assert lib.bd_kv_proj_grouped_allgather(p, 1, N.BD_F16, 0, 2, 0, None, None, None) == N.BD_ERR_ARG
    assert lib.bd_launch_count() == before


@pytest.mark.parametrize("L,chunks", [(0, 4), (1, 4), (255, 4), (300, 4), (8192, 4), (8192, 1),
                                      (8192, 3), (65536, 8), (1000, 100)])
def test_host_pipeline_row_blocks_partition_the_tokens(L, chunks):
    """The host pipeline's row blocks tile [0, L) exactly, in order, each a whole number of
    256-row CTA-pair tiles except the last (host logic of fused_kv_proj_grouped_host)."""
    from paper_2510_01718_b200.kv_proj import _chunk_bounds
    b = _chunk_bounds(L, chunks)
    if L == 0:
        assert b == []
        return
    assert b[0][0] == 0 and b[-1][1] == L
    assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
    assert all((r1 - r0) % 256 == 0 for r0, r1 in b[:-1])
    assert len(b) <= max(1, chunks)
