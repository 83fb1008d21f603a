"""The GPU bench harness keeps the reference's CSV contract (ref bench.py:23-35,
test_cli.py:98-128): the reference columns first, in order, then the GPU columns;
``flop_ratio`` printed with 4 decimals; >= 5 reps and >= 2 warm-ups enforced."""

import csv

import pytest
from conftest import ROOT
import torch

from paper_2510_01718_b200 import benchmark as B

REF_COLUMNS = ("operator", "seq_len", "d", "d_h", "n_heads", "precision", "threads",
               "median_ns", "tokens_per_sec", "speedup", "flop_ratio")


def test_csv_columns_extend_the_reference_schema():
    assert B.CSV_COLUMNS[:len(REF_COLUMNS)] == REF_COLUMNS
    assert B.DEFAULT_SEQ_LENS[0] == 64 and B.DEFAULT_SEQ_LENS[-1] == 65536


def test_record_row_and_csv(tmp_path):
    rec = B.BenchRecord(operator=B.FUSED_OPERATOR, seq_len=1024, d=32, d_h=8, n_heads=4,
                        dtype=torch.float16, reps=5, warmup_reps=2, median_ns=1000.0,
                        tokens_per_sec=1.024e9, speedup_vs_baseline=1.25, flop_ratio=32 / 24,
                        tflops=10.0, roofline_frac=0.01, inner_calls=20)
    path = tmp_path / "b.csv"
    B.write_csv(path, [rec])
    rows = list(csv.reader(path.open()))
    assert tuple(rows[0]) == B.CSV_COLUMNS
    row = dict(zip(rows[0], rows[1]))
    assert row["flop_ratio"] == "1.3333"          # ref test_acceptance.py:199-224
    assert row["operator"] == "k_proj_bda_fused" and row["dtype"] == "fp16"
    with pytest.raises(ValueError):
        B.BenchRecord(operator="x", seq_len=1, d=2, d_h=1, n_heads=1, dtype=torch.float16,
                      reps=4, warmup_reps=2, median_ns=1.0, tokens_per_sec=1.0,
                      speedup_vs_baseline=1.0, flop_ratio=1.0, tflops=0.0, roofline_frac=0.0,
                      inner_calls=1)
    with pytest.raises(ValueError):
        B.time_operator_ns(lambda: None, reps=4)


def test_reference_arm_prints_one_contract_line():
    """`bench.py --impl reference` (the driver's reference arm) runs the oracle port on the
    host cores and prints ONE JSON line with the contract's keys, on this CPU-only box."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1", "--tokens", "256"],
                         capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
