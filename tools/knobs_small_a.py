"""Development aid: timing-only variant of the small-L PAIR kernel in which every column
block's pair reads its OWN copy of the x rows (rows offset by 256 x column block inside an
x allocation 64x taller than L; build with -DUNSHARED_A) — tests whether the 32+ pairs of
a row block reading the same A lines is an L2 hot spot.  Writes xb/kv_proj_tc_ua.cu."""
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
s = (ROOT / "paper_2510_01718_b200/csrc/kv_proj_tc.cu").read_text()


def rep(a, b):
    global s
    assert s.count(a) == 1, a[:70]
    s = s.replace(a, b)


rep("          tma_load_2d_pair(sA + kb * a_kb, &P.map_a, kb * BK, m0, bar, pol);",
    """#ifdef UNSHARED_A
          tma_load_2d_pair(sA + kb * a_kb, &P.map_a, kb * BK,
                           m0 + (static_cast<int>(blockIdx.x) / CGS % 64) * (BM * CGS), bar, pol);
#else
          tma_load_2d_pair(sA + kb * a_kb, &P.map_a, kb * BK, m0, bar, pol);
#endif""")
rep("    if (!encode_2d(&P.map_a, xb, bf16, q.K, q.L, q.ldx, BK, a_rows, &err) ||",
    """#ifdef UNSHARED_A
    if (!encode_2d(&P.map_a, xb, bf16, q.K, q.L * 64, q.ldx, BK, a_rows, &err) ||
#else
    if (!encode_2d(&P.map_a, xb, bf16, q.K, q.L, q.ldx, BK, a_rows, &err) ||
#endif""")
(ROOT / "xb").mkdir(exist_ok=True)
(ROOT / "xb/kv_proj_tc_ua.cu").write_text(s)
print("wrote xb/kv_proj_tc_ua.cu")
