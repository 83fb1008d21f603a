"""Development aid: timing-only knobs in the stamped persistent kernel
(exp/kv_proj_tc_tl.cu from tools/instrument.py), to bisect what sets the cfg2 tile period.
Each knob is a -D flag (results are garbage with any knob set):
  NOMMA    the MMA issuer skips tcgen05.mma (commits still arrive: loads, epilogue, barriers
           run as usual) — removes the MMA's shared-memory operand reads
  NOSTG    the epilogue skips its st.shared staging writes (the TMA stores still run)
  NOSTORE  the epilogue skips staging and TMA stores"""
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
p = ROOT / "exp/kv_proj_tc_tl.cu"
s = p.read_text()
cut = s.find('// Small-L ("decode") kernel')
head, tail = s[:cut], s[cut:]


def rep(a, b):
    global head
    assert head.count(a) == 1, a[:60]
    head = head.replace(a, b)


rep("              tc_mma_f16_pair(d_tmem, adesc, bdesc, idesc, (j | ks) != 0 ? 1u : 0u);",
    "#ifndef NOMMA\n              tc_mma_f16_pair(d_tmem, adesc, bdesc, idesc, (j | ks) != 0 ? 1u : 0u);\n#endif")
rep('''          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(o[0]),
                       "r"(o[1]), "r"(o[2]), "r"(o[3])
                       : "memory");''', '''#if !defined(NOSTG) && !defined(NOSTORE)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(o[0]),
                       "r"(o[1]), "r"(o[2]), "r"(o[3])
                       : "memory");
#else
          if (o[0] == 0x12345u && o[1] == 0x777u) asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(o[0]),
                       "r"(o[1]), "r"(o[2]), "r"(o[3])
                       : "memory");
#endif''')
rep('''            if (prm.world > 0) {
              // all-gather fused into the epilogue''', '''#ifdef NOSTORE
            if (false) {
#else
            if (prm.world > 0) {
#endif
              // all-gather fused into the epilogue''')
rep('''            } else if (P.head_major)
              asm volatile(''', '''            }
#ifndef NOSTORE
            else if (P.head_major)
              asm volatile(''')
rep('''                  "r"(stg0), "r"(bcol), "r"(brow)
                  : "memory");
            tma_store_commit();''', '''                  "r"(stg0), "r"(bcol), "r"(brow)
                  : "memory");
#endif
            tma_store_commit();''')
p.write_text(head + tail)
print("knobs added to", p)
