"""Development aid: write exp/kv_proj_tc_tl.cu — the TC kernel with per-CTA clock stamps
(globaltimer + clock64 into a __device__ table read back by bd_debug_timeline) for
tools/timeline.py.  Build:  cd paper_2510_01718_b200/csrc && nvcc <build flags> -I. \
    -o ../../exp/tl.so capi.cu kv_proj_exact.cu ../../exp/kv_proj_tc_tl.cu"""
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
import sys
SRC = sys.argv[1] if len(sys.argv) > 1 else "paper_2510_01718_b200/csrc/kv_proj_tc.cu"
s = (ROOT / SRC).read_text()
# patterns apply to the persistent kernel only: set the small-L kernel and after aside
_cut = s.find("// Small-L (\"decode\") kernel")
tail = s[_cut:] if _cut >= 0 else ""
s = s[:_cut] if _cut >= 0 else s


def rep(a, b):
    global s
    assert s.count(a) == 1, a[:70]
    s = s.replace(a, b)


i = s.index("namespace bdk {")
s = (s[:i] + "__device__ unsigned long long g_tl[148][96];\n"
     + '#define GT() ({unsigned long long _g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g)); _g;})\n'
     + "#define CK() ((unsigned long long)clock64())\n" + s[i:])
s += '''
extern "C" int bd_debug_timeline(unsigned long long* dst) {
  return (int)cudaMemcpyFromSymbol(dst, g_tl, sizeof(g_tl));
}
'''
rep('''  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();''', '''  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  unsigned long long* TL = g_tl[blockIdx.x];
  if (threadIdx.x == 0) { TL[0] = GT(); TL[1] = CK(); }''')
rep('''    for (int s = 0; s < A_SLOTS; ++s) {
      mbar_init(&a_full[s], 1);''', '''    TL[2] = CK();
    for (int s = 0; s < A_SLOTS; ++s) {
      mbar_init(&a_full[s], 1);''')
rep('''    mbar_init(rfull, 1);
    fence_mbar_init();''', '''    mbar_init(rfull, 1);
    fence_mbar_init();
    TL[3] = CK();''')
rep('''    tmem_relinquish<CG>();
  }''', '''    tmem_relinquish<CG>();
    if (lane == 0) TL[4] = CK();
  }''')
rep('''  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;''', '''  tc_fence_after();
  if (threadIdx.x == 0) TL[5] = CK();
  const uint32_t tmem_base = *tmem_slot;''')
rep('''      griddep_wait();
      for (int t = t_begin; t < t_end; t += t_step) {''', '''      griddep_wait();
      if (lane == 0) { TL[6] = CK(); TL[45] = GT(); }
      for (int t = t_begin; t < t_end; t += t_step) {''')
for lead in ("0", "lead"):
    a = f'''            const uint32_t bar = mapa_shared(smem_u32(&b_full[s]), {lead});'''
    if s.count(a) == 1:
        rep(a, a + '''
            if (b_iter == 0) TL[7] = CK();''')
rep('''        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();''', '''        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        if (lane == 0 && it < 8) TL[8 + it] = CK();
        unsigned long long bw = 0;''')
rep('''          mbar_wait(&b_full[bs], (b_iter / BST) & 1u);''', '''          const unsigned long long w0 = CK();
          mbar_wait(&b_full[bs], (b_iter / BST) & 1u);
          bw += CK() - w0;''')
for m in ("0x3", "pmask"):
    a = f'''        if (elect_one()) tc_commit_pair(&tfull[acc], {m});
        __syncwarp();'''
    if s.count(a) == 1:
        rep(a, a + '''
        if (lane == 0 && it < 8) { TL[16 + it] = CK(); TL[48 + it] = bw; }''')
rep('''      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();''', '''      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (leader && it < 8) TL[24 + it] = CK();''')
for lead in ("0", "lead"):
    a = f'''        mbar_arrive_remote(mapa_shared(smem_u32(&tempty[acc]), {lead}));'''
    if s.count(a) == 1:
        rep(a, a + '''
        if (it < 8) TL[32 + it] = CK();''')
rep('''    if (lane == 0) tma_store_wait_all<0>();''', '''    if (lane == 0) tma_store_wait_all<0>();
    if (leader) { TL[40] = CK(); TL[41] = GT(); TL[42] = t_end - t_begin; }''')
rep('''        const bool reload_a = P.num_kb > A_SLOTS || key != prev_key;  // the resident operand
        prev_key = key;
        const int my_m0''', '''        const bool reload_a = P.num_kb > A_SLOTS || key != prev_key;  // the resident operand
        if (t == t_begin && lane == 0) TL[43] = CK() + (reload_a ? 0 : 1);
        prev_key = key;
        const int my_m0''')
rep('''            mbar_wait(&a_empty[s], ((a_iter / A_SLOTS) & 1u) ^ 1u);''', '''            mbar_wait(&a_empty[s], ((a_iter / A_SLOTS) & 1u) ^ 1u);
            if (a_iter == 0 && lane == 0) TL[44] = CK();''')
_ext = s.index('extern "C" int bd_debug_timeline')
s = s[:_ext] + tail + "\n" + s[_ext:]
(ROOT / "exp/kv_proj_tc_tl.cu").write_text(s)
print("wrote exp/kv_proj_tc_tl.cu")
