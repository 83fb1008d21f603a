"""Development aid: write xb/kv_proj_tc_stl.cu — the shipped kernels with globaltimer
stamps in the small-L (decode) kernel, kept for the last 8 launches of every CTA index
(read back by bd_debug_small_timeline).  Build + analysis: tools/small_timeline2.py.

Stamps (ns, globaltimer): 0 entry, 1 after TMEM alloc + sync, 2 producer after PDL wait,
3 MMA issuer saw the last k-block land, 4 epilogue saw the MMAs done, 5 epilogue stores
drained, 6 before TMEM dealloc."""
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
src = (ROOT / "paper_2510_01718_b200/csrc/kv_proj_tc.cu").read_text()
cut = src.find('// Small-L ("decode") kernel')
head, s = src[:cut], src[cut:]


def rep(a, b, count=1):
    global s
    assert s.count(a) == count, (s.count(a), a[:80])
    s = s.replace(a, b)


rep('''  const uint32_t rank = CGS == 2 ? cluster_ctarank() : 0u;  // 0 = pair leader
''', '''  const uint32_t rank = CGS == 2 ? cluster_ctarank() : 0u;  // 0 = pair leader
  __shared__ unsigned long long* TLp;
  if (threadIdx.x == 0) {
    const unsigned slot = atomicAdd(&g_stl_cnt[blockIdx.x % 512], 1u) & 7u;
    TLp = g_stl[slot][blockIdx.x % 512];
    TLp[0] = GT();
  }
''')
rep('''  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();
''', '''  const uint32_t tmem_base = *tmem_slot;
  unsigned long long* TL = TLp;
  if (threadIdx.x == 0) TL[1] = GT();
  griddep_launch_dependents();
''')
rep('''    griddep_wait();
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();  // C is shared by the row... and re-read''',
    '''    griddep_wait();
    if (lane == 0) TL[2] = GT();
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();  // C is shared by the row... and re-read''')
rep('''        mbar_wait(&full[kb], 0);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a0 = smem_u32(sA + kb * a_kb);''', '''        mbar_wait(&full[kb], 0);
        tc_fence_after();
        if (lane == 0 && kb + 1 == P.num_kb) TL[3] = GT();
        if (lane == 0 && kb == 0) TL[7] = GT();
        if (elect_one()) {
          const uint32_t a0 = smem_u32(sA + kb * a_kb);''')
rep('''    mbar_wait(done, 0);
    tc_fence_after();
    if constexpr (kTma) {''', '''    mbar_wait(done, 0);
    tc_fence_after();
    if (warp == 2 && lane == 0) TL[4] = GT();
    if constexpr (kTma) {''')
rep('''    if constexpr (kCheck) {
      if (__any_sync(0xffffffffu, nonfinite2<kBF16>(chk)) && lane == 0) atomicExch(prm.flag, 1);
    }
  }
  tc_fence_before();''', '''    if constexpr (kCheck) {
      if (__any_sync(0xffffffffu, nonfinite2<kBF16>(chk)) && lane == 0) atomicExch(prm.flag, 1);
    }
    if (warp == 2 && lane == 0) TL[5] = GT();
  }
  tc_fence_before();''')
rep('''  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CGS>(tmem_base, BNS);
  }''', '''  if (threadIdx.x == 0) TL[6] = GT();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CGS>(tmem_base, BNS);
  }''')
i = head.index("namespace bdk {")
head = (head[:i] + "__device__ unsigned long long g_stl[8][512][8];\n__device__ unsigned g_stl_cnt[512];\n"
        + '#define GT() ({unsigned long long _g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g) :: "memory"); _g;})\n'
        + head[i:])
s = head + s + '''
extern "C" int bd_debug_small_timeline(unsigned long long* dst) {
  return (int)cudaMemcpyFromSymbol(dst, g_stl, sizeof(g_stl));
}
extern "C" int bd_debug_small_reset() {
  static unsigned z[512] = {};
  static unsigned long long zz[8 * 512 * 8] = {};
  cudaMemcpyToSymbol(g_stl_cnt, z, sizeof(z));
  return (int)cudaMemcpyToSymbol(g_stl, zz, sizeof(zz));
}
'''
# timing-only knobs (-DSKIP_LOADS / -DSKIP_MMA / -DSKIP_STORES / -DSKIP_REP): bisect
# where a decode launch's time goes (results are garbage with any knob set)
s = s.replace("""      for (int kb = 0; kb < P.num_kb; ++kb) {
        if constexpr (CGS == 2) {
          if (rank == 0) mbar_arrive_expect_tx(&full[kb], CGS * (a_kb + BS_BYTES));""",
"""#ifdef SKIP_LOADS
      for (int kb = 0; kb < P.num_kb; ++kb) if (rank == 0) mbar_arrive(&full[kb]);
      for (int kb = 0; kb < 0; ++kb) {
#else
      for (int kb = 0; kb < P.num_kb; ++kb) {
#endif
        if constexpr (CGS == 2) {
          if (rank == 0) mbar_arrive_expect_tx(&full[kb], CGS * (a_kb + BS_BYTES));""")
s = s.replace("""#pragma unroll
          for (int ks = 0; ks < BK / UK; ++ks) {
            const uint64_t ad = make_smem_desc(a0 + ks * (UK * 2), 16, 1024);""",
"""#ifndef SKIP_MMA
#pragma unroll
#else
          if (kb < 0)
#endif
          for (int ks = 0; ks < BK / UK; ++ks) {
            const uint64_t ad = make_smem_desc(a0 + ks * (UK * 2), 16, 1024);""")
s = s.replace("""        *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);""",
"""#ifndef SKIP_STORES
        *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);
#else
        if (o[0] == 0x12345678u) *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);
#endif""")
s = s.replace("""      xr[j] = (live && P.has_rep && col < P.N)""", """#ifdef SKIP_REP
      xr[j] = make_uint4(j, 0, 0, 0); if (false)
#endif
      xr[j] = (live && P.has_rep && col < P.N)""")
# -DSPIN: the MMA issuer's and the epilogue's barrier waits poll with test_wait
s = s.replace("""        mbar_wait(&full[kb], 0);
        tc_fence_after();
        if (lane == 0 && kb + 1 == P.num_kb) TL[3] = GT();""", """#ifdef SPIN
        mbar_wait_spin(&full[kb], 0);
#else
        mbar_wait(&full[kb], 0);
#endif
        tc_fence_after();
        if (lane == 0 && kb + 1 == P.num_kb) TL[3] = GT();""")
s = s.replace("""    mbar_wait(done, 0);
    tc_fence_after();
    if (warp == 2 && lane == 0) TL[4] = GT();""", """#ifdef SPIN
    mbar_wait_spin(done, 0);
#else
    mbar_wait(done, 0);
#endif
    tc_fence_after();
    if (warp == 2 && lane == 0) TL[4] = GT();""")
(ROOT / "xb").mkdir(exist_ok=True)
(ROOT / "xb/kv_proj_tc_stl.cu").write_text(s)
print("wrote xb/kv_proj_tc_stl.cu")
