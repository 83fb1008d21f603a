"""Development aid: write xb/mla_attn_tl.cu — the MLA attention kernel with clock64 stamps
of CTA 0's first work item (tiles j < 64), read back by bd_debug_attn_timeline; analysed
by tools/attn_timeline.py.  Build (from the repo root):
  python tools/instrument_attn.py && C=paper_2510_01718_b200/csrc && nvcc <lib flags> -I$C \\
    -o xb/attnstamp.so $C/capi.cu $C/kv_proj_exact.cu $C/kv_proj_tc.cu xb/mla_attn_tl.cu
Stamps: [0] producer issues K_j, [1] producer issues V_j, [2] MMA issuer saw P_j, [3] MMA
issued S_j, [4] softmax warp 2 saw S_j, [5] softmax warp 2 published P_j."""
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
s = (ROOT / "paper_2510_01718_b200/csrc/mla_attn.cu").read_text()


def rep(a, b):
    global s
    assert s.count(a) == 1, a[:70]
    s = s.replace(a, b)


rep('''template <bool kBF16>
__global__ void __launch_bounds__(THREADS, 1) mla_attn_kernel(''', '''__device__ long long g_attn_tl[6][64];
#define ATTN_STAMP(k, j) \\
  do { if (blockIdx.x == 0 && item_it == 0 && (j) < 64) g_attn_tl[k][j] = clock64(); } while (0)

template <bool kBF16>
__global__ void __launch_bounds__(THREADS, 1) mla_attn_kernel(''')
rep('''        if (elect_one()) {
          uint8_t* dk = sK + st * K_BYTES;''', '''        if (elect_one()) {
          ATTN_STAMP(0, j);
          uint8_t* dk = sK + st * K_BYTES;''')
rep('''        if (elect_one()) {
          uint8_t* dv = sV + st * V_BYTES;''', '''        if (elect_one()) {
          ATTN_STAMP(1, j);
          uint8_t* dv = sV + st * V_BYTES;''')
rep('''        tc_commit(&s_full[sb]);
        tc_commit(&k_empty[st]);''', '''        tc_commit(&s_full[sb]);
        tc_commit(&k_empty[st]);
        ATTN_STAMP(3, static_cast<int>(s_it - s_item0));''')
rep('''    uint32_t s_it = 0, pv_it = 0, item_it = 0;
    const uint32_t q0 = smem_u32(sQ);''', '''    uint32_t s_it = 0, pv_it = 0, item_it = 0, s_item0 = 0;
    const uint32_t q0 = smem_u32(sQ);''')
rep('''      mbar_wait(q_full, item_it & 1u);
      const uint32_t s_base = s_it;''', '''      mbar_wait(q_full, item_it & 1u);
      const uint32_t s_base = s_it;
      s_item0 = s_it;''')
rep('''        if (j == 0) mbar_wait(o_free, (item_it & 1u) ^ 1u);  // previous item's O read out
        tc_fence_after();''', '''        if (j == 0) mbar_wait(o_free, (item_it & 1u) ^ 1u);  // previous item's O read out
        tc_fence_after();
        if (lane == 0) ATTN_STAMP(2, j);''')
rep('''    uint32_t s_it = 0, pv_it = 0;
    const float c2 = prm.scale_log2;
    for (int w = static_cast<int>(blockIdx.x); w < prm.total_items; w += G) {''', '''    uint32_t s_it = 0, pv_it = 0, item_it = 0;
    const float c2 = prm.scale_log2;
    for (int w = static_cast<int>(blockIdx.x); w < prm.total_items; w += G, ++item_it) {''')
rep('''        mbar_wait(&s_full[sb], (s_it / S_BUFS) & 1u);
        tc_fence_after();''', '''        mbar_wait(&s_full[sb], (s_it / S_BUFS) & 1u);
        tc_fence_after();
        if (warp == 2 && lane == 0) ATTN_STAMP(4, j);''')
rep('''        if (lane == 0) mbar_arrive(&p_full[sb]);''', '''        if (lane == 0) mbar_arrive(&p_full[sb]);
        if (warp == 2 && lane == 0) ATTN_STAMP(5, j);''')
s = s.rstrip() + '''

extern "C" int bd_debug_attn_timeline(long long* dst) {
  return (int)cudaMemcpyFromSymbol(dst, bdk::attn::g_attn_tl, sizeof(bdk::attn::g_attn_tl));
}
'''
(ROOT / "xb").mkdir(exist_ok=True)
(ROOT / "xb/mla_attn_tl.cu").write_text(s)
print("wrote xb/mla_attn_tl.cu")
