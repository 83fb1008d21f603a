// mla_attn_2tile64.cu — PARKED experiment (not built): a two-query-tile variant of
// csrc/mla_attn.cu with 64-key K/V tiles, three K/V stages and S double-buffered per query
// tile.  It halves the K/V bytes per FLOP and holds a row's 64 scores in registers (one
// TMEM pass).  It was wired into launch_mla_attention behind BD_ATTN_KERNEL and was
// parity-green on tests/test_mla_attn_gpu.py (14/14, first build).  It was SLOWER than the
// shipped one-tile kernel (interleaved, one box): L = 8192: 825 vs 1096 TFLOP/s; L = 32768:
// 904–918 vs 1022–1024.  ncu at L = 8192: tensor pipe active 50 % of active cycles, stall
// samples dominated by long-scoreboard (the softmax's tcgen05.ld waits) — with 64-key
// tiles every per-tile hand-off (TMEM load, P store, barrier round trip) is paid per 64
// keys instead of 128.  See profiles/r02_attention_study.md.  Uses the AttnParams,
// constants and helpers of csrc/mla_attn.cu (paste before `encode` to rebuild).
// ---------------------------------------------------------------------------------
// Two-query-tile kernel: a work item is a PAIR of 128-query tiles of one
// head, both consuming every 64-key K/V tile — half the K/V bytes per FLOP of the one-tile
// kernel, whose tile period is set by how fast the SM can take in K/V (80 KB per 128 keys
// per 128 queries; profiles/r02_attention_study.md).  S is double-buffered per query tile
// (S_x(j+1) runs on the tensor core while softmax x works on S_x(j)); 64-key tiles keep a
// row's scores (64 FP32) in registers for a single TMEM pass and leave shared memory for
// three K/V stages beside both Q tiles.  Warps: 0 TMA producer, 1 TMEM allocator + MMA
// issuer, 2-5 softmax + epilogue of query tile A, 6-9 of query tile B.
// TMEM: S_x[b] at columns 128 x + 64 b (P_x[b] over its first 32), O_x at 256 + 128 x.
constexpr int BKV2 = 64;
constexpr int THREADS2 = 320;
constexpr uint32_t KBLK2 = 64 * 64 * 2;   // 64 rows x 64 16-bit cols (SW128): 8 KB
constexpr uint32_t K2_BYTES = 3 * KBLK2;  // [K'nope 0:64 | K'nope 64:128 | k_pe]
constexpr uint32_t V2_BYTES = 2 * KBLK2;  // two 64-column MN-major panels
constexpr int KV2_STAGES = 3;
constexpr size_t SMEM2_BYTES = 1024 + 2 * Q_BYTES + KV2_STAGES * (K2_BYTES + V2_BYTES) + 256;
static_assert(SMEM2_BYTES <= 232448, "smem (two-tile kernel)");

// item w -> (head, query-tile pair), in L2-sized head groups, longest pairs first
__device__ __forceinline__ void item2_of(const AttnParams& p, int w, int& h, int& qp) {
  const int n_qp = (p.n_qt + 1) / 2;
  const int per = p.hgroup * n_qp;
  const int grp = w / per, r = w - grp * per;
  const int rest = p.H - grp * p.hgroup;
  const int gh = rest < p.hgroup ? rest : p.hgroup;
  qp = n_qp - 1 - r / gh;
  h = grp * p.hgroup + r % gh;
}

template <bool kBF16>
__global__ void __launch_bounds__(THREADS2, 1) mla_attn2_kernel(const __grid_constant__ AttnParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                       // Q_A | Q_B
  uint8_t* sK = sQ + 2 * Q_BYTES;           // KV2_STAGES
  uint8_t* sV = sK + KV2_STAGES * K2_BYTES;  // KV2_STAGES
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + KV2_STAGES * V2_BYTES);
  uint64_t* q_full = bars;
  uint64_t* q_empty = q_full + 1;
  uint64_t* k_full = q_empty + 1;
  uint64_t* k_empty = k_full + KV2_STAGES;
  uint64_t* v_full = k_empty + KV2_STAGES;
  uint64_t* v_empty = v_full + KV2_STAGES;
  uint64_t* s_full = v_empty + KV2_STAGES;  // [x][b]
  uint64_t* p_full = s_full + 4;            // [x][b] (the x tile's 4 softmax warps)
  uint64_t* pv_done = p_full + 4;           // [x] (MMA commit after every PV_x)
  uint64_t* o_free = pv_done + 2;           // [x] (4 warps, after reading O_x)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < KV2_STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&pv_done[x], 1);
      mbar_init(&o_free[x], 4);
    }
    fence_mbar_init();
    tma_prefetch_desc(&prm.map_q);
    tma_prefetch_desc(&prm.map_k);
    tma_prefetch_desc(&prm.map_kpe);
    tma_prefetch_desc(&prm.map_v);
  }
  if (warp == 1) {
    tmem_alloc<1>(tmem_slot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();

  const int G = static_cast<int>(gridDim.x);
  const int nkt_all = (prm.L + BKV2 - 1) / BKV2;
  const int n_items = ((prm.n_qt + 1) / 2) * prm.H;
  // key tiles of query tile x of pair qp (0: the tile lies past L)
  auto n_tiles = [&](int qp, int x) {
    const int qt = 2 * qp + x;
    if (qt >= prm.n_qt) return 0;
    if (!prm.causal) return nkt_all;
    const int n = 2 * qt + 2;  // keys up to the tile's last query
    return n < nkt_all ? n : nkt_all;
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    griddep_wait();
    const uint64_t pol_q = policy_evict_first();
    const uint64_t pol_kv = policy_evict_last();  // K/V tiles are re-read by later queries
    uint32_t kv_it = 0, item_it = 0;
    for (int zk = 0, w = zz_item(0, G); w < n_items; w = zz_item(++zk, G), ++item_it) {
      int h, qp;
      item2_of(prm, w, h, qp);
      const int nA = n_tiles(qp, 0), nB = n_tiles(qp, 1);
      const int jmax = nA > nB ? nA : nB;
      const int nq = nB > 0 ? 2 : 1;
      mbar_wait(q_empty, (item_it & 1u) ^ 1u);
      if (elect_one()) {
        mbar_arrive_expect_tx(q_full, nq * Q_BYTES);
        for (int x = 0; x < nq; ++x)
          for (int b = 0; b < 3; ++b)
            tma_load_3d(sQ + x * Q_BYTES + b * KBLK, &prm.map_q, 64 * b, h, (2 * qp + x) * BQ,
                        q_full, pol_q);
      }
      __syncwarp();
      for (int j = 0; j < jmax; ++j, ++kv_it) {
        const uint32_t st = kv_it % KV2_STAGES, ph = ((kv_it / KV2_STAGES) & 1u) ^ 1u;
        mbar_wait(&k_empty[st], ph);
        if (elect_one()) {
          uint8_t* dk = sK + st * K2_BYTES;
          mbar_arrive_expect_tx(&k_full[st], K2_BYTES);
          tma_load_3d(dk, &prm.map_k, 0, j * BKV2, h, &k_full[st], pol_kv);
          tma_load_3d(dk + KBLK2, &prm.map_k, 64, j * BKV2, h, &k_full[st], pol_kv);
          tma_load_2d(dk + 2 * KBLK2, &prm.map_kpe, 0, j * BKV2, &k_full[st], pol_kv);
        }
        __syncwarp();
        mbar_wait(&v_empty[st], ph);
        if (elect_one()) {
          uint8_t* dv = sV + st * V2_BYTES;
          mbar_arrive_expect_tx(&v_full[st], V2_BYTES);
          tma_load_3d(dv, &prm.map_v, 0, j * BKV2, h, &v_full[st], pol_kv);
          tma_load_3d(dv + KBLK2, &prm.map_v, 64, j * BKV2, h, &v_full[st], pol_kv);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    // Per key tile j: PV_A(j), S_A(j+2), PV_B(j), S_B(j+2) — S_x(j+1) was issued one tile
    // earlier into x's other S buffer, so the softmax of tile j+1 overlaps these.
    constexpr uint32_t idesc_s = make_idesc_f16(kBF16, BQ, BKV2, /*a_mn=*/false, /*b_mn=*/false);
    constexpr uint32_t idesc_o = make_idesc_f16(kBF16, BQ, DV, /*a_mn=*/false, /*b_mn=*/true);
    uint32_t kv_s = 0, kv_v = 0, item_it = 0;
    uint32_t s_cnt[2] = {0u, 0u}, p_cnt[2] = {0u, 0u}, x_items[2] = {0u, 0u};
    auto issue_s = [&](int x, uint32_t st) {  // S_x(next) = Q_x K^T into buffer s_cnt & 1
      if (elect_one()) {
        const uint32_t q0 = smem_u32(sQ + x * Q_BYTES);
        const uint32_t k0 = smem_u32(sK + st * K2_BYTES);
        const uint32_t d = tmem_base + 128u * x + 64u * (s_cnt[x] & 1u);
#pragma unroll
        for (int ks = 0; ks < 12; ++ks) {
          const uint32_t sub = (ks & 3) * 32;
          tc_mma_f16(d, make_smem_desc(q0 + (ks >> 2) * KBLK + sub, 16, 1024),
                     make_smem_desc(k0 + (ks >> 2) * KBLK2 + sub, 16, 1024), idesc_s,
                     ks != 0 ? 1u : 0u);
        }
        tc_commit(&s_full[2 * x + (s_cnt[x] & 1u)]);
      }
      __syncwarp();
      ++s_cnt[x];
    };
    for (int zk = 0, w = zz_item(0, G); w < n_items; w = zz_item(++zk, G), ++item_it) {
      int h, qp;
      item2_of(prm, w, h, qp);
      const int nA = n_tiles(qp, 0), nB = n_tiles(qp, 1);
      const int jmax = nA > nB ? nA : nB;
      mbar_wait(q_full, item_it & 1u);
      for (int t = 0; t < 2 && t < jmax; ++t, ++kv_s) {  // S of key tiles 0 and 1
        const uint32_t st = kv_s % KV2_STAGES;
        mbar_wait(&k_full[st], (kv_s / KV2_STAGES) & 1u);
        tc_fence_after();
        if (t < nA) issue_s(0, st);
        if (t < nB) issue_s(1, st);
        if (elect_one()) tc_commit(&k_empty[st]);
        __syncwarp();
      }
      if (jmax <= 2 && elect_one()) tc_commit(q_empty);  // every S of the item issued
      __syncwarp();
      for (int j = 0; j < jmax; ++j, ++kv_v) {
        const uint32_t vst = kv_v % KV2_STAGES;
        mbar_wait(&v_full[vst], (kv_v / KV2_STAGES) & 1u);
        const uint32_t kst = kv_s % KV2_STAGES;
        bool k_ready = false;
        for (int x = 0; x < 2; ++x) {
          const int n = x == 0 ? nA : nB;
          if (j >= n) continue;
          const uint32_t b = p_cnt[x] & 1u;
          mbar_wait(&p_full[2 * x + b], (p_cnt[x] >> 1) & 1u);
          ++p_cnt[x];
          if (j == 0) mbar_wait(&o_free[x], (x_items[x] & 1u) ^ 1u);  // previous O_x read out
          tc_fence_after();
          if (elect_one()) {
            const uint32_t v0 = smem_u32(sV + vst * V2_BYTES);
            const uint32_t pa = tmem_base + 128u * x + 64u * b;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              tc_mma_f16_ts(tmem_base + 256u + 128u * x, pa + ks * 8,
                            make_smem_desc(v0 + ks * (16 * 128), KBLK2, 1024), idesc_o,
                            (j | ks) != 0 ? 1u : 0u);
            tc_commit(&pv_done[x]);
          }
          __syncwarp();
          if (j + 2 < n) {
            if (!k_ready) {
              mbar_wait(&k_full[kst], (kv_s / KV2_STAGES) & 1u);
              tc_fence_after();
              k_ready = true;
            }
            issue_s(x, kst);
          }
        }
        if (elect_one()) {
          tc_commit(&v_empty[vst]);  // both PVs of tile j issued
          if (k_ready) {
            tc_commit(&k_empty[kst]);                     // both S of tile j + 2 issued
            if (j + 3 == jmax) tc_commit(q_empty);        // the item's last S issued
          }
        }
        __syncwarp();
        if (k_ready) ++kv_s;
      }
      if (nA > 0) ++x_items[0];
      if (nB > 0) ++x_items[1];
    }
  } else {
    // ---------------------------------------------------------------- softmax + epilogue
    const uint32_t x = (warp - 2) >> 2;  // query tile A (0) or B (1)
    const uint32_t quad = warp & 3;
    const uint32_t lane_base = (quad * 32u) << 16;
    const uint32_t to = tmem_base + lane_base + 256u + 128u * x;  // O_x
    uint32_t s_it = 0, pv_it = 0;
    const float c2 = prm.scale_log2;
    for (int zk = 0, w = zz_item(0, G); w < n_items; w = zz_item(++zk, G)) {
      int h, qp;
      item2_of(prm, w, h, qp);
      const int n = n_tiles(qp, static_cast<int>(x));
      if (n == 0) continue;
      const int qt = 2 * qp + static_cast<int>(x);
      const int row = qt * BQ + static_cast<int>(quad * 32 + lane);  // query (token) index
      float m = -INFINITY;  // running max, in log2 units of scale*s
      float l = 0.f;
      for (int j = 0; j < n; ++j, ++s_it) {
        const uint32_t b = s_it & 1u;
        mbar_wait(&s_full[2 * x + b], (s_it >> 1) & 1u);
        tc_fence_after();
        const uint32_t ta = tmem_base + lane_base + 128u * x + 64u * b;
        uint32_t sr[64];
        tmem_ld_32x32b_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        tmem_ld_32x32b_x32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tmem_ld_wait();
        // mask: causal (key > query) and keys past L
        int valid = prm.L - j * BKV2;
        if (prm.causal) valid = min(valid, row - j * BKV2 + 1);
        float mx0 = -INFINITY, mx1 = -INFINITY;
        if (valid >= BKV2) {
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            mx0 = fmaxf(mx0, __uint_as_float(sr[c]));
            mx1 = fmaxf(mx1, __uint_as_float(sr[c + 1]));
          }
        } else {
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            if (c >= valid) sr[c] = __float_as_uint(-INFINITY);
            mx0 = fmaxf(mx0, __uint_as_float(sr[c]));
          }
        }
        const float m_tile = fmaxf(mx0, mx1) * c2;
        if (m_tile > m + RESCALE_LOG2) {
          // lazy rescale: the reference max moves (always on the first tile)
          if (j > 0) {
            const float alpha = ex2(m - m_tile);
            l *= alpha;
            // O_x row *= alpha: PV_x(j-1) must have landed (PV_x(j) waits for our P_x(j))
            mbar_wait(&pv_done[x], (pv_it - 1) & 1u);
            tc_fence_after();
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              uint32_t o[32];
              tmem_ld_32x32b_x32(to + cc * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st_32x32b_x32(to + cc * 32, o);
            }
            tmem_st_wait();
          }
          m = m_tile;
        }
        // p = exp2(s c2 - m), l += p, P packed to 16 bit over S's first 32 columns
        uint32_t pk[32];
        float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float p0 = ex2(fmaf(__uint_as_float(sr[c]), c2, -m));
          const float p1 = ex2(fmaf(__uint_as_float(sr[c + 1]), c2, -m));
          ls0 += p0;
          ls1 += p1;
          pk[c >> 1] = pack_p<kBF16>(p0, p1);
        }
        l += ls0 + ls1;
        tmem_st_32x32b_x32(ta, pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[2 * x + b]);
        ++pv_it;  // PV_x(j) will be the pv_it-th PV_x issued
        // observe every pv_done phase (PV_x(j-1): see the one-tile kernel)
        if (j > 0) mbar_wait(&pv_done[x], (pv_it - 2) & 1u);
      }
      // epilogue: O_x / l straight to global (this thread's row: 256 contiguous bytes)
      mbar_wait(&pv_done[x], (pv_it - 1) & 1u);
      tc_fence_after();
      const float inv = 1.0f / l;
      const bool live = row < prm.L;
      uint16_t* dst = static_cast<uint16_t*>(prm.out) +
                      static_cast<int64_t>(live ? row : 0) * prm.ldo_tok +
                      static_cast<int64_t>(h) * prm.ldo_head;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(to + cc * 32, o);
        tmem_ld_wait();
        if (live) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 v;
            v.x = pack2<kBF16>(__uint_as_float(o[8 * g + 0]) * inv, __uint_as_float(o[8 * g + 1]) * inv);
            v.y = pack2<kBF16>(__uint_as_float(o[8 * g + 2]) * inv, __uint_as_float(o[8 * g + 3]) * inv);
            v.z = pack2<kBF16>(__uint_as_float(o[8 * g + 4]) * inv, __uint_as_float(o[8 * g + 5]) * inv);
            v.w = pack2<kBF16>(__uint_as_float(o[8 * g + 6]) * inv, __uint_as_float(o[8 * g + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + cc * 32 + g * 8) = v;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[x]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 512);
  }
}

