// attention_2cta.cu -- §8 row a6 on a CTA pair: zero-copy paged attention with cta_group::2 MMAs.
//
// Same math as attention.cu:
//   O[b,p,h] = sum_{t in A(p)} softmax_t(scale q_p.k_t) v_t,  A(p) = {t : t/bs in T[b,h/E], t <= P+p}
// with causal masking in absolute positions.
//
// Cluster of 2 CTAs = (b, group g, 128-token q-tile, head pair {h0, h0+1} of g). CTA r holds the
// 128 query rows of head h0+r; every tcgen05.mma is M=256 (both CTAs' rows) and issued by CTA 0.
// Each page is split across the pair: CTA r loads keys [r*bs/2, (r+1)*bs/2) of K and head-dim
// columns [64r, 64r+64) of V, so per SM the tensor core reads 6 KB of shared memory per 64-cycle
// S MMA (96 B/clk, under the 128 B/clk limit that caps a 1-CTA 128x128 SS MMA) and the TMA / L2
// traffic per FLOP halves. P (fp16) aliases S^b; the MMA computes S(n+1) while the softmax of S(n)
// runs. Both softmax warpgroups work on every page: WG w owns key columns [w BS/2, (w+1) BS/2) of
// each S^b and keeps its own running max / sum and accumulator O_w (P.V of its half of the keys),
// so the two WGs never exchange anything per page; the epilogue merges (m_w, l_w, O_w).
// TMEM per CTA: S^0 [0,128) S^1 [128,256) O_0 [256,384) O_1 [384,512).
// Warps: 0-7 softmax (WG = warp/4, lane quarter = warp%4), 8-9 V bf16->fp16 converters,
// 10 TMA producer, 11 TMEM alloc + MMA issuer.
#include "common.cuh"
#include "geo.cuh"
#include "out_store.cuh"

namespace cpa {

#ifdef CPA_TRACE
__device__ long long g_trace2[32][2048];
#define TRACE2(e, i) \
  do { if (blockIdx.x == 0 && (i) < 2048) g_trace2[e][i] = clock64(); } while (0)
#else
#define TRACE2(e, i) do {} while (0)
#endif

template <int BS>
struct Attn2Cfg {
  static constexpr int D = 128;
  static constexpr int kQBytes = 128 * D * 2;           // this CTA's Q tile
  static constexpr int kKHalf = (BS / 2) * D * 2;       // half of a K page (keys)
  static constexpr int kVHalf = BS * 64 * 2;            // half of a V page (head-dim columns)
#ifndef CPA_KSTAGES
#define CPA_KSTAGES 4
#endif
#ifndef CPA_VSTAGES
#define CPA_VSTAGES 4
#endif
  static constexpr int kKStages = CPA_KSTAGES, kVStages = CPA_VSTAGES;
  static constexpr int kConvWarps = 2;
  static constexpr int kThreads = 12 * 32;       // 8 softmax + 2 converter + TMA + MMA warps
  static constexpr int kSmem = kQBytes + kKStages * kKHalf + kVStages * kVHalf + 1024 + 512;
  static_assert(kSmem <= 232448, "shared memory budget");
};

template <int BS, bool PF16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    k_paged_attn_2cta(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k_half,
                      const __grid_constant__ CUtensorMap tm_v, Geo g, AttnArgs args) {
  using Cfg = Attn2Cfg<BS>;
  constexpr int D = Cfg::D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::kQBytes;
  uint8_t* sV = sK + Cfg::kKStages * Cfg::kKHalf;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + Cfg::kVStages * Cfg::kVHalf);
  uint64_t* q_full = bars;                          // leader: both Q tiles landed (tx)
  uint64_t* k_full = q_full + 1;                    // leader: both K halves landed (tx)
  uint64_t* k_empty = k_full + Cfg::kKStages;       // both: K stage consumed (multicast commit)
  uint64_t* v_full = k_empty + Cfg::kKStages;       // local: own V half landed (tx)
  uint64_t* v_empty = v_full + Cfg::kVStages;       // both: V stage consumed (multicast commit)
  uint64_t* v_ready = v_empty + Cfg::kVStages;      // leader: both V halves converted (4 arrivals)
  uint64_t* s_full = v_ready + Cfg::kVStages;       // both [2]: S^b computed (multicast commit)
  uint64_t* p_full = s_full + 2;                    // leader [2][2]: P^b columns of WG w written
  uint64_t* pv_done = p_full + 4;                   // both [2]: last P.V into O_w complete
  uint64_t* o_full = pv_done + 2;                   // both: every MMA complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);
  int* n_blocks_s = reinterpret_cast<int*>(tmem_slot + 1);
  int* row_start_s = n_blocks_s + 1;
  int* n_diag_s = row_start_s + 1;

  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
  // ---- tile coordinates; one cluster = one (b, g, q-tile, head pair). Execution-group-major order
  // (heaviest q-tile first within a group) so the clusters in flight share few groups' KV pages in L2.
  const int cl = (int)blockIdx.x >> 1;
  const int HP = g.E / 2;
  const int nqt = (g.C + 127) / 128;
  const int hp = cl % HP;
  const int qt = nqt - 1 - (cl / HP) % nqt;
  const int bg = cl / (HP * nqt);
  const int grp = bg % g.Gn;
  const int b = bg / g.Gn;
  const int p0 = qt * 128;
  const int h = grp * g.E + hp * 2 + (int)cta;  // this CTA's query head
  const int kvh = group_kv_head(g, grp);

  const uint32_t warp = warp_id(), lane = lane_id();
  constexpr uint32_t kConvWarp0 = 8, kTmaWarp = 10, kMmaWarp = 11;

  if (warp == kTmaWarp && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k_half);
    tma_prefetch_desc(&tm_v);
    mbar_init(q_full, 1);
    for (int s = 0; s < Cfg::kKStages; ++s) { mbar_init(k_full + s, 1); mbar_init(k_empty + s, 1); }
    for (int s = 0; s < Cfg::kVStages; ++s) {
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
      mbar_init(v_ready + s, 2 * Cfg::kConvWarps);
    }
    mbar_init(s_full, 1);
    mbar_init(s_full + 1, 1);
    for (int i = 0; i < 4; ++i) mbar_init(p_full + i, 8);  // 4 softmax warps of WG w x 2 CTAs
    mbar_init(pv_done, 1);
    mbar_init(pv_done + 1, 1);
    mbar_init(o_full, 1);
    fence_barrier_init();
    const int last_abs = g.P + min(p0 + 127, g.C - 1);
    const int jmax = last_abs / g.bs;
    const int r = b * g.Gn + grp;
    int start = 0, n = jmax + 1;
    if (args.indptr != nullptr) {
      start = args.indptr[r];
      int lo = start, hi = args.indptr[r + 1];  // first index with kv_indices > jmax
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (args.indices[mid] <= jmax) lo = mid + 1; else hi = mid;
      }
      n = lo - start;
    }
    // table entries before n_diag are fully visible to every row of the tile (no causal mask)
    const int jfull = (g.P + p0 + 1) / g.bs - 1;  // last block with j*bs + bs - 1 <= P + p0
    int nd = jfull + 1;
    if (args.indptr != nullptr) {
      int lo = start, hi = start + n;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (args.indices[mid] <= jfull) lo = mid + 1; else hi = mid;
      }
      nd = lo - start;
    }
    *n_blocks_s = n;
    *row_start_s = start;
    *n_diag_s = min(nd, n);
  }
  if (warp == kMmaWarp) tmem_alloc2<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // peer barriers initialised, TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int N = *n_blocks_s;
  const int row_start = *row_start_s;
  const int n_diag = *n_diag_s;

  if (warp == kTmaWarp) {
    if (N > 0) {  // ------------------------------------------------------------ TMA producer
      if (elect_one()) {
        if (leader) mbar_expect_tx(q_full, 2 * Cfg::kQBytes);
        tma_load_4d_2sm(sQ, &tm_q, q_full, 0, h, p0, b);
        tma_load_4d_2sm(sQ + 128 * 128, &tm_q, q_full, 64, h, p0, b);
      }
      __syncwarp();
      const int32_t* ptab = args.page_table + (long long)b * g.maxb;
      for (int n = 0; n < N; ++n) {
        const int j = args.indptr != nullptr ? __ldg(args.indices + row_start + n) : n;
        const int page = __ldg(ptab + j);
        const int ks = n % Cfg::kKStages, vs = n % Cfg::kVStages;
        mbar_wait(k_empty + ks, ((n / Cfg::kKStages) & 1) ^ 1);
        if (elect_one()) {
          if (leader) mbar_expect_tx(k_full + ks, 2 * Cfg::kKHalf);
          uint8_t* dst = sK + ks * Cfg::kKHalf;
          tma_load_4d_2sm(dst, &tm_k_half, k_full + ks, 0, (int)cta * (BS / 2), kvh, page);
          tma_load_4d_2sm(dst + (BS / 2) * 128, &tm_k_half, k_full + ks, 64, (int)cta * (BS / 2), kvh, page);
        }
        __syncwarp();
        mbar_wait(v_empty + vs, ((n / Cfg::kVStages) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(v_full + vs, Cfg::kVHalf);
          tma_load_4d(sV + vs * Cfg::kVHalf, &tm_v, v_full + vs, 64 * (int)cta, 0, kvh, page);
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    if (leader && N > 0) {  // ---------------------------------------------------- MMA issuer (CTA 0)
      constexpr uint32_t idesc_s = umma_idesc_bf16(256, BS, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(256, D, 0, 1) & ~(PF16 ? ((7u << 7) | (7u << 10)) : 0u);
      const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
      auto issue_s = [&](int n) {  // S^{n%2} = Q K_n^T, M=256 (both CTAs' rows), N=BS, K=d
        const uint32_t d_tm = tmem + (n & 1) * 128;
        const uint32_t kb = k_base + (n % Cfg::kKStages) * Cfg::kKHalf;
        if (elect_one()) {
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ad = umma_desc_sw128(q_base + a * 128 * 128 + kk * 32, 16, 1024);
              const uint64_t bd = umma_desc_sw128(kb + a * (BS / 2) * 128 + kk * 32, 16, 1024);
              mma2_ss(d_tm, ad, bd, idesc_s, (a | kk) != 0);
            }
          tc_commit2(s_full + (n & 1));
          tc_commit2(k_empty + n % Cfg::kKStages);
        }
        __syncwarp();
      };
      // O_w += P_w V_n[w-half keys]: WG w's P (keys [w BS/2, (w+1) BS/2) of page n, fp16 packed over its
      // S^b columns) times those V rows; M=256, N=d (64 cols per CTA), K=BS/2
      auto issue_pv = [&](int n, int w) {
        const uint32_t p_tm = tmem + (n & 1) * 128 + w * (BS / 2);
        const uint32_t o_tm = tmem + 256 + w * 128;
        const uint32_t vb = v_base + (n % Cfg::kVStages) * Cfg::kVHalf + w * (BS / 2) * 128;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BS / 32; ++kk) {
            const uint64_t bd = umma_desc_sw128(vb + kk * 16 * 128, BS * 128, 1024);
            mma2_ts(o_tm, p_tm + kk * 8, bd, idesc_o, (n > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit2(pv_done + w);
          if (w == 1) tc_commit2(v_empty + n % Cfg::kVStages);
        }
        __syncwarp();
      };
      auto wait_k = [&](int n) {
        mbar_wait(k_full + n % Cfg::kKStages, (n / Cfg::kKStages) & 1);
        tc_fence_after();
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int n = 0; n < 2 && n < N; ++n) {
        wait_k(n);
        issue_s(n);
      }
      for (int n = 0; n < N; ++n) {
        mbar_wait(v_ready + n % Cfg::kVStages, (n / Cfg::kVStages) & 1);
        if (lane == 0) TRACE2(1, n);
        mbar_wait(p_full + 2 * (n & 1), (n >> 1) & 1);
        if (lane == 0) TRACE2(2, n);
        tc_fence_after();
        issue_pv(n, 0);
        mbar_wait(p_full + 2 * (n & 1) + 1, (n >> 1) & 1);
        tc_fence_after();
        issue_pv(n, 1);
        if (lane == 0) TRACE2(9, n);
        if (n + 2 < N) {
          wait_k(n + 2);
          if (lane == 0) TRACE2(10, n);
          issue_s(n + 2);
        }
        if (lane == 0) TRACE2(3, n);
      }
      if (elect_one()) tc_commit2(o_full);
      __syncwarp();
    }
  } else if (warp >= kConvWarp0) {  // --------------------------------------- V bf16 -> fp16
    const int ct = (warp - kConvWarp0) * 32 + lane;
    for (int n = 0; n < N; ++n) {
      const int vs = n % Cfg::kVStages;
      mbar_wait(v_full + vs, (n / Cfg::kVStages) & 1);
      if (ct == 0) TRACE2(7, n);
#ifndef CPA_EXP_NO_CONV
      if constexpr (PF16) {
#else
      if constexpr (false) {
#endif
        // all loads first (16 x 16 B in flight per thread), then convert + store
        constexpr int kPer = Cfg::kVHalf / 16 / (Cfg::kConvWarps * 32);
        uint4* tile = reinterpret_cast<uint4*>(sV + vs * Cfg::kVHalf);
        uint4 w[kPer];
#pragma unroll
        for (int i = 0; i < kPer; ++i) w[i] = tile[ct + i * Cfg::kConvWarps * 32];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          w[i].x = bf16x2_to_f16x2(w[i].x);
          w[i].y = bf16x2_to_f16x2(w[i].y);
          w[i].z = bf16x2_to_f16x2(w[i].z);
          w[i].w = bf16x2_to_f16x2(w[i].w);
          tile[ct + i * Cfg::kConvWarps * 32] = w[i];
        }
        fence_proxy_async_smem();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(v_ready + vs, 0);
      if (ct == 0) TRACE2(8, n);
    }
  } else {  // ------------------------------------------------------------------ softmax / epilogue
    __shared__ float xml[2][2][128];  // [WG][m, l][row] for the final merge
    const int wg = warp >> 2, quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int p = p0 + row;
    const int lim = min(g.P + p, g.L - 1);
    const float sl2 = g.scale * 1.4426950408889634f;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    constexpr int HC = BS / 2;                                // key columns of a page per WG
    const uint32_t s_tm0 = tmem + lane_off + wg * HC;         // WG's columns of S^0 (this row's lanes)
    const uint32_t o_tm = tmem + lane_off + 256 + wg * 128;  // O_wg
    float m_run = -INFINITY, l_run = 0.f;
    // Both WGs work on every page: WG w owns key columns [w BS/2, (w+1) BS/2) of each S^b with its own
    // running max / sum and its own accumulator O_w (no cross-WG exchange until the epilogue merge).
    for (int n = 0; n < N; ++n) {
      const uint32_t s_tm = s_tm0 + (n & 1) * 128;
      if (row == 0) TRACE2(4 + 16 * wg, n);
      mbar_wait(s_full + (n & 1), (n >> 1) & 1);
      if (row == 0) TRACE2(5 + 16 * wg, n);
      tc_fence_after();
#ifdef CPA_EXP_NO_SOFTMAX  // A/B only: MMA / TMA / converter pipeline alone (wrong results)
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(p_full + 2 * (n & 1) + wg, 0);
      continue;
#endif
      uint32_t sv[HC / 32][32];
#pragma unroll
      for (int k = 0; k < HC / 32; ++k) tmem_ld32(s_tm + k * 32, sv[k]);
      tmem_wait_ld();
      if (n >= n_diag) {  // block crosses the causal diagonal of this tile: mask in absolute positions
        const int j = args.indptr != nullptr ? __ldg(args.indices + row_start + n) : n;
        const int tbase = j * g.bs + wg * HC;
#pragma unroll
        for (int k = 0; k < HC / 32; ++k)
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (tbase + k * 32 + c > lim) sv[k][c] = __float_as_uint(-INFINITY);
      }
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int k = 0; k < HC / 32; ++k)
#pragma unroll
        for (int c = 0; c < 32; c += 8)
#pragma unroll
          for (int w4 = 0; w4 < 4; ++w4)
            m4[w4] = fmax3(m4[w4], __uint_as_float(sv[k][c + 2 * w4]), __uint_as_float(sv[k][c + 2 * w4 + 1]));
      const float m_blk = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * sl2;
      float f = 1.f;
      const bool rescale = m_blk > m_run + 8.0f;  // lazy rescale (first block always lands here)
      if (rescale) {
        if (m_run != -INFINITY) f = fast_exp2(m_run - m_blk);
        m_run = m_blk;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      if (row == 0) TRACE2(11 + 16 * wg, n);
      // P = exp2(s*sl2 - m): packed f32x2 FFMA; pairs chosen by use_poly_exp on a degree-3
      // polynomial (FMA pipe), the rest on MUFU.EX2; 4 partial f32x2 sums; fp16 pack; stored over S.
      float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
      for (int k = 0; k < HC / 32; ++k) {
        uint32_t pk[16];
#pragma unroll
        for (int q2 = 0; q2 < 16; ++q2) {
          float2 x = ffma2(make_float2(__uint_as_float(sv[k][2 * q2]), __uint_as_float(sv[k][2 * q2 + 1])), sl2, -m_use);
          float2 e;
          if (PF16 && use_poly_exp(q2)) {
            e = exp2_poly2(x);
          } else {
            e.x = fast_exp2(x.x);
            e.y = fast_exp2(x.y);
          }
          acc[q2 & 3] = fadd2(acc[q2 & 3], e);
          pk[q2] = PF16 ? pack_f16x2(e.x, e.y) : pack_bf16x2(e.x, e.y);
        }
        tmem_st16(s_tm + k * 16, pk);
      }
      const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
      l_run = l_run * f + ((a01.x + a01.y) + (a23.x + a23.y));
      if (row == 0) TRACE2(12 + 16 * wg, n);
      // rescale O_wg (own rows) after this WG's previous P.V completed, before PV_wg(n) is issued
      if (__any_sync(0xffffffffu, rescale && n > 0)) {
        mbar_wait(pv_done + wg, (n - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t o[32];
          tmem_ld32(o_tm + c0, o);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
          tmem_st16(o_tm + c0, *reinterpret_cast<uint32_t(*)[16]>(o));
          tmem_st16(o_tm + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(o + 16));
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(p_full + 2 * (n & 1) + wg, 0);
      if (row == 0) TRACE2(6 + 16 * wg, n);
    }
    // ---- epilogue: merge the two half-softmaxes, O = (O_0 a_0 + O_1 a_1) / (l_0 a_0 + l_1 a_1),
    // a_b = 2^(m_b - m); WG b normalises and stores output columns [64b, 64b+64).
    xml[wg][0][row] = m_run;
    xml[wg][1][row] = l_run;
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");  // warps q and q+4
    const float m0 = xml[0][0][row], l0 = xml[0][1][row], m1 = xml[1][0][row], l1 = xml[1][1][row];
    const float mm = fmaxf(m0, m1);
    const float a0 = l0 > 0.f ? fast_exp2(m0 - mm) : 0.f, a1 = l1 > 0.f ? fast_exp2(m1 - mm) : 0.f;
    const float lt = l0 * a0 + l1 * a1;
    const float inv = lt > 0.f ? 1.0f / lt : 0.f;
    const float c0f = a0 * inv, c1f = a1 * inv;
    const bool has0 = N > 0, has1 = N > 0;  // both accumulators are written on every page
    const bool store = p < g.C;
    if (N > 0) {
      mbar_wait(o_full, 0);
      tc_fence_after();
    }
    const uint32_t ob0 = tmem + lane_off + 256 + wg * (D / 2), ob1 = ob0 + 128;
    const long long obase =
        (long long)b * args.o_bstride + (long long)p * args.o_stride + (long long)h * D + wg * (D / 2);
#pragma unroll
    for (int cc = 0; cc < D / 2; cc += 32) {
      uint32_t o0[32], o1[32];
      if (has0) tmem_ld32(ob0 + cc, o0);
      if (has1) tmem_ld32(ob1 + cc, o1);
      tmem_wait_ld();
      float v[32];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        v[c] = (has0 ? __uint_as_float(o0[c]) * c0f : 0.f) + (has1 ? __uint_as_float(o1[c]) * c1f : 0.f);
      if (store) store_o_row32(args, obase + cc, v);
    }
  }
  tc_fence_before();
  cluster_sync();  // no CTA leaves while the pair's MMAs / remote arrivals may still touch it
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem);
  }
}

template <int BS, bool PF16>
static cudaError_t launch_2cta_t(const CUtensorMap& tq, const CUtensorMap& tk_half, const CUtensorMap& tv,
                                 const Geo& g, const AttnArgs& a, cudaStream_t st) {
  using Cfg = Attn2Cfg<BS>;
  auto kern = k_paged_attn_2cta<BS, PF16>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
  if (e != cudaSuccess) return e;
  const int nqt = (g.C + 127) / 128;
  const int clusters = nqt * g.B * g.Gn * (g.E / 2);
  kern<<<2 * clusters, Cfg::kThreads, Cfg::kSmem, st>>>(tq, tk_half, tv, g, a);
  return cudaGetLastError();
}

bool attn_2cta_supported(const Geo& g) { return g.d == 128 && (g.bs == 64 || g.bs == 128) && g.E % 2 == 0; }

cudaError_t launch_paged_attention_2cta(const CUtensorMap& tq, const CUtensorMap& tk_half, const CUtensorMap& tv,
                                        const Geo& g, const AttnArgs& a, cudaStream_t st, int* launches) {
  ++*launches;
  const bool pf16 = !(g.flags & (1u << 8));
  if (g.bs == 128) return pf16 ? launch_2cta_t<128, true>(tq, tk_half, tv, g, a, st)
                               : launch_2cta_t<128, false>(tq, tk_half, tv, g, a, st);
  if (g.bs == 64) return pf16 ? launch_2cta_t<64, true>(tq, tk_half, tv, g, a, st)
                              : launch_2cta_t<64, false>(tq, tk_half, tv, g, a, st);
  return cudaErrorInvalidValue;
}

}  // namespace cpa

#ifdef CPA_TRACE
extern "C" __attribute__((visibility("default"))) int cpa_debug_trace2(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, cpa::g_trace2, sizeof(cpa::g_trace2));
}
#endif
