// attention_ks4.cu -- §8 row a6 on a CTA pair, four key slices sharing one running max.
//
// Same math and work units as attention_2cta.cu:
//   O[b,p,h] = sum_{t in A(p)} softmax_t(scale q_p.k_t) v_t,  A(p) = {t : t/bs in T[b,h/E], t <= P+p},
// causal masking in absolute positions; unit = (b, group, 128-token q-tile, head pair), CTA r of the
// pair holds head h0+r's 128 query rows, every tcgen05.mma is M=256 issued by CTA 0, each page's keys /
// V columns are split across the pair.
//
// What differs from the key-split kernel (two warpgroups with two running maxima and two O accumulators,
// DESIGN.md §6): 16 softmax warps, four per SMSP. Warp w owns the 32 TMEM lanes (rows) 32(w%4).. and the
// key slice [32(w/4), 32(w/4)+32) of every page. The four warps of a lane quarter exchange their slice
// maxima through shared memory once per page (a 128-thread named barrier) and all use the same running
// max, so their P slices accumulate into ONE O (one P.V batch of K=128 per page) and the lazy rescale
// decision is identical in all four. That frees TMEM for a third S buffer: S^0 S^1 S^2 O = 512 columns,
// so S(n+3) is issued right after P.V(n) in one batch of 16 MMAs and the softmax of a page never waits
// for the tensor pipe. Per page the MMA warp probes two barriers: P(n) (32 warp arrivals) and the load
// barrier of page n+3, which carries K(n+3) and V(n) (the producer pairs them), so V needs no probe.
// P (fp16) of slice s is stored over the first 16 of the slice's own 32 S columns (no slice writes
// columns another slice has not read yet); the P.V MMA k-steps address those columns.
// fp16 V pool only (CPA_F_V_F16), d = 128, bs = 128, per-unit grid (no stream-K).
#include "common.cuh"
#include "geo.cuh"
#include "launch.cuh"
#include "out_store.cuh"
#include "attn_units.cuh"

namespace cpa {

struct Ks4Cfg {
  static constexpr int D = 128, BS = 128;
  static constexpr int kQBytes = 128 * D * 2;      // this CTA's Q tile
  static constexpr int kKHalf = (BS / 2) * D * 2;  // half of a K page (keys)
  static constexpr int kVHalf = BS * 64 * 2;       // half of a V page (head-dim columns)
  static constexpr int kStages = 4;                // K and V rings (load barrier m carries K(m), V(m-3))
  static constexpr int kSoftWarps = 16;
  static constexpr int kThreads = (kSoftWarps + 2) * 32;  // + TMA producer + MMA issuer
  static constexpr int kSmem = kQBytes + kStages * (kKHalf + kVHalf) + 1024 + 512;
  static_assert(kSmem + 8192 <= 232448, "shared memory budget");
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Ks4Cfg::kThreads, 1)
    k_paged_attn_ks4(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k_half,
                     const __grid_constant__ CUtensorMap tm_v, Geo g, AttnArgs args) {
  using Cfg = Ks4Cfg;
  constexpr int D = Cfg::D, BS = Cfg::BS, NS = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::kQBytes;
  uint8_t* sV = sK + NS * Cfg::kKHalf;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + NS * Cfg::kVHalf);
  uint64_t* q_full = bars;              // leader: both Q tiles landed (tx)
  uint64_t* ld_full = q_full + 1;       // leader [NS]: load m = K(m) (m < G) + V(m-3) (m >= 3) landed (tx)
  uint64_t* k_empty = ld_full + NS;     // both [NS]: K stage consumed by S (multicast commit)
  uint64_t* v_empty = k_empty + NS;     // both [NS]: V stage consumed by P.V (multicast commit)
  uint64_t* s_full = v_empty + NS;      // both [3]: S^b computed (multicast commit)
  uint64_t* p_full = s_full + 3;        // leader [3]: P^b written by all 16 softmax warps of both CTAs
  // both [3]: P.V(n) accumulated into O, ring by n % 3: when a softmax warp at page n waits for P.V(n-1),
  // S(n) has landed, so every MMA before S(n) (P.V(n-3), hence P.V(n-4)) is complete and the barrier of
  // P.V(n-1) is at most one phase behind (a single barrier could be two behind: P.V(n-2) follows S(n))
  uint64_t* pv_done = p_full + 3;
  uint64_t* o_full = pv_done + 3;       // both: every MMA of the unit complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);
  int* unit_s = reinterpret_cast<int*>(tmem_slot + 1);  // {start, n, nd}
  __shared__ float xm[2][4][128];  // [page parity][key slice][row]: slice maxima for the shared max
  __shared__ float xl[4][128];     // [key slice][row]: slice row sums for the epilogue

  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
  const int cl = (int)blockIdx.x >> 1;
  const uint32_t warp = warp_id(), lane = lane_id();
  constexpr uint32_t kTmaWarp = 16, kMmaWarp = 17;
  const Unit uc = unit_coords(g, cl);
  const int kvh = group_kv_head(g, uc.grp);

  if (warp == kTmaWarp) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k_half);
      tma_prefetch_desc(&tm_v);
      mbar_init(q_full, 1);
      for (int s = 0; s < NS; ++s) {
        mbar_init(ld_full + s, 1);
        mbar_init(k_empty + s, 1);
        mbar_init(v_empty + s, 1);
      }
      for (int b = 0; b < 3; ++b) {
        mbar_init(s_full + b, 1);
        mbar_init(p_full + b, 2 * Cfg::kSoftWarps);
        mbar_init(pv_done + b, 1);
      }
      mbar_init(o_full, 1);
      fence_barrier_init();
    }
    __syncwarp();
    pdl_wait();  // tables complete
    int s, n, nd;
    unit_table_warp(g, args, cl, &s, &n, &nd);
    if (lane == 0) { unit_s[0] = s; unit_s[1] = n; unit_s[2] = nd; }
  }
  if (warp == kMmaWarp) tmem_alloc2<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  pdl_wait();
  const uint32_t tmem = *tmem_slot;
  const int st = unit_s[0], G = unit_s[1], nd = unit_s[2];

  if (warp == kTmaWarp) {  // ------------------------------------------------------------ TMA producer
    if (G > 0) {
      const int h = uc.grp * g.E + uc.hp * 2 + (int)cta;
      if (elect_one()) {
        if (leader) mbar_expect_tx(q_full, 2 * Cfg::kQBytes);
        tma_load_4d_2sm(sQ, &tm_q, q_full, 0, h, uc.qt * 128, uc.b);
        tma_load_4d_2sm(sQ + 128 * 128, &tm_q, q_full, 64, h, uc.qt * 128, uc.b);
      }
      __syncwarp();
      const int32_t* ptab = args.page_table + (long long)uc.b * g.maxb;
      auto page_of = [&](int t) {
        const int j = args.indptr != nullptr ? __ldg(args.indices + st + t) : t;
        return __ldg(ptab + j);
      };
      // load m: K(m) if m < G, V(m-3) if m >= 3, both completing on ld_full[m % NS]
      for (int m = 0; m < G + 3; ++m) {
        const int ls = m % NS;
        const bool hasK = m < G, hasV = m >= 3;
        if (hasK) mbar_wait(k_empty + ls, ((m / NS) & 1) ^ 1);
        if (hasV) mbar_wait(v_empty + (m - 3) % NS, (((m - 3) / NS) & 1) ^ 1);
        const int pk = hasK ? page_of(m) : 0, pv = hasV ? page_of(m - 3) : 0;
        if (elect_one()) {
          if (leader) mbar_expect_tx(ld_full + ls, (hasK ? 2 * Cfg::kKHalf : 0) + (hasV ? 2 * Cfg::kVHalf : 0));
          if (hasK) {
            uint8_t* dst = sK + ls * Cfg::kKHalf;
            tma_load_4d_2sm(dst, &tm_k_half, ld_full + ls, 0, (int)cta * (BS / 2), kvh, pk);
            tma_load_4d_2sm(dst + (BS / 2) * 128, &tm_k_half, ld_full + ls, 64, (int)cta * (BS / 2), kvh, pk);
          }
          if (hasV)
            tma_load_4d_2sm(sV + ((m - 3) % NS) * Cfg::kVHalf, &tm_v, ld_full + ls, 64 * (int)cta, 0, kvh, pv);
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    if (leader && G > 0) {  // ---------------------------------------------------- MMA issuer (CTA 0)
      constexpr uint32_t idesc_s = umma_idesc_bf16(256, BS, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(256, D, 0, 1) & ~((7u << 7) | (7u << 10));  // fp16 P, V
      const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
      auto wait_ld = [&](int m) {
        mbar_wait(ld_full + m % NS, (m / NS) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int n) {  // S^{n%3} = Q K_n^T, M=256, N=BS, K=d
        const uint32_t d_tm = tmem + (n % 3) * 128;
        const uint32_t kb = k_base + (n % NS) * Cfg::kKHalf;
        if (elect_one()) {
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ad = umma_desc_sw128(q_base + a * 128 * 128 + kk * 32, 16, 1024);
              const uint64_t bd = umma_desc_sw128(kb + a * (BS / 2) * 128 + kk * 32, 16, 1024);
              mma2_ss(d_tm, ad, bd, idesc_s, (a | kk) != 0);
            }
          tc_commit2(s_full + n % 3);
          tc_commit2(k_empty + n % NS);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int n) {  // O += P_n V_n, M=256, N=d, K=BS; slice s's P in columns [32s, 32s+16)
        const uint32_t p_tm = tmem + (n % 3) * 128;
        const uint32_t vb = v_base + (n % NS) * Cfg::kVHalf;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BS / 16; ++kk) {
            const uint64_t bd = umma_desc_sw128(vb + kk * 16 * 128, BS * 128, 1024);
            mma2_ts(tmem + 384, p_tm + 32 * (kk >> 1) + 8 * (kk & 1), bd, idesc_o, (n > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit2(pv_done + n % 3);
          tc_commit2(v_empty + n % NS);
          if (n == G - 1) tc_commit2(o_full);
        }
        __syncwarp();
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int n = 0; n < 3 && n < G; ++n) {
        wait_ld(n);
        issue_s(n);
      }
      for (int n = 0; n < G; ++n) {
        mbar_wait(p_full + n % 3, (n / 3) & 1);
        wait_ld(n + 3);  // V(n) (and K(n+3) when n+3 < G)
        issue_pv(n);
        if (n + 3 < G) issue_s(n + 3);
      }
    }
  } else {  // ------------------------------------------------------------------ softmax / epilogue
    const int quarter = warp & 3, slice = warp >> 2;
    const int row = quarter * 32 + lane;
    const float sl2 = g.scale * 1.4426950408889634f;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t o_tm = tmem + lane_off + 384 + slice * 32;  // this warp's 32 O columns (rescale, epilogue)
    const int p = uc.qt * 128 + row;
    const int lim = min(g.P + p, g.L - 1);
    const uint32_t bar_id = 1 + quarter;
    float m_run = -INFINITY, l_run = 0.f;
    for (int n = 0; n < G; ++n) {
      const uint32_t s_tm = tmem + lane_off + (n % 3) * 128 + slice * 32;
      mbar_wait(s_full + n % 3, (n / 3) & 1);
      tc_fence_after();
      uint32_t sv[32];
      tmem_ld32(s_tm, sv);
      tmem_wait_ld();
      if (n >= nd) {  // block crosses the tile's causal diagonal: mask in absolute positions
        const int j = args.indptr != nullptr ? __ldg(args.indices + st + n) : n;
        const int tbase = j * g.bs + slice * 32;
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (tbase + c > lim) sv[c] = __float_as_uint(-INFINITY);
      }
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 32; c += 8)
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) m4[w4] = fmax3(m4[w4], __uint_as_float(sv[c + 2 * w4]), __uint_as_float(sv[c + 2 * w4 + 1]));
      // the quarter's four slice maxima -> the page max of this row (identical in all four warps)
      xm[n & 1][slice][row] = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
      const float m_blk =
          fmaxf(fmaxf(xm[n & 1][0][row], xm[n & 1][1][row]), fmaxf(xm[n & 1][2][row], xm[n & 1][3][row])) * sl2;
      float f = 1.f;
#ifndef CPA_RESCALE_THRESH
#define CPA_RESCALE_THRESH 8.0f
#endif
      const bool rescale = m_blk > m_run + CPA_RESCALE_THRESH;  // lazy rescale (first block always lands here)
      if (rescale) {
        if (m_run != -INFINITY) f = fast_exp2(m_run - m_blk);
        m_run = m_blk;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      // P = exp2(s*sl2 - m): packed FFMA2, 1/4 of the pairs on the FMA-pipe polynomial, fp16 pack
      float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
      uint32_t pk[16];
#pragma unroll
      for (int q2 = 0; q2 < 16; ++q2) {
        const float2 x = ffma2(make_float2(__uint_as_float(sv[2 * q2]), __uint_as_float(sv[2 * q2 + 1])), sl2, -m_use);
        float2 e;
        if (use_poly_exp(q2)) {
          e = exp2_poly2(x);
        } else {
          e.x = fast_exp2(x.x);
          e.y = fast_exp2(x.y);
        }
        acc[q2 & 3] = fadd2(acc[q2 & 3], e);
        pk[q2] = pack_f16x2(e.x, e.y);
      }
      tmem_st16(s_tm, pk);  // over this slice's first 16 S columns (only this warp reads them)
      const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
      l_run = l_run * f + ((a01.x + a01.y) + (a23.x + a23.y));
      // rescale this warp's 32 O columns of its rows after P.V(n-1), before P.V(n) (all four warps of the
      // quarter take the same decision, so every column of a rescaled row is scaled once)
      if (__any_sync(0xffffffffu, rescale && n > 0)) {
        mbar_wait(pv_done + (n - 1) % 3, ((n - 1) / 3) & 1);
        tc_fence_after();
        uint32_t o[32];
        tmem_ld32(o_tm, o);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
        tmem_st16(o_tm, *reinterpret_cast<uint32_t(*)[16]>(o));
        tmem_st16(o_tm + 16, *reinterpret_cast<uint32_t(*)[16]>(o + 16));
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(p_full + n % 3, 0);
    }
    // ---- epilogue: l = sum of the four slice sums (same running max), O / l, warp stores its 32 columns
    xl[slice][row] = l_run;
    asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
    const float lt = (xl[0][row] + xl[1][row]) + (xl[2][row] + xl[3][row]);
    const float inv = lt > 0.f ? 1.0f / lt : 0.f;
    if (G > 0) {
      mbar_wait(o_full, 0);
      tc_fence_after();
    }
    uint32_t o[32];
    tmem_ld32(o_tm, o);  // warp-collective: every lane, valid row or not
    tmem_wait_ld();
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = G > 0 ? __uint_as_float(o[c]) * inv : 0.f;
    const int h = uc.grp * g.E + uc.hp * 2 + (int)cta;
    if (p < g.C)
      store_o_row32(args, (long long)uc.b * args.o_bstride + (long long)p * args.o_stride + (long long)h * D + slice * 32, v);
  }
  tc_fence_before();
  cluster_sync();  // no CTA leaves while the pair's MMAs / remote arrivals may still touch it
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem);
  }
}

bool attn_ks4_supported(const Geo& g) {
  return g.d == 128 && g.bs == 128 && g.E % 2 == 0 && (g.flags & (1u << 12)) != 0;  // CPA_F_V_F16
}

cudaError_t launch_paged_attention_ks4(const CUtensorMap& tq, const CUtensorMap& tk_half, const CUtensorMap& tv,
                                       const Geo& g, const AttnArgs& a, cudaStream_t st, int* launches) {
  cudaError_t e;
  const int units = (g.C + 127) / 128 * g.B * g.Gn * (g.E / 2);
  if ((e = cudaFuncSetAttribute(k_paged_attn_ks4, cudaFuncAttributeMaxDynamicSharedMemorySize, Ks4Cfg::kSmem)) !=
      cudaSuccess)
    return e;
  ++*launches;
  return launch_ex(k_paged_attn_ks4, dim3(2 * units), dim3(Ks4Cfg::kThreads), Ks4Cfg::kSmem, st, use_pdl(g), tq,
                   tk_half, tv, g, a);
}

}  // namespace cpa
