// attention_2cta.cu -- §8 row a6 on a CTA pair: zero-copy paged attention with cta_group::2 MMAs.
//
// Same math as attention.cu:
//   O[b,p,h] = sum_{t in A(p)} softmax_t(scale q_p.k_t) v_t,  A(p) = {t : t/bs in T[b,h/E], t <= P+p}
// with causal masking in absolute positions.
//
// Work unit u = (b, group g, 128-token q-tile, head pair {h0, h0+1} of g) over the unit's visible
// table prefix (N_u pages). CTA r of the pair holds the 128 query rows of head h0+r; every
// tcgen05.mma is M=256 (both CTAs' rows) and issued by CTA 0. Each page is split across the pair:
// CTA r loads keys [r*bs/2, (r+1)*bs/2) of K and head-dim columns [64r, 64r+64) of V, so per SM the
// tensor core reads 6 KB of shared memory per 64-cycle S MMA (96 B/clk, under the 128 B/clk limit
// that caps a 1-CTA 128x128 SS MMA) and the TMA / L2 traffic per FLOP halves. P (fp16) aliases S^b;
// the MMA computes S(n+1) while the softmax of S(n) runs. Both softmax warpgroups work on every page:
// WG w owns key columns [w BS/2, (w+1) BS/2) of each S^b and keeps its own running max / sum and
// accumulator O_w (P.V of its half of the keys); the epilogue merges (m_w, l_w, O_w).
//
// Scheduling. Non-persistent (sched == nullptr): one cluster per unit, heaviest q-tile first within
// an execution group (group-major, so the clusters in flight share few groups' KV pages in L2).
// Persistent stream-K (sched != nullptr, see k_sk_schedule): one cluster per co-resident SM pair;
// the concatenated page lists of all units (same order) are cut into equal contiguous ranges, so
// every cluster gets the same number of pages whatever the unit count (no wave quantisation: e.g.
// 64 units on 74 SM pairs at one KV group per GPU). A cluster walks its items (unit, page range);
// the K/V / S / P pipelines run continuously across items, Q is double-buffered; a unit cut by a
// range boundary is written as unnormalised partials (O, m, l) and merged by k_sk_fixup.
// TMEM per CTA: S^0 [0,128) S^1 [128,256) O_0 [256,384) O_1 [384,512).
// Warps: 0-7 softmax (WG = warp/4, lane quarter = warp%4), 8-9 V bf16->fp16 converters,
// 10 TMA producer, 11 TMEM alloc + MMA issuer.
#include "common.cuh"
#include "geo.cuh"
#include "launch.cuh"
#include "out_store.cuh"
#include "attn_units.cuh"

namespace cpa {

#ifdef CPA_TRACE
__device__ long long g_trace2[32][2048];
#define TRACE2(e, i) \
  do { if (blockIdx.x == 0 && (i) < 2048) g_trace2[e][i] = clock64(); } while (0)
#else
#define TRACE2(e, i) do {} while (0)
#endif

template <int BS, bool PERSIST = false>
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
  static constexpr int kQBufs = PERSIST ? 2 : 1;  // persistent: next item's Q prefetched
  static constexpr int kSmem = kQBufs * kQBytes + kKStages * kKHalf + kVStages * kVHalf + 1024 + 512;
  static_assert(kSmem + 2048 <= 232448, "shared memory budget");
};

// Page range [lo, hi) of persistent cluster c in segment s (a segment = the units of one (b, group)
// row; every cluster takes the c-th equal share of every segment, segment after segment, so all
// clusters read the same group's KV pages at the same time, as in the per-unit grid).
__device__ __forceinline__ void sk_range(const SkSched& sk, int c, int s, int* lo, int* hi) {
  const int b0 = sk.pre[s * sk.seg_units], b1 = sk.pre[(s + 1) * sk.seg_units];
  const long long T = b1 - b0;
  *lo = b0 + (int)(T * c / sk.clusters);
  *hi = b0 + (int)(T * (c + 1) / sk.clusters);
}
// Unit containing global page x (last u with pre[u] <= x).
__device__ __forceinline__ int sk_unit_of(const SkSched& sk, int x) {
  int lo = 0, hi = sk.units;  // first u with pre[u] > x, minus one
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sk.pre[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

// Stream-K schedule (one CTA): per unit its table start / length / fully-visible prefix, and the
// exclusive prefix sum of the lengths (sched->pre[U] = total pages).
__global__ void __launch_bounds__(1024) k_sk_schedule(Geo g, AttnArgs args, SkSched sk) {
  __shared__ int part[1024];
  const int U = sk.units, tid = threadIdx.x;
  const int per = (U + 1023) / 1024;
  const int u0 = min(U, tid * per), u1 = min(U, u0 + per);
  int sum = 0;
  for (int u = u0; u < u1; ++u) {
    int s, n, nd;
    unit_table(g, args, u, &s, &n, &nd);
    sk.start[u] = s;
    sk.len[u] = n;
    sk.nd[u] = nd;
    sum += n;
  }
  part[tid] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele scan of the per-thread sums
    const int v = tid >= off ? part[tid - off] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int run = part[tid] - sum;
  for (int u = u0; u < u1; ++u) {
    sk.pre[u] = run;
    run += sk.len[u];
  }
  if (tid == 1023) sk.pre[U] = part[1023];
  __syncthreads();
  // fixup part lists, one share (c, s) per thread: the share that holds a unit's FIRST page and not
  // its last owns the merge; its parts are its own item of that unit (slot 0 if it is the share's
  // first item, else 1) and the first item (slot 0) of every later non-empty share up to the one
  // holding the unit's last page
  for (int cs = tid; cs < sk.clusters * sk.segments; cs += 1024) {
    const int c = cs % sk.clusters, sg = cs / sk.clusters;
    int* fx = sk.fix + (long long)cs * kSkFixStride;
    fx[0] = 0;
    int lo, hi;
    sk_range(sk, c, sg, &lo, &hi);
    if (lo >= hi) continue;
    const int u = sk_unit_of(sk, hi - 1);
    const int base = sk.pre[u], len = sk.len[u];
    if (base < lo || base + len <= hi) continue;
    int n = 0;
    fx[2 + n++] = (c * sk.segments + sg) * 2 + (sk_unit_of(sk, lo) == u ? 0 : 1);
    const int x = base + len - 1;
    for (int cc = c + 1; cc < sk.clusters && n < kSkFixStride - 2; ++cc) {
      int l2, h2;
      sk_range(sk, cc, sg, &l2, &h2);
      if (l2 > x) break;
      if (l2 < h2) fx[2 + n++] = (cc * sk.segments + sg) * 2;
    }
    fx[1] = u;
    fx[0] = n;
  }
}

// Walks the items (unit, page range [a, e) of the unit's list) of one cluster, in order. Every role
// of the cluster runs its own cursor over the same deterministic sequence. Non-persistent: the one
// item of the prologue (whole unit); persistent: the units overlapping the cluster's page range.
template <bool PERSIST>
struct ItemCursor {
  int idx, u, a, e, start, nd, len;
  int cur, hi, seg, c;
  bool valid, first_in_seg;
  __device__ __forceinline__ void load(const SkSched& sk) {  // unit u, from page cur (next segments if done)
    for (;;) {
      if (cur >= hi) {
        if (++seg >= sk.segments) break;
        sk_range(sk, c, seg, &cur, &hi);
        u = sk_unit_of(sk, cur);
        first_in_seg = true;
        continue;
      }
      const int base = sk.pre[u];
      len = sk.len[u];
      a = cur - base;
      e = min(hi - base, len);
      if (e > a) {
        start = sk.start[u];
        nd = sk.nd[u];
        valid = true;
        return;
      }
      cur = base + len;
      ++u;
    }
    valid = false;
  }
  __device__ __forceinline__ void init(const SkSched& sk, int c, const int* single) {
    idx = 0;
    if constexpr (!PERSIST) {  // single[] = {unit, start, n, nd}
      u = single[0]; start = single[1]; len = single[2]; nd = single[3];
      a = 0; e = len; valid = len > 0; cur = hi = 0;
      return;
    } else {
    this->c = c;
    seg = 0;
    sk_range(sk, c, 0, &cur, &hi);
    u = sk_unit_of(sk, cur);
    first_in_seg = true;
    load(sk);
    }
  }
  __device__ __forceinline__ void next(const SkSched& sk) {
    ++idx;
    if constexpr (!PERSIST) { valid = false; return; }
    cur = sk.pre[u] + e;
    ++u;
    first_in_seg = false;
    load(sk);
  }
  // partial-output slot of the current item (only a segment range's first / last item can be cut)
  __device__ __forceinline__ int slot(const SkSched& sk) const {
    return (c * sk.segments + seg) * 2 + (first_in_seg ? 0 : 1);
  }
};

template <int BS, bool PF16, bool PERSIST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    k_paged_attn_2cta(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k_half,
                      const __grid_constant__ CUtensorMap tm_v, Geo g, AttnArgs args, SkSched sk) {
  using Cfg = Attn2Cfg<BS, PERSIST>;
  using Cursor = ItemCursor<PERSIST>;
  constexpr int D = Cfg::D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                   // [2] Q buffers (item parity)
  uint8_t* sK = sQ + Cfg::kQBufs * Cfg::kQBytes;
  uint8_t* sV = sK + Cfg::kKStages * Cfg::kKHalf;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + Cfg::kVStages * Cfg::kVHalf);
  uint64_t* q_full = bars;                          // leader [2]: both Q tiles of buffer q landed (tx)
  uint64_t* q_empty = q_full + 2;                   // both [2]: last S of the buffer's item done (multicast)
  uint64_t* k_full = q_empty + 2;                   // leader: both K halves landed (tx)
  uint64_t* k_empty = k_full + Cfg::kKStages;       // both: K stage consumed (multicast commit)
  uint64_t* v_full = k_empty + Cfg::kKStages;       // local: own V half landed (tx)
  uint64_t* v_empty = v_full + Cfg::kVStages;       // both: V stage consumed (multicast commit)
  uint64_t* v_ready = v_empty + Cfg::kVStages;      // leader: both V halves converted (4 arrivals)
  uint64_t* s_full = v_ready + Cfg::kVStages;       // both [2]: S^b computed (multicast commit)
  uint64_t* p_full = s_full + 2;                    // leader [2][2]: P^b columns of WG w written
  uint64_t* pv_done = p_full + 4;                   // both [2]: last P.V into O_w complete
  uint64_t* o_full = pv_done + 2;                   // both: every MMA of the item complete
  uint64_t* o_empty = o_full + 1;                   // leader: epilogue read O (16 warp arrivals)
  uint64_t* stag = o_empty + 1;                     // local [4][2]: WG0 quarter q done with page's max
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stag + 8);
  int* total_s = reinterpret_cast<int*>(tmem_slot + 1);
  int* single_s = total_s + 1;  // non-persistent unit: {unit, start, n, nd}

  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
  const int cl = (int)blockIdx.x >> 1;
  const uint32_t warp = warp_id(), lane = lane_id();
  constexpr uint32_t kConvWarp0 = 8, kTmaWarp = 10, kMmaWarp = 11;
  const bool vf16 = PF16 && (g.flags & (1u << 12)) != 0;  // CPA_F_V_F16: V pages already fp16
  // fp16 V pool: K and V of a page complete on ONE barrier (k_full), so the MMA warp probes once per page
  // for its operands (before S(n); P.V(n) is issued after S(n)) instead of twice. A probe costs ~90 cycles
  // even on a completed phase; measured neutral at 128K (the binding chain is the lagging softmax
  // warpgroup), kept for the shorter MMA-warp loop.
#ifndef CPA_NO_KV_BAR
  const bool kvbar = vf16 && Cfg::kKStages == Cfg::kVStages;
#else
  const bool kvbar = false;
#endif

  if (warp == kTmaWarp) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k_half);
      tma_prefetch_desc(&tm_v);
      for (int i = 0; i < 2; ++i) { mbar_init(q_full + i, 1); mbar_init(q_empty + i, 1); }
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
      mbar_init(o_empty, 16);  // 8 softmax warps x 2 CTAs
      for (int i = 0; i < 8; ++i) mbar_init(stag + i, 1);
      fence_barrier_init();
    }
    __syncwarp();
    if constexpr (PERSIST) pdl_wait();  // tables complete; the other threads wait at the cluster barrier below
    if constexpr (PERSIST) {
      if (lane == 0) {  // stream-K: share cl of every segment
      int total = 0;
      for (int s = 0; s < sk.segments; ++s) {
        int lo, hi;
        sk_range(sk, cl, s, &lo, &hi);
        total += hi - lo;
      }
      *total_s = total;
      }
    }
  }
  if (warp == kMmaWarp) tmem_alloc2<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // peer barriers initialised, TMEM allocated in both CTAs
  tc_fence_after();
  if constexpr (!PERSIST) {
    // one cluster = one whole unit. Its Q tile does not depend on the predecessor kernels (only the
    // tables do), so it is requested before the PDL wait and the table lookup, overlapping their latency
    if (warp == kTmaWarp) {
      const Unit uc = unit_coords(g, cl);
      if (elect_one()) {
        if (leader) mbar_expect_tx(q_full, 2 * Cfg::kQBytes);
        const int h = uc.grp * g.E + uc.hp * 2 + (int)cta;
        tma_load_4d_2sm(sQ, &tm_q, q_full, 0, h, uc.qt * 128, uc.b);
        tma_load_4d_2sm(sQ + 128 * 128, &tm_q, q_full, 64, h, uc.qt * 128, uc.b);
      }
      __syncwarp();
      pdl_wait();  // tables complete
      int s, n, nd;
      unit_table_warp(g, args, cl, &s, &n, &nd);  // the unit's visible table prefix (whole warp)
      if (lane == 0) {
        single_s[0] = cl; single_s[1] = s; single_s[2] = n; single_s[3] = nd;
        *total_s = n;
      }
      // an empty unit: its Q tile must land before the CTA may exit
      if (n == 0 && leader) mbar_wait(q_full, 0);
    }
    __syncthreads();  // single_s / total_s published to the CTA
  }
  pdl_wait();  // (PDL) every thread: the predecessor's writes (tables) are visible before any access
  const uint32_t tmem = *tmem_slot;
  const int G = *total_s;  // pages this cluster processes (all items)

  if (warp == kTmaWarp) {
    if (G > 0) {  // ------------------------------------------------------------ TMA producer
      int n = 0;
      Cursor it;
      for (it.init(sk, cl, single_s); it.valid; it.next(sk)) {
        const int i = it.idx;
        const Unit uc = unit_coords(g, it.u);
        const int h = uc.grp * g.E + uc.hp * 2 + (int)cta;
        const int kvh = group_kv_head(g, uc.grp);
        const int qb = PERSIST ? (i & 1) : 0;
        if constexpr (PERSIST) {  // (per-unit grid: requested in the prologue)
          mbar_wait(q_empty + qb, ((i >> 1) & 1) ^ 1);
          if (elect_one()) {
            if (leader) mbar_expect_tx(q_full + qb, 2 * Cfg::kQBytes);
            uint8_t* dq = sQ + qb * Cfg::kQBytes;
            tma_load_4d_2sm(dq, &tm_q, q_full + qb, 0, h, uc.qt * 128, uc.b);
            tma_load_4d_2sm(dq + 128 * 128, &tm_q, q_full + qb, 64, h, uc.qt * 128, uc.b);
          }
          __syncwarp();
        }
        const int32_t* ptab = args.page_table + (long long)uc.b * g.maxb;
        const int st = it.start;
        for (int t = it.a; t < it.e; ++t, ++n) {
          const int j = args.indptr != nullptr ? __ldg(args.indices + st + t) : t;
          const int page = __ldg(ptab + j);
          const int ks = n % Cfg::kKStages, vs = n % Cfg::kVStages;
          mbar_wait(k_empty + ks, ((n / Cfg::kKStages) & 1) ^ 1);
          if (elect_one()) {
            if (leader) mbar_expect_tx(k_full + ks, 2 * Cfg::kKHalf + (kvbar ? 2 * Cfg::kVHalf : 0));
            uint8_t* dst = sK + ks * Cfg::kKHalf;
            tma_load_4d_2sm(dst, &tm_k_half, k_full + ks, 0, (int)cta * (BS / 2), kvh, page);
            tma_load_4d_2sm(dst + (BS / 2) * 128, &tm_k_half, k_full + ks, 64, (int)cta * (BS / 2), kvh, page);
          }
          __syncwarp();
          mbar_wait(v_empty + vs, ((n / Cfg::kVStages) & 1) ^ 1);
          if (elect_one()) {
            if (kvbar) {  // fp16 pool, merged barrier: both V halves complete on the page's K barrier
              tma_load_4d_2sm(sV + vs * Cfg::kVHalf, &tm_v, k_full + ks, 64 * (int)cta, 0, kvh, page);
            } else if (vf16) {  // fp16 pool: both halves signal the leader's v_full directly (no conversion relay)
              if (leader) mbar_expect_tx(v_full + vs, 2 * Cfg::kVHalf);
              tma_load_4d_2sm(sV + vs * Cfg::kVHalf, &tm_v, v_full + vs, 64 * (int)cta, 0, kvh, page);
            } else {
              mbar_expect_tx(v_full + vs, Cfg::kVHalf);
              tma_load_4d(sV + vs * Cfg::kVHalf, &tm_v, v_full + vs, 64 * (int)cta, 0, kvh, page);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == kMmaWarp) {
    if (leader && G > 0) {  // ---------------------------------------------------- MMA issuer (CTA 0)
      constexpr uint32_t idesc_s = umma_idesc_bf16(256, BS, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(256, D, 0, 1) & ~(PF16 ? ((7u << 7) | (7u << 10)) : 0u);
      const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
      // item cursor of the S issue (runs 2 pages ahead of the P.V issue)
      Cursor si;
      si.init(sk, cl, single_s);
      int s_left = si.e - si.a;
      auto issue_s = [&](int n) {  // S^{n%2} = Q_item K_n^T, M=256 (both CTAs' rows), N=BS, K=d
        const int s_item = si.idx;
        const bool first = s_left == si.e - si.a;
        if (first) {
          mbar_wait(q_full + (PERSIST ? (s_item & 1) : 0), PERSIST ? ((s_item >> 1) & 1) : 0);
          tc_fence_after();
        }
        const uint32_t qb = q_base + (PERSIST ? (s_item & 1) : 0) * Cfg::kQBytes;
        const uint32_t d_tm = tmem + (n & 1) * 128;
        const uint32_t kb = k_base + (n % Cfg::kKStages) * Cfg::kKHalf;
        const bool last = s_left == 1;
        if (elect_one()) {
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ad = umma_desc_sw128(qb + a * 128 * 128 + kk * 32, 16, 1024);
              const uint64_t bd = umma_desc_sw128(kb + a * (BS / 2) * 128 + kk * 32, 16, 1024);
              mma2_ss(d_tm, ad, bd, idesc_s, (a | kk) != 0);
            }
          tc_commit2(s_full + (n & 1));
          tc_commit2(k_empty + n % Cfg::kKStages);
          if (PERSIST && last) tc_commit2(q_empty + (s_item & 1));
        }
        __syncwarp();
        if (last) {
          si.next(sk);
          if (si.valid) s_left = si.e - si.a;
        } else {
          --s_left;
        }
      };
      // O_w += P_w V_n[w-half keys]: WG w's P (keys [w BS/2, (w+1) BS/2) of page n, fp16 packed over its
      // S^b columns) times those V rows; M=256, N=d (64 cols per CTA), K=BS/2
      // commits == false: the caller commits later (P.V(n,1) -> S(n+2) back to back, commits after)
      auto issue_pv = [&](int n, int w, bool first, bool last, bool commits = true) {
        const uint32_t p_tm = tmem + (n & 1) * 128 + w * (BS / 2);
        const uint32_t o_tm = tmem + 256 + w * 128;
        const uint32_t vb = v_base + (n % Cfg::kVStages) * Cfg::kVHalf + w * (BS / 2) * 128;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BS / 32; ++kk) {
            const uint64_t bd = umma_desc_sw128(vb + kk * 16 * 128, BS * 128, 1024);
            mma2_ts(o_tm, p_tm + kk * 8, bd, idesc_o, (!first || kk > 0) ? 1u : 0u);
          }
          if (commits) {
            tc_commit2(pv_done + w);
            if (w == 1) {
              tc_commit2(v_empty + n % Cfg::kVStages);
              if (last) tc_commit2(o_full);
            }
          }
        }
        __syncwarp();
      };
      auto pv1_commits = [&](int n, bool last) {
        if (elect_one()) {
          tc_commit2(pv_done + 1);
          tc_commit2(v_empty + n % Cfg::kVStages);
          if (last) tc_commit2(o_full);
        }
        __syncwarp();
      };
      auto wait_k = [&](int n) {
        mbar_wait(k_full + n % Cfg::kKStages, (n / Cfg::kKStages) & 1);
        tc_fence_after();
      };
      for (int n = 0; n < 2 && n < G; ++n) {
        wait_k(n);
        issue_s(n);
      }
      int n = 0;
      Cursor it;
      for (it.init(sk, cl, single_s); it.valid; it.next(sk)) {
        const int i = it.idx;
        for (int t = it.a; t < it.e; ++t, ++n) {
          const bool first = t == it.a, last = t + 1 == it.e;
          if (PERSIST && first && i > 0) mbar_wait(o_empty, (i - 1) & 1);  // previous item's O read out of TMEM
          // V(n): with the merged K+V barrier it landed before S(n) was issued (no wait here)
          if (!kvbar) mbar_wait((vf16 ? v_full : v_ready) + n % Cfg::kVStages, (n / Cfg::kVStages) & 1);
          if (lane == 0) TRACE2(1, n);
          mbar_wait(p_full + 2 * (n & 1), (n >> 1) & 1);
          if (lane == 0) TRACE2(2, n);
          tc_fence_after();
          issue_pv(n, 0, first, last);
#ifndef CPA_NO_MMA_REORDER
          if constexpr (!PERSIST) {
          // the loop's critical latency is P(n, WG1) -> P.V(n,1) -> S(n+2) -> WG0's page n+2: wait for
          // K(n+2) before P(n,1), issue P.V(n,1) and S(n+2) back to back, commit P.V(n,1)'s barriers after
          // (per-unit grid only: in the persistent grid this order broke parity)
          const bool more = n + 2 < G;
          if (more) wait_k(n + 2);
          mbar_wait(p_full + 2 * (n & 1) + 1, (n >> 1) & 1);
          tc_fence_after();
          issue_pv(n, 1, first, last, false);
          if (lane == 0) TRACE2(9, n);
          if (more) issue_s(n + 2);
          pv1_commits(n, last);
          } else {
          mbar_wait(p_full + 2 * (n & 1) + 1, (n >> 1) & 1);
          tc_fence_after();
          issue_pv(n, 1, first, last);
          if (lane == 0) TRACE2(9, n);
          if (n + 2 < G) {
            wait_k(n + 2);
            if (lane == 0) TRACE2(10, n);
            issue_s(n + 2);
          }
          }
#else
          mbar_wait(p_full + 2 * (n & 1) + 1, (n >> 1) & 1);
          tc_fence_after();
          issue_pv(n, 1, first, last);
          if (lane == 0) TRACE2(9, n);
          if (n + 2 < G) {
            wait_k(n + 2);
            if (lane == 0) TRACE2(10, n);
            issue_s(n + 2);
          }
#endif
          if (lane == 0) TRACE2(3, n);
        }
      }
    }
  } else if (warp >= kConvWarp0) {  // --------------------------------------- V bf16 -> fp16
    const int ct = (warp - kConvWarp0) * 32 + lane;
#ifdef CPA_TRACE
    // trace builds, fp16 pool: the idle converter warps observe the tensor-pipe completions of cluster 0
    // (S(n) landed; P.V(n,0) done; P.V(n,1) + S(n+2) done; K(n) landed) for tools/attn_trace2.py
    if (vf16 && !PERSIST && blockIdx.x == 0 && lane == 0) {
      for (int n = 0; n < G; ++n) {
        if (warp == kConvWarp0) {
          mbar_wait(s_full + (n & 1), (n >> 1) & 1);
          TRACE2(14, n);
          mbar_wait(pv_done, n & 1);
          TRACE2(15, n);
        } else {
          mbar_wait(k_full + n % Cfg::kKStages, (n / Cfg::kKStages) & 1);
          TRACE2(31, n);
          mbar_wait(pv_done + 1, n & 1);
          TRACE2(30, n);
        }
      }
    }
#endif
    for (int n = 0; n < (vf16 ? 0 : G); ++n) {  // fp16 pool: nothing to convert or relay
      const int vs = n % Cfg::kVStages;
      mbar_wait(v_full + vs, (n / Cfg::kVStages) & 1);
      if (ct == 0) TRACE2(7, n);
#ifndef CPA_EXP_NO_CONV
      if (PF16 && !(g.flags & (1u << 12))) {  // CPA_F_V_F16: the pool already holds fp16 V
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
    const float sl2 = g.scale * 1.4426950408889634f;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    constexpr int HC = BS / 2;                                // key columns of a page per WG
    const uint32_t s_tm0 = tmem + lane_off + wg * HC;         // WG's columns of S^0 (this row's lanes)
    const uint32_t o_tm = tmem + lane_off + 256 + wg * 128;  // O_wg
    int n = 0;
    Cursor it;
    for (it.init(sk, cl, single_s); it.valid; it.next(sk)) {
      const int i = it.idx;
      const Unit uc = unit_coords(g, it.u);
      const int p0 = uc.qt * 128;
      const int h = uc.grp * g.E + uc.hp * 2 + (int)cta;  // this CTA's query head
      const int p = p0 + row;
      const int lim = min(g.P + p, g.L - 1);
      const int st = it.start, nd = it.nd, ta = it.a, te = it.e;
      float m_run = -INFINITY, l_run = 0.f;
      // Both WGs work on every page: WG w owns key columns [w BS/2, (w+1) BS/2) of each S^b with its
      // own running max / sum and its own accumulator O_w (no cross-WG exchange until the merge).
      for (int t = ta; t < te; ++t, ++n) {
        const uint32_t s_tm = s_tm0 + (n & 1) * 128;
        if (row == 0) TRACE2(4 + 16 * wg, n);
#ifndef CPA_NO_STAGGER
        // WG1 starts a page when WG0 (same rows, same SMSP) has finished its TMEM load + block max of
        // that page, so one warp's non-MUFU phase overlaps the other's exponentials
        if (wg == 1) mbar_wait(stag + quarter * 2 + (n & 1), (n >> 1) & 1);
        if (row == 0 && wg == 1) TRACE2(29, n);
#endif
        mbar_wait(s_full + (n & 1), (n >> 1) & 1);
        if (row == 0) TRACE2(5 + 16 * wg, n);
        tc_fence_after();
#ifdef CPA_EXP_NO_SOFTMAX  // A/B only: MMA / TMA / converter pipeline alone (wrong results)
        __syncwarp();
#ifndef CPA_NO_STAGGER
        if (wg == 0 && lane == 0) mbar_arrive(stag + quarter * 2 + (n & 1));
#endif
        if (lane == 0) mbar_arrive_cluster(p_full + 2 * (n & 1) + wg, 0);
        continue;
#endif
        uint32_t sv[HC / 32][32];
#ifndef CPA_EXP_NO_TMEM
#pragma unroll
        for (int k = 0; k < HC / 32; ++k) tmem_ld32(s_tm + k * 32, sv[k]);
        tmem_wait_ld();
#else  // A/B only (wrong results): the softmax math on register values, no TMEM traffic
#pragma unroll
        for (int k = 0; k < HC / 32; ++k)
#pragma unroll
          for (int c = 0; c < 32; ++c) sv[k][c] = __float_as_uint((float)((lane + c + n) & 7));
#endif
        if (t >= nd) {  // block crosses the causal diagonal of this tile: mask in absolute positions
          const int j = args.indptr != nullptr ? __ldg(args.indices + st + t) : t;
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
#ifndef CPA_RESCALE_THRESH
#define CPA_RESCALE_THRESH 8.0f
#endif
        const bool rescale = m_blk > m_run + CPA_RESCALE_THRESH;  // lazy rescale (first block always lands here)
        if (rescale) {
          if (m_run != -INFINITY) f = fast_exp2(m_run - m_blk);
          m_run = m_blk;
        }
        const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
        if (row == 0) TRACE2(11 + 16 * wg, n);
#ifndef CPA_NO_STAGGER
        if (wg == 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(stag + quarter * 2 + (n & 1));
          if (row == 0) TRACE2(13, n);
        }
#endif
        // P = exp2(s*sl2 - m): packed f32x2 FFMA; pairs chosen by use_poly_exp on a degree-3
        // polynomial (FMA pipe), the rest on MUFU.EX2; 4 partial f32x2 sums; fp16 pack; stored over S.
        float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
        for (int k = 0; k < HC / 32; ++k) {
          uint32_t pk[16];
#pragma unroll
          for (int q2 = 0; q2 < 16; ++q2) {
#ifdef CPA_EXP_TMEM_ONLY  // A/B only (wrong results): TMEM load + store of every page, no softmax math
            pk[q2] = sv[k][2 * q2] ^ sv[k][2 * q2 + 1];
            continue;
#endif
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
#ifndef CPA_EXP_NO_TMEM
          tmem_st16(s_tm + k * 16, pk);
#else
          if (pk[0] == 0x12345u && pk[15] == 0x6789u) tmem_st16(s_tm + k * 16, pk);  // keep the math live
#endif
        }
        const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
        l_run = l_run * f + ((a01.x + a01.y) + (a23.x + a23.y));
        if (row == 0) TRACE2(12 + 16 * wg, n);
        // rescale O_wg (own rows) after this WG's previous P.V completed, before PV_wg(n) is issued;
        // not on an item's first page (its P.V overwrites O)
        if (__any_sync(0xffffffffu, rescale && t > ta)) {
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
      // ---- item epilogue: merge the two half-softmaxes, O = (O_0 a_0 + O_1 a_1) / (l_0 a_0 + l_1 a_1),
      // a_w = 2^(m_w - m); WG w stores output columns [64w, 64w+64). A unit cut by a stream-K range
      // boundary is stored unnormalised with (m, l) for k_sk_fixup.
      xml[wg][0][row] = m_run;
      xml[wg][1][row] = l_run;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");  // warps q and q+4
      const float m0 = xml[0][0][row], l0 = xml[0][1][row], m1 = xml[1][0][row], l1 = xml[1][1][row];
      // (persistent grid: xml is rewritten by the next item's epilogue; the mbarrier chain already orders
      // that after these reads, this barrier makes it explicit for the race checker)
      if constexpr (PERSIST) asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
      const float mm = fmaxf(m0, m1);
      const float a0 = l0 > 0.f ? fast_exp2(m0 - mm) : 0.f, a1 = l1 > 0.f ? fast_exp2(m1 - mm) : 0.f;
      const float lt = l0 * a0 + l1 * a1;
      const bool partial = PERSIST && (ta > 0 || te < it.len);
      // a row with no visible key in this item (possible only in a stream-K share made of pages past
      // the row's diagonal) contributes nothing: (m, l, O) = (-inf, 0, 0). (Its m is -inf but l is a
      // tiny positive sum of the polynomial exp2's clamped 2^-126 terms, so a_w = 2^(m_w - mm) is NaN.)
      const bool empty_row = !(lt > 0.f);
      const float inv = partial ? 1.f : (lt > 0.f ? 1.0f / lt : 0.f);
      const float c0f = a0 * inv, c1f = a1 * inv;
      mbar_wait(o_full, i & 1);
      tc_fence_after();
      const uint32_t ob0 = tmem + lane_off + 256 + wg * (D / 2), ob1 = ob0 + 128;
      // stream O from TMEM to global 32 columns at a time (final rows, or unnormalised partials)
      const long long obase = (long long)uc.b * args.o_bstride + (long long)p * args.o_stride +
                              (long long)h * D + wg * (D / 2);
      const int slot = partial ? it.slot(sk) : 0;
      const int prow = (int)cta * 128 + row;
      float* pdst = partial ? sk.part_o + ((long long)slot * 256 + prow) * D + wg * (D / 2) : nullptr;
#pragma unroll
      for (int cc = 0; cc < D / 2; cc += 32) {
        uint32_t o0[32], o1[32];
        tmem_ld32(ob0 + cc, o0);  // warp-collective (.sync.aligned): every lane, valid row or not
        tmem_ld32(ob1 + cc, o1);
        tmem_wait_ld();
        float v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c)
          v[c] = (PERSIST && empty_row) ? 0.f : __uint_as_float(o0[c]) * c0f + __uint_as_float(o1[c]) * c1f;
        if (!partial) {
          if (p < g.C) store_o_row32(args, obase + cc, v);
        } else {
          float4* dst = reinterpret_cast<float4*>(pdst + cc);
#pragma unroll
          for (int c = 0; c < 32; c += 4) dst[c / 4] = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
        }
      }
      if constexpr (PERSIST) {
        // O read out of TMEM: hand it to the next item's first P.V
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(o_empty, 0);
        if (partial && wg == 0) {
          sk.part_ml[((long long)slot * 256 + prow) * 2] = empty_row ? -INFINITY : mm;
          sk.part_ml[((long long)slot * 256 + prow) * 2 + 1] = empty_row ? 0.f : lt;
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync();  // no CTA leaves while the pair's MMAs / remote arrivals may still touch it
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem);
  }
}

// Merge of stream-K partials. Block (c, s) owns the unit of segment s that STARTS in cluster c's
// share and continues past it; its parts are cluster c's slot for that item and slot 0 (first item
// of the share) of every following cluster up to the one holding the unit's last page.
// O = sum_k O_k 2^(m_k - m) / sum_k l_k 2^(m_k - m), m = max_k m_k.
__global__ void __launch_bounds__(256) k_sk_fixup(Geo g, AttnArgs args, SkSched sk) {
  // block = (share cs, chunk of 8 rows): 32 blocks per share, one row per warp
  const int chunk = blockIdx.x & 31, cs = blockIdx.x >> 5;
  const int* fx = sk.fix + (long long)cs * kSkFixStride;
  const int np = fx[0];
  if (np == 0) return;
  const int unit = fx[1];
  const int* parts = fx + 2;
  const Unit uc = unit_coords(g, unit);
  const int D = g.d;
  // thread = (row r, 4 consecutive columns): a warp per row
  const int tx = threadIdx.x & 31;
  {
    const int r = chunk * 8 + (threadIdx.x >> 5);
    const int p = uc.qt * 128 + (r & 127);
    if (p >= g.C) return;
    float m = -INFINITY;
    for (int k = 0; k < np; ++k) m = fmaxf(m, sk.part_ml[((long long)parts[k] * 256 + r) * 2]);
    float l = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < np; ++k) {
      const long long pr = (long long)parts[k] * 256 + r;
      const float mk = sk.part_ml[pr * 2], lk = sk.part_ml[pr * 2 + 1];
      const float w = lk > 0.f ? exp2f(mk - m) : 0.f;
      l += lk * w;
      const float4 o = reinterpret_cast<const float4*>(sk.part_o + pr * D)[tx];
      acc.x += o.x * w; acc.y += o.y * w; acc.z += o.z * w; acc.w += o.w * w;
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const int h = uc.grp * g.E + uc.hp * 2 + (r >> 7);
    const long long off = (long long)uc.b * args.o_bstride + (long long)p * args.o_stride + (long long)h * D + tx * 4;
    const float v0 = acc.x * inv, v1 = acc.y * inv, v2 = acc.z * inv, v3 = acc.w * inv;
    for (int k = 0; k < args.n_out; ++k) {
      if (args.out_f32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(args.outs[k]) + off) = make_float4(v0, v1, v2, v3);
      } else {
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(args.outs[k]) + off) =
            make_uint2(pack_bf16x2(v0, v1), pack_bf16x2(v2, v3));
      }
    }
  }
}

template <int BS, bool PF16>
static cudaError_t launch_2cta_t(const CUtensorMap& tq, const CUtensorMap& tk_half, const CUtensorMap& tv,
                                 const Geo& g, const AttnArgs& a, const SkSched* sk, cudaStream_t st, int* launches) {
  cudaError_t e;
  const int units = (g.C + 127) / 128 * g.B * g.Gn * (g.E / 2);
  if (sk == nullptr) {
    using Cfg = Attn2Cfg<BS, false>;
    auto kern = k_paged_attn_2cta<BS, PF16, false>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem)) != cudaSuccess)
      return e;
    ++*launches;
    SkSched none{};
    return launch_ex(kern, dim3(2 * units), dim3(Cfg::kThreads), Cfg::kSmem, st, use_pdl(g), tq, tk_half, tv, g, a,
                     none);
  }
  using Cfg = Attn2Cfg<BS, true>;
  auto kern = k_paged_attn_2cta<BS, PF16, true>;
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem)) != cudaSuccess)
    return e;
  *launches += 3;
  k_sk_schedule<<<1, 1024, 0, st>>>(g, a, *sk);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  kern<<<2 * sk->clusters, Cfg::kThreads, Cfg::kSmem, st>>>(tq, tk_half, tv, g, a, *sk);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_sk_fixup<<<sk->clusters * sk->segments * 32, 256, 0, st>>>(g, a, *sk);
  return cudaGetLastError();
}

bool attn_2cta_supported(const Geo& g) { return g.d == 128 && (g.bs == 64 || g.bs == 128) && g.E % 2 == 0; }

// Co-resident clusters of the 2-CTA kernel on this device (persistent grid size), cached per device.
int attn_2cta_max_clusters(const Geo& g) {
  static int cached[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const int which = g.bs == 128 ? 0 : 1;
  if (dev >= 0 && dev < 64 && cached[dev][which] > 0) return cached[dev][which];
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(Attn2Cfg<128, true>::kThreads);
  cfg.gridDim = dim3(2);
  int n = 0;
  cudaError_t e;
  if (g.bs == 128) {
    cudaFuncSetAttribute(k_paged_attn_2cta<128, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Attn2Cfg<128, true>::kSmem);
    cfg.dynamicSmemBytes = Attn2Cfg<128, true>::kSmem;
    e = cudaOccupancyMaxActiveClusters(&n, k_paged_attn_2cta<128, true, true>, &cfg);
  } else {
    cudaFuncSetAttribute(k_paged_attn_2cta<64, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Attn2Cfg<64, true>::kSmem);
    cfg.dynamicSmemBytes = Attn2Cfg<64, true>::kSmem;
    e = cudaOccupancyMaxActiveClusters(&n, k_paged_attn_2cta<64, true, true>, &cfg);
  }
  if (e != cudaSuccess || n < 1) {
    cudaGetLastError();
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    n = sms / 2;
  }
  if (dev >= 0 && dev < 64) cached[dev][which] = n;
  return n;
}

cudaError_t launch_paged_attention_2cta(const CUtensorMap& tq, const CUtensorMap& tk_half, const CUtensorMap& tv,
                                        const Geo& g, const AttnArgs& a, const SkSched* sk, cudaStream_t st,
                                        int* launches) {
  const bool pf16 = !(g.flags & (1u << 8));
  if (g.bs == 128) return pf16 ? launch_2cta_t<128, true>(tq, tk_half, tv, g, a, sk, st, launches)
                               : launch_2cta_t<128, false>(tq, tk_half, tv, g, a, sk, st, launches);
  if (g.bs == 64) return pf16 ? launch_2cta_t<64, true>(tq, tk_half, tv, g, a, sk, st, launches)
                              : launch_2cta_t<64, false>(tq, tk_half, tv, g, a, sk, st, launches);
  return cudaErrorInvalidValue;
}


// ================================================================================================
// Row-split variant (default for d = 128, bs = 128, even E, per-unit grid): the same cluster pair
// and M=256 MMAs, but the 8 softmax warps split the CTA's 128 query rows instead of each page's keys:
// warp w owns TMEM lanes (rows) [32(w%4) + 16(w/4), +16) and all 128 keys of every page, accessed
// with the 16-lane tcgen05.ld/st shapes (16x256b: thread t holds rows t/4 and t/4+8, column pairs
// 8r + 2(t%4) + {0,1}; P is stored with 16x128b, column 4r + t%4 = the fp16 pair of those keys). Each
// row has ONE running max, so both warps' P.V accumulate into a single O, and the 128 TMEM columns
// this frees hold a third S buffer:
//   TMEM per CTA: S^0 [0,128) S^1 [128,256) S^2 [256,384) O [384,512).
// S(n+3) is issued right after P.V(n) (in-order tensor pipe), so the softmax of page n+1 never waits
// for the P.V of page n; the tensor core has a full page of slack (with two buffers S(n+2) had to wait
// for the lagging warpgroup's P(n)). Row max over a page = 32 values per thread plus
// two xor-shuffles across the row's 4 threads; the row sum is a per-thread partial reduced at the end.
// Warps: 0-7 softmax, 8-9 V bf16 -> fp16 converters (bf16 pool only), 10 TMA producer, 11 TMEM alloc +
// MMA issuer (CTA 0 issues for the pair).
struct AttnRsCfg {
  static constexpr int BS = 128, D = 128;
  static constexpr int kQBytes = 128 * D * 2;
  static constexpr int kKHalf = (BS / 2) * D * 2;  // keys [r*64, r*64+64) of a page
  static constexpr int kVHalf = BS * 64 * 2;       // head-dim columns [64r, 64r+64) of a page
  static constexpr int kKStages = 4, kVStages = 4;
  static constexpr int kConvWarps = 2;
  static constexpr int kThreads = 12 * 32;
  static constexpr int kSmem = kQBytes + kKStages * kKHalf + kVStages * kVHalf + 1024 + 1024;
  static_assert(kSmem + 2048 <= 232448, "shared memory budget");
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    k_paged_attn_rs(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k_half,
                    const __grid_constant__ CUtensorMap tm_v, Geo g, AttnArgs args) {
  using Cfg = AttnRsCfg;
  constexpr int D = Cfg::D, BS = Cfg::BS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::kQBytes;
  uint8_t* sV = sK + Cfg::kKStages * Cfg::kKHalf;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + Cfg::kVStages * Cfg::kVHalf);
  uint64_t* q_full = bars;                          // leader: both Q tiles landed (tx)
  uint64_t* k_full = q_full + 1;                    // leader: both K halves landed (tx)
  uint64_t* k_empty = k_full + Cfg::kKStages;       // both: K stage consumed (multicast commit)
  uint64_t* v_full = k_empty + Cfg::kKStages;       // leader (fp16 pool: both halves, tx) / local (bf16)
  uint64_t* v_empty = v_full + Cfg::kVStages;       // both: V stage consumed (multicast commit)
  uint64_t* v_ready = v_empty + Cfg::kVStages;      // leader: both V halves converted (bf16 pool)
  uint64_t* s_full = v_ready + Cfg::kVStages;       // both [3]: S^b computed (multicast commit)
  uint64_t* p_full = s_full + 3;                    // leader [3]: P^b written by all 16 softmax warps
  uint64_t* pv_done = p_full + 3;                   // both [2]: P.V of a page of that parity complete
  uint64_t* o_full = pv_done + 2;                   // both: every MMA of the unit complete
  uint64_t* stag = o_full + 1;                      // local [4 quarters][4]: warp q done with page max
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stag + 16);
  int* single_s = reinterpret_cast<int*>(tmem_slot + 1);  // {unit, start, n, nd}
  float* l_s = reinterpret_cast<float*>(single_s + 4);    // [128] row sums for the epilogue

  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
  const int cl = (int)blockIdx.x >> 1;
  const uint32_t warp = warp_id(), lane = lane_id();
  constexpr uint32_t kConvWarp0 = 8, kTmaWarp = 10, kMmaWarp = 11;
  const bool vf16 = (g.flags & (1u << 12)) != 0;  // CPA_F_V_F16: V pages already fp16

  if (warp == kTmaWarp) {
    if (lane == 0) {
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
      for (int b = 0; b < 3; ++b) { mbar_init(s_full + b, 1); mbar_init(p_full + b, 16); }
      mbar_init(pv_done, 1);
      mbar_init(pv_done + 1, 1);
      mbar_init(o_full, 1);
      for (int i = 0; i < 16; ++i) mbar_init(stag + i, 1);
      fence_barrier_init();
    }
    __syncwarp();
    pdl_wait();  // tables complete; the other threads wait at the cluster barrier below
    int s, n, nd;
    unit_table_warp(g, args, cl, &s, &n, &nd);
    if (lane == 0) { single_s[0] = cl; single_s[1] = s; single_s[2] = n; single_s[3] = nd; }
  }
  if (warp == kMmaWarp) tmem_alloc2<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers initialised, TMEM allocated in both CTAs
  tc_fence_after();
  pdl_wait();
  const uint32_t tmem = *tmem_slot;
  const int G = single_s[2];  // pages of this unit
  const Unit uc = unit_coords(g, cl);

  if (warp == kTmaWarp) {
    if (G > 0) {  // ------------------------------------------------------------ TMA producer
      const int h = uc.grp * g.E + uc.hp * 2 + (int)cta;
      const int kvh = group_kv_head(g, uc.grp);
      if (elect_one()) {
        if (leader) mbar_expect_tx(q_full, 2 * Cfg::kQBytes);
        tma_load_4d_2sm(sQ, &tm_q, q_full, 0, h, uc.qt * 128, uc.b);
        tma_load_4d_2sm(sQ + 128 * 128, &tm_q, q_full, 64, h, uc.qt * 128, uc.b);
      }
      __syncwarp();
      const int32_t* ptab = args.page_table + (long long)uc.b * g.maxb;
      const int st = single_s[1];
      for (int t = 0; t < G; ++t) {
        const int j = args.indptr != nullptr ? __ldg(args.indices + st + t) : t;
        const int page = __ldg(ptab + j);
        const int ks = t % Cfg::kKStages, vs = t % Cfg::kVStages;
        mbar_wait(k_empty + ks, ((t / Cfg::kKStages) & 1) ^ 1);
        if (elect_one()) {
          if (leader) mbar_expect_tx(k_full + ks, 2 * Cfg::kKHalf);
          uint8_t* dst = sK + ks * Cfg::kKHalf;
          tma_load_4d_2sm(dst, &tm_k_half, k_full + ks, 0, (int)cta * (BS / 2), kvh, page);
          tma_load_4d_2sm(dst + (BS / 2) * 128, &tm_k_half, k_full + ks, 64, (int)cta * (BS / 2), kvh, page);
        }
        __syncwarp();
        mbar_wait(v_empty + vs, ((t / Cfg::kVStages) & 1) ^ 1);
        if (elect_one()) {
          if (vf16) {  // both halves signal the leader's v_full directly
            if (leader) mbar_expect_tx(v_full + vs, 2 * Cfg::kVHalf);
            tma_load_4d_2sm(sV + vs * Cfg::kVHalf, &tm_v, v_full + vs, 64 * (int)cta, 0, kvh, page);
          } else {
            mbar_expect_tx(v_full + vs, Cfg::kVHalf);
            tma_load_4d(sV + vs * Cfg::kVHalf, &tm_v, v_full + vs, 64 * (int)cta, 0, kvh, page);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    if (leader && G > 0) {  // ---------------------------------------------------- MMA issuer (CTA 0)
      constexpr uint32_t idesc_s = umma_idesc_bf16(256, BS, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(256, D, 0, 1) & ~((7u << 7) | (7u << 10));  // fp16 A/B
      const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
      auto wait_k = [&](int n) {
        mbar_wait(k_full + n % Cfg::kKStages, (n / Cfg::kKStages) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int n) {  // S^{n%3} = Q K_n^T, M=256 (both CTAs' rows), N=BS, K=d
        const uint32_t d_tm = tmem + (n % 3) * 128;
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
          tc_commit2(s_full + n % 3);
          tc_commit2(k_empty + n % Cfg::kKStages);
        }
        __syncwarp();
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int n = 0; n < 3 && n < G; ++n) {
        wait_k(n);
        issue_s(n);
      }
      for (int n = 0; n < G; ++n) {
        mbar_wait((vf16 ? v_full : v_ready) + n % Cfg::kVStages, (n / Cfg::kVStages) & 1);
        mbar_wait(p_full + n % 3, (n / 3) & 1);
        tc_fence_after();
        // O += P^{n%3} V_n: M=256, N=d (64 columns per CTA), K=BS keys (P fp16 pairs over S^b [0, 64))
        const uint32_t p_tm = tmem + (n % 3) * 128;
        const uint32_t vb = v_base + (n % Cfg::kVStages) * Cfg::kVHalf;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BS / 16; ++kk) {
            const uint64_t bd = umma_desc_sw128(vb + kk * 16 * 128, BS * 128, 1024);
            mma2_ts(tmem + 384, p_tm + kk * 8, bd, idesc_o, (n > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit2(pv_done + (n & 1));
          tc_commit2(v_empty + n % Cfg::kVStages);
          if (n + 1 == G) tc_commit2(o_full);
        }
        __syncwarp();
        if (n + 3 < G) {  // S^{n%3} is free once P.V(n) (issued just before, in-order pipe) has read it
          wait_k(n + 3);
          issue_s(n + 3);
        }
      }
    }
  } else if (warp >= kConvWarp0) {  // --------------------------------------- V bf16 -> fp16
    const int ct = (warp - kConvWarp0) * 32 + lane;
    for (int n = 0; n < (vf16 ? 0 : G); ++n) {
      const int vs = n % Cfg::kVStages;
      mbar_wait(v_full + vs, (n / Cfg::kVStages) & 1);
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
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(v_ready + vs, 0);
    }
  } else {  // ------------------------------------------------------------------ softmax / epilogue
    const int quarter = warp & 3, hf = warp >> 2;
    const int base = quarter * 32 + hf * 16;  // this warp's 16 rows (TMEM lanes)
    const int t0 = lane & 3, t1 = lane >> 2;
    const int ra = base + t1, rb = ra + 8;    // the thread's two rows
    const float sl2 = g.scale * 1.4426950408889634f;
    const uint32_t lane_off = (uint32_t)base << 16;
    const int p0 = uc.qt * 128;
    const int lim_a = min(g.P + p0 + ra, g.L - 1), lim_b = min(g.P + p0 + rb, g.L - 1);
    const int st = single_s[1], nd = single_s[3];
    float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
    for (int t = 0; t < G; ++t) {
      const int b = t % 3;
#ifndef CPA_NO_STAGGER
      // the two warps of an SMSP (same quarter): the second starts a page once the first has its max
      if (hf == 1) mbar_wait(stag + quarter * 4 + (t & 3), (t >> 2) & 1);
#endif
      mbar_wait(s_full + b, (t / 3) & 1);
      tc_fence_after();
      uint32_t sv[64];
      tmem_ld_16x256b_x16(tmem + lane_off + b * 128, sv);
      tmem_wait_ld();
      if (t >= nd) {  // block crosses the causal diagonal of this tile: mask in absolute positions
        const int j = args.indptr != nullptr ? __ldg(args.indices + st + t) : t;
        const int tb = j * g.bs + 2 * t0;
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (tb + 8 * r + e > lim_a) sv[4 * r + e] = __float_as_uint(-INFINITY);
            if (tb + 8 * r + e > lim_b) sv[4 * r + 2 + e] = __float_as_uint(-INFINITY);
          }
      }
      float ma0 = -INFINITY, ma1 = -INFINITY, mb0 = -INFINITY, mb1 = -INFINITY;
#pragma unroll
      for (int r = 0; r < 16; r += 2) {
        ma0 = fmax3(ma0, __uint_as_float(sv[4 * r]), __uint_as_float(sv[4 * r + 1]));
        ma1 = fmax3(ma1, __uint_as_float(sv[4 * r + 4]), __uint_as_float(sv[4 * r + 5]));
        mb0 = fmax3(mb0, __uint_as_float(sv[4 * r + 2]), __uint_as_float(sv[4 * r + 3]));
        mb1 = fmax3(mb1, __uint_as_float(sv[4 * r + 6]), __uint_as_float(sv[4 * r + 7]));
      }
      float mxa = fmaxf(ma0, ma1), mxb = fmaxf(mb0, mb1);
      mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 1));
      mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 1));
      mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 2));
      mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 2));
      const float mba = mxa * sl2, mbb = mxb * sl2;
      float fa = 1.f, fb = 1.f;
      const bool ra_s = mba > m_a + CPA_RESCALE_THRESH, rb_s = mbb > m_b + CPA_RESCALE_THRESH;  // lazy rescale
      if (ra_s) {
        if (m_a != -INFINITY) fa = fast_exp2(m_a - mba);
        m_a = mba;
      }
      if (rb_s) {
        if (m_b != -INFINITY) fb = fast_exp2(m_b - mbb);
        m_b = mbb;
      }
      const float ua = (m_a == -INFINITY) ? 0.f : m_a, ub = (m_b == -INFINITY) ? 0.f : m_b;
#ifndef CPA_NO_STAGGER
      if (hf == 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(stag + quarter * 4 + (t & 3));
      }
#endif
      // P = exp2(s*sl2 - m) per row: packed FFMA2 on each column pair, 1/4 of the pairs on the FMA-pipe
      // polynomial, the rest on MUFU.EX2; fp16 pairs stored over S^b columns [0, 64) (16x128b).
      float2 acc_a = {0.f, 0.f}, acc_b = {0.f, 0.f};
      uint32_t pk[32];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const float2 xa = ffma2(make_float2(__uint_as_float(sv[4 * r]), __uint_as_float(sv[4 * r + 1])), sl2, -ua);
        const float2 xb = ffma2(make_float2(__uint_as_float(sv[4 * r + 2]), __uint_as_float(sv[4 * r + 3])), sl2, -ub);
        float2 ea, eb;
        if (use_poly_exp(2 * r)) {
          ea = exp2_poly2(xa);
        } else {
          ea.x = fast_exp2(xa.x);
          ea.y = fast_exp2(xa.y);
        }
        if (use_poly_exp(2 * r + 1)) {
          eb = exp2_poly2(xb);
        } else {
          eb.x = fast_exp2(xb.x);
          eb.y = fast_exp2(xb.y);
        }
        acc_a = fadd2(acc_a, ea);
        acc_b = fadd2(acc_b, eb);
        pk[2 * r] = pack_f16x2(ea.x, ea.y);
        pk[2 * r + 1] = pack_f16x2(eb.x, eb.y);
      }
      tmem_st_16x128b_x16(tmem + lane_off + b * 128, pk);
      l_a = l_a * fa + (acc_a.x + acc_a.y);
      l_b = l_b * fb + (acc_b.x + acc_b.y);
      // rescale O's rows (this warp's 16) after the previous P.V completed, before P.V(t) is issued;
      // not on the first page (its P.V overwrites O). pv_done[x] completes once per page of parity x and
      // P.V(t-3) is complete here (S(t) was issued after it), so its phase is known within one.
      if (__any_sync(0xffffffffu, (ra_s || rb_s) && t > 0)) {
        mbar_wait(pv_done + ((t - 1) & 1), ((t - 1) >> 1) & 1);
        tc_fence_after();
        uint32_t o[64];
        tmem_ld_16x256b_x16(tmem + lane_off + 384, o);
        tmem_wait_ld();
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          o[4 * r] = __float_as_uint(__uint_as_float(o[4 * r]) * fa);
          o[4 * r + 1] = __float_as_uint(__uint_as_float(o[4 * r + 1]) * fa);
          o[4 * r + 2] = __float_as_uint(__uint_as_float(o[4 * r + 2]) * fb);
          o[4 * r + 3] = __float_as_uint(__uint_as_float(o[4 * r + 3]) * fb);
        }
        tmem_st_16x256b_x16(tmem + lane_off + 384, o);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(p_full + b, 0);
    }
    // ---- epilogue: O / l. Row sums: reduce the row's 4 partials, exchange through shared memory so
    // that warp (q, hf) stores output columns [64 hf, 64 hf + 64) of the quarter's 32 rows (32x32b).
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
    if (t0 == 0) {
      l_s[ra] = l_a;
      l_s[rb] = l_b;
    }
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");  // warps q and q+4
    const int row = quarter * 32 + lane;
    const float lt = l_s[row];
    const float inv = lt > 0.f ? 1.0f / lt : 0.f;
    mbar_wait(o_full, 0);
    tc_fence_after();
    const int h = uc.grp * g.E + uc.hp * 2 + (int)cta;
    const int p = p0 + row;
    const long long obase = (long long)uc.b * args.o_bstride + (long long)p * args.o_stride + (long long)h * D + hf * 64;
    const uint32_t ob = tmem + ((uint32_t)(quarter * 32) << 16) + 384 + hf * 64;
#pragma unroll
    for (int cc = 0; cc < 64; cc += 32) {
      uint32_t o[32];
      tmem_ld32(ob + cc, o);  // warp-collective: every lane, valid row or not
      tmem_wait_ld();
      float v[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = __uint_as_float(o[c]) * inv;
      if (p < g.C) store_o_row32(args, obase + cc, v);
    }
  }
  tc_fence_before();
  cluster_sync();  // no CTA leaves while the pair's MMAs / remote arrivals may still touch it
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem);
  }
}

bool attn_rs_supported(const Geo& g) { return g.d == 128 && g.bs == 128 && g.E % 2 == 0 && !(g.flags & (1u << 8)); }

cudaError_t launch_paged_attention_rs(const CUtensorMap& tq, const CUtensorMap& tk_half, const CUtensorMap& tv,
                                      const Geo& g, const AttnArgs& a, cudaStream_t st, int* launches) {
  using Cfg = AttnRsCfg;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_paged_attn_rs, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem)) !=
      cudaSuccess)
    return e;
  const int units = (g.C + 127) / 128 * g.B * g.Gn * (g.E / 2);
  ++*launches;
  return launch_ex(k_paged_attn_rs, dim3(2 * units), dim3(Cfg::kThreads), Cfg::kSmem, st, use_pdl(g), tq, tk_half, tv,
                   g, a);
}

}  // namespace cpa

#ifdef CPA_TRACE
extern "C" __attribute__((visibility("default"))) int cpa_debug_trace2(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, cpa::g_trace2, sizeof(cpa::g_trace2));
}
#endif
