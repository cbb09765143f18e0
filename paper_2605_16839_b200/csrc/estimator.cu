// estimator.cu -- §8 rows a1/a2: pooled-query max-threshold block scores on sm_100a.
//
// SPEC.md:220-228 + 269 (pooled variant): for each (b, h, q-block i) the block-mean query
// qbar; for each KV block j <= pb+i the tile max over its causal keys of scale*qbar.k_t.
// One execution group (b, g) is one GEMM: A = qbar rows r = hl*nqb + i (E*nqb rows, padded
// to 128), B = each K page of KV head g*E/(Hq/Hkv) streamed by TMA through the page table;
// D = 128 x bs fp32 in TMEM; the epilogue takes the per-row max over the page's keys.
// qbar is split hi = bf16(qbar), lo = bf16(qbar - hi) and both are accumulated into the same
// TMEM tile, so the score carries ~2^-16 relative error instead of bf16's 2^-8 (K2).
#include "common.cuh"
#include "geo.cuh"
#include "launch.cuh"

namespace cpa {

// ---------------------------------------------------------------- a1: pool Q
// grid (nqb + 1, B, ceil(Hq*d/128)), block 256 threads = 16 token parts x 16 slab threads; a slab
// thread owns 8 consecutive elements (one uint4) of a 128-element slice of [Hq*d] (narrow slices: at one
// KV group per GPU, Hq*d = 512, 512-element slices gave only nqb + 1 CTAs); each part sums
// 1/16 of the q-block's tokens with all its loads in flight at once (8 for bs = 128), the parts are
// combined in shared memory. Blocks x = nqb zero the padding rows [R, Rpad) of qbar (padded MMA rows
// must be finite). qbar: [2][B*Gn*Rpad][d] bf16 (hi rows, then lo rows).
constexpr int kPoolParts = 16;
constexpr int kSlabT = 16;  // slab threads per CTA (kSlabT * 8 elements of [Hq*d])
__global__ void __launch_bounds__(kPoolParts * kSlabT) k_pool_q(const __nv_bfloat16* __restrict__ q, Geo g,
                                                 __nv_bfloat16* __restrict__ qbar, int* __restrict__ mstar_key,
                                                 unsigned* __restrict__ tables_done) {
  __shared__ float part[kPoolParts - 1][kSlabT][9];
  const int i = blockIdx.x, b = blockIdx.y;
  pdl_trigger();  // block_scores may start its prologue; it waits for this grid before reading qbar
  if (i == 0 && b == 0 && blockIdx.z == 0 && threadIdx.x == 0) *tables_done = 0u;  // k_mask_union's counter
  const long long nrows = (long long)g.B * g.Gn * g.Rpad;
  if (i == g.nqb) {  // padding rows of the groups z, z + gridDim.z, ... of batch b
    const int npad = g.Rpad - g.R, per_row = g.d / 8;  // uint4 per row
    for (int grp = blockIdx.z; grp < g.Gn; grp += gridDim.z)
      for (int x = threadIdx.x; x < npad * per_row; x += blockDim.x) {
        const long long row = ((long long)b * g.Gn + grp) * g.Rpad + g.R + x / per_row;
        const int e = (x % per_row) * 8;
        *reinterpret_cast<uint4*>(qbar + row * g.d + e) = make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(qbar + (nrows + row) * g.d + e) = make_uint4(0u, 0u, 0u, 0u);
      }
    pdl_wait();  // this grid completes only after its predecessor (the append of the chunk's K/V)
    return;
  }
  const int st = threadIdx.x % kSlabT, pt = threadIdx.x / kSlabT;
  const int x0 = (blockIdx.z * kSlabT + st) * 8;  // element offset in [0, Hq*d)
  const bool active = x0 < g.Hq * g.d;         // last slab may be partial (Hq*d % 512 != 0)
  const int p0 = i * g.bs, p1 = min(p0 + g.bs, g.C);
  const int nq = (p1 - p0 + kPoolParts - 1) / kPoolParts;
  const int a0 = min(p0 + pt * nq, p1), a1 = active ? min(a0 + nq, p1) : a0;
  const uint4* src = reinterpret_cast<const uint4*>(q + (long long)b * g.b_stride + x0);
  const long long stride = g.q_stride / 8;  // uint4 per token
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  auto add = [&](const uint4& w) {
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      acc[2 * c] += __uint_as_float(ws[c] << 16);
      acc[2 * c + 1] += __uint_as_float(ws[c] & 0xffff0000u);
    }
  };
  int p = a0;
  for (; p + 8 <= a1; p += 8) {
    uint4 w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) w[u] = __ldg(src + (long long)(p + u) * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) add(w[u]);
  }
  for (; p < a1; ++p) add(__ldg(src + (long long)p * stride));
  if (pt > 0) {
#pragma unroll
    for (int c = 0; c < 8; ++c) part[pt - 1][st][c] = acc[c];
  }
  __syncthreads();
  pdl_wait();  // this grid completes only after its predecessor (the append of the chunk's K/V)
  if (pt != 0 || !active) return;
  for (int k = 0; k < kPoolParts - 1; ++k)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] += part[k][st][c];
  const int h = x0 / g.d, e = x0 % g.d;
  const float inv = 1.0f / float(p1 - p0);
  uint32_t hi[4], lo[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float m0 = acc[2 * c] * inv, m1 = acc[2 * c + 1] * inv;
    const __nv_bfloat16 h0 = __float2bfloat16_rn(m0), h1 = __float2bfloat16_rn(m1);
    hi[c] = pack_bf16x2(__bfloat162float(h0), __bfloat162float(h1));
    lo[c] = pack_bf16x2(m0 - __bfloat162float(h0), m1 - __bfloat162float(h1));
  }
  const int grp = h / g.E, hl = h % g.E;
  const long long row = ((long long)b * g.Gn + grp) * g.Rpad + hl * g.nqb + i;
  *reinterpret_cast<uint4*>(qbar + row * g.d + e) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  *reinterpret_cast<uint4*>(qbar + (nrows + row) * g.d + e) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  if (e == 0) mstar_key[row] = float_key(-INFINITY);
}

// ---------------------------------------------------------------- a2: block scores
#ifndef CPA_SCORE_STAGES
#define CPA_SCORE_STAGES 4
#endif
template <int D, int BS>
struct ScoreCfg {
  static constexpr int kAtoms = D / 64;            // 128-byte swizzle atoms along d
  static constexpr int kStages = (D * BS * 2 * CPA_SCORE_STAGES + 2 * 128 * D * 2 + 1280 <= 232448 - 1024)
                                     ? CPA_SCORE_STAGES : 4;
  static constexpr int kABytes = 128 * D * 2;      // one 128-row qbar tile
  static constexpr int kKBytes = BS * D * 2;       // one K page
  static constexpr int kTmemCols = (2 * BS) <= 32 ? 32 : (2 * BS);
  static constexpr int kSmem = 2 * kABytes + kStages * kKBytes + 1024 /*align*/ + 256 /*bars*/;
};

template <int D, int BS>
__global__ void __launch_bounds__(192, 1)
    k_block_scores(const __grid_constant__ CUtensorMap tm_qbar, const __grid_constant__ CUtensorMap tm_k,
                   const int32_t* __restrict__ page_table, Geo g, int pages_per_cta,
                   float* __restrict__ scores, int* __restrict__ mstar_key) {
  using Cfg = ScoreCfg<D, BS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA_hi = smem;
  uint8_t* sA_lo = smem + Cfg::kABytes;
  uint8_t* sK = smem + 2 * Cfg::kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sK + Cfg::kStages * Cfg::kKBytes);
  uint64_t* bar_a = bars;                          // A tiles landed
  uint64_t* full = bars + 1;                       // [kStages] K page landed
  uint64_t* empty = full + Cfg::kStages;           // [kStages] K page consumed
  uint64_t* acc_full = empty + Cfg::kStages;       // [2] accumulator ready
  uint64_t* acc_empty = acc_full + 2;              // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int bg = blockIdx.z, b = bg / g.Gn, grp = bg % g.Gn;
  const int rt = blockIdx.y;
  const int j0 = blockIdx.x * pages_per_cta;
  const int j1 = min(g.nkvb, j0 + pages_per_cta);
  const int n_pages = j1 - j0;
  if (n_pages <= 0) return;  // uniform across the CTA
  const int kvh = group_kv_head(g, grp);
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qbar);
    tma_prefetch_desc(&tm_k);
    mbar_init(bar_a, 1);
    for (int s = 0; s < Cfg::kStages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(acc_full + s, 1); mbar_init(acc_empty + s, 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();  // mask_union may be scheduled (it waits for this grid)

  // TMA / MMA roles: whole warp runs the loop (warp-uniform values live in uniform registers),
  // one elected lane issues each TMA / tcgen05 instruction.
  if (warp == 0) {  // ---------------- TMA producer
    const int row0 = bg * g.Rpad + rt * 128;
    const int nrows = g.B * g.Gn * g.Rpad;
    const uint64_t pol = l2_policy_evict_first();
    auto load_k = [&](int n) {
      const int s = n % Cfg::kStages;
      const int page = __ldg(page_table + (long long)b * g.maxb + j0 + n);
      mbar_wait(empty + s, ((n / Cfg::kStages) & 1) ^ 1);
      uint8_t* dst = sK + s * Cfg::kKBytes;
      if (elect_one()) {
        mbar_expect_tx(full + s, Cfg::kKBytes);
#pragma unroll
        for (int a = 0; a < Cfg::kAtoms; ++a)
          tma_load_4d_hint(dst + a * BS * 128, &tm_k, full + s, 64 * a, 0, kvh, page, pol);
      }
      __syncwarp();
    };
    // (PDL) the first pages of the ring before waiting for the predecessors, if they are prefix pages
    // (j < pb): only the chunk's own pages [pb, nkvb) are written by this step's append, and the page
    // table / earlier pages were complete before the append started (its pdl_wait)
    int n0 = 0;
    while (n0 < Cfg::kStages && n0 < n_pages && j0 + n0 < g.pb) load_k(n0++);
    pdl_wait();  // qbar (pool_q) and the appended K pages are complete
    if (elect_one()) {
      mbar_expect_tx(bar_a, 2 * Cfg::kABytes);
#pragma unroll
      for (int a = 0; a < Cfg::kAtoms; ++a) {
        tma_load_2d(sA_hi + a * 128 * 128, &tm_qbar, bar_a, 64 * a, row0);
        tma_load_2d(sA_lo + a * 128 * 128, &tm_qbar, bar_a, 64 * a, nrows + row0);
      }
    }
    __syncwarp();
    for (int n = n0; n < n_pages; ++n) load_k(n);
  } else if (warp == 1) {  // ---------------- MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(128, BS, 0, 0);
    mbar_wait(bar_a, 0);
    tc_fence_after();
    const uint32_t a_hi = smem_u32(sA_hi), a_lo = smem_u32(sA_lo);
    for (int n = 0; n < n_pages; ++n) {
      const int s = n % Cfg::kStages, acc = n & 1;
      mbar_wait(full + s, (n / Cfg::kStages) & 1);
      mbar_wait(acc_empty + acc, ((n >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t kb = smem_u32(sK + s * Cfg::kKBytes);
      const uint32_t d_tm = tmem + acc * BS;
      if (elect_one()) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const uint32_t abase = half ? a_lo : a_hi;
#pragma unroll
          for (int a = 0; a < Cfg::kAtoms; ++a)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ad = umma_desc_sw128(abase + a * 128 * 128 + kk * 32, 16, 1024);
              const uint64_t bd = umma_desc_sw128(kb + a * BS * 128 + kk * 32, 16, 1024);
              mma_ss(d_tm, ad, bd, idesc, (half | a | kk) != 0);
            }
        }
        tc_commit(empty + s);
        tc_commit(acc_full + acc);
      }
      __syncwarp();
    }
  } else {  // ---------------- epilogue: warps 2..5, one accumulator row per thread
    const int quarter = warp & 3;
    const int r_loc = quarter * 32 + lane;
    const int r = rt * 128 + r_loc;
    const bool valid_row = r < g.R;
    const int i = valid_row ? r % g.nqb : 0;
    const int lim = g.P + min((i + 1) * g.bs, g.C) - 1;  // last absolute key the pooled query sees
    pdl_wait();  // (PDL) the row-max keys (pool_q) are initialised before this warp touches them
    float row_best = -INFINITY;
    for (int n = 0; n < n_pages; ++n) {
      const int acc = n & 1, j = j0 + n;
      mbar_wait(acc_full + acc, (n >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + acc * BS;
      float mx = -INFINITY;
      const int tbase = j * g.bs;
      const bool needs_mask = tbase + BS - 1 > lim;
      if constexpr (BS >= 32) {
#pragma unroll
        for (int c0 = 0; c0 < BS; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(taddr + c0, v);
          tmem_wait_ld();
          if (needs_mask) {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (tbase + c0 + c <= lim) mx = fmaxf(mx, __uint_as_float(v[c]));
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c) mx = fmaxf(mx, __uint_as_float(v[c]));
          }
        }
      } else {
        uint32_t v[16];
        tmem_ld16(taddr, v);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c < BS && tbase + c <= lim) mx = fmaxf(mx, __uint_as_float(v[c]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + acc);
      const bool causal = valid_row && j <= g.pb + i;
      const float m = causal ? mx * g.scale : -INFINITY;
      scores[((long long)bg * g.nkvb + j) * g.Rpad + r] = m;
      row_best = fmaxf(row_best, m);
    }
    if (valid_row) atomicMax(mstar_key + (long long)bg * g.Rpad + r, float_key(row_best));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
}

// ---------------------------------------------------------------- NEXT-1: exact tile-max scores
// SPEC.md:223 (the spec's default scorer): m[b,h,i,j] = max over the causal pairs (p in q-block i,
// t in block j, t <= P+p) of scale * q_p . k_t, i.e. the tile max of the full QK^T. CTA = (b, head h,
// q-block i, split of the pages j <= pb+i); A = the q-block's bs x d query tile (TMA from q), B = each K
// page; D = bs x bs fp32 in TMEM; epilogue: per-row masked max -> warp max -> CTA max (named barrier),
// written in the same [B*Gn][nkvb][Rpad] score layout (row r = hl*nqb + i) as the pooled estimator.
// Not the hot path: it costs a full QK^T (~half of dense attention); selected by CPA_F_EXACT_SCORES.
template <int D, int BS>
struct ExactCfg {
  static constexpr int kAtoms = D / 64;
  static constexpr int kStages = 4;
  static constexpr int kQBytes = 128 * D * 2;
  static constexpr int kKBytes = BS * D * 2;
  static constexpr int kTmemCols = (2 * BS) <= 32 ? 32 : (2 * BS);
  static constexpr int kSmem = kQBytes + kStages * kKBytes + 1024 + 256;
};

template <int D, int BS>
__global__ void __launch_bounds__(192, 1)
    k_block_scores_exact(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const int32_t* __restrict__ page_table, Geo g, int pages_per_cta,
                         float* __restrict__ scores, int* __restrict__ mstar_key) {
  using Cfg = ExactCfg<D, BS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + Cfg::kQBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sK + Cfg::kStages * Cfg::kKBytes);
  uint64_t* bar_q = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* acc_full = empty + Cfg::kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  __shared__ float wmax[4];

  const int bh = blockIdx.z, b = bh / g.Hq, h = bh % g.Hq;
  const int i = blockIdx.y;
  const int jmax = g.pb + i;  // causal-valid blocks
  const int j0 = blockIdx.x * pages_per_cta;
  const int j1 = min(jmax + 1, j0 + pages_per_cta);
  const int n_pages = j1 - j0;
  if (n_pages <= 0) return;
  const int grp = h / g.E, hl = h % g.E;
  const int kvh = h / g.kv_per_q;
  const int p0 = i * g.bs;  // q-block i = chunk positions [p0, p0 + bs)
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    mbar_init(bar_q, 1);
    for (int s = 0; s < Cfg::kStages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(acc_full + s, 1); mbar_init(acc_empty + s, 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // ---------------- TMA producer (queries of the q-block: 128 rows, rows >= bs unused)
    if (elect_one()) {
      mbar_expect_tx(bar_q, Cfg::kQBytes);
#pragma unroll
      for (int a = 0; a < Cfg::kAtoms; ++a) tma_load_4d(sQ + a * 128 * 128, &tm_q, bar_q, 64 * a, h, p0, b);
    }
    __syncwarp();
    for (int n = 0; n < n_pages; ++n) {
      const int s = n % Cfg::kStages;
      const int page = __ldg(page_table + (long long)b * g.maxb + j0 + n);
      mbar_wait(empty + s, ((n / Cfg::kStages) & 1) ^ 1);
      if (elect_one()) {
        mbar_expect_tx(full + s, Cfg::kKBytes);
#pragma unroll
        for (int a = 0; a < Cfg::kAtoms; ++a)
          tma_load_4d(sK + s * Cfg::kKBytes + a * BS * 128, &tm_k, full + s, 64 * a, 0, kvh, page);
      }
      __syncwarp();
    }
  } else if (warp == 1) {  // ---------------- MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(128, BS, 0, 0);
    mbar_wait(bar_q, 0);
    tc_fence_after();
    const uint32_t qa = smem_u32(sQ);
    for (int n = 0; n < n_pages; ++n) {
      const int s = n % Cfg::kStages, acc = n & 1;
      mbar_wait(full + s, (n / Cfg::kStages) & 1);
      mbar_wait(acc_empty + acc, ((n >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t kb = smem_u32(sK + s * Cfg::kKBytes);
      if (elect_one()) {
#pragma unroll
        for (int a = 0; a < Cfg::kAtoms; ++a)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ss(tmem + acc * BS, umma_desc_sw128(qa + a * 128 * 128 + kk * 32, 16, 1024),
                   umma_desc_sw128(kb + a * BS * 128 + kk * 32, 16, 1024), idesc, (a | kk) != 0);
        tc_commit(empty + s);
        tc_commit(acc_full + acc);
      }
      __syncwarp();
    }
  } else {  // ---------------- epilogue: warps 2..5, one query row per thread
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int p = p0 + row;
    const bool valid = row < g.bs && p < g.C;
    const int lim = valid ? g.P + p : -1;  // t <= P + p
    const int r = hl * g.nqb + i;
    const long long bg = (long long)b * g.Gn + grp;
    float best = -INFINITY;
    for (int n = 0; n < n_pages; ++n) {
      const int acc = n & 1, j = j0 + n;
      mbar_wait(acc_full + acc, (n >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + acc * BS;
      const int tbase = j * g.bs;
      float mx = -INFINITY;
      if constexpr (BS >= 32) {
#pragma unroll
        for (int c0 = 0; c0 < BS; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(taddr + c0, v);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (tbase + c0 + c <= lim) mx = fmaxf(mx, __uint_as_float(v[c]));
        }
      } else {
        uint32_t v[16];
        tmem_ld16(taddr, v);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c < BS && tbase + c <= lim) mx = fmaxf(mx, __uint_as_float(v[c]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + acc);
      // tile max over the 128 query rows: warp max on order-preserving int keys, then 4 warps
      const int wk = __reduce_max_sync(0xffffffffu, float_key(mx));
      if (lane == 0) wmax[quarter] = key_float(wk);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (row == 0) {
        const float m = fmaxf(fmaxf(wmax[0], wmax[1]), fmaxf(wmax[2], wmax[3])) * g.scale;
        scores[(bg * g.nkvb + j) * g.Rpad + r] = m;
        best = fmaxf(best, m);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    if (row == 0) atomicMax(mstar_key + bg * g.Rpad + r, float_key(best));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
}

// scores / row-max initialisation for the exact scorer: every causal-invalid tile stays -inf
__global__ void k_scores_init(Geo g, float* __restrict__ scores, int* __restrict__ mstar_key) {
  const long long ns = (long long)g.B * g.Gn * g.nkvb * g.Rpad, nm = (long long)g.B * g.Gn * g.Rpad;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < ns; x += (long long)gridDim.x * blockDim.x) {
    scores[x] = -INFINITY;
    if (x < nm) mstar_key[x] = float_key(-INFINITY);
  }
}

template <int D, int BS>
static cudaError_t launch_exact_t(const CUtensorMap& tq, const CUtensorMap& tk, const int32_t* pt, const Geo& g,
                                  float* scores, int* mstar_key, int num_sms, cudaStream_t st) {
  using Cfg = ExactCfg<D, BS>;
  auto kern = k_block_scores_exact<D, BS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
  if (e != cudaSuccess) return e;
  const long long units = (long long)g.B * g.Hq * g.nqb;
  int splits = (int)((2LL * num_sms + units - 1) / units);
  if (splits < 1) splits = 1;
  if (splits > g.nkvb) splits = g.nkvb;
  const int ppc = (g.nkvb + splits - 1) / splits;
  splits = (g.nkvb + ppc - 1) / ppc;
  kern<<<dim3(splits, g.nqb, g.B * g.Hq), 192, Cfg::kSmem, st>>>(tq, tk, pt, g, ppc, scores, mstar_key);
  return cudaGetLastError();
}

cudaError_t launch_block_scores_exact(const CUtensorMap& tq, const CUtensorMap& tk, const int32_t* pt,
                                      const Geo& g, float* scores, int* mstar_key, int num_sms, cudaStream_t st,
                                      int* launches) {
  k_scores_init<<<1024, 256, 0, st>>>(g, scores, mstar_key);
  *launches += 2;
#define CPA_SC(DD, BB) \
  if (g.d == DD && g.bs == BB) return launch_exact_t<DD, BB>(tq, tk, pt, g, scores, mstar_key, num_sms, st);
  CPA_SC(64, 16) CPA_SC(64, 32) CPA_SC(64, 64) CPA_SC(64, 128)
  CPA_SC(128, 16) CPA_SC(128, 32) CPA_SC(128, 64) CPA_SC(128, 128)
#undef CPA_SC
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- launchers
int score_smem_bytes(int d, int bs) {
#define CPA_SC(DD, BB) if (d == DD && bs == BB) return ScoreCfg<DD, BB>::kSmem;
  CPA_SC(64, 16) CPA_SC(64, 32) CPA_SC(64, 64) CPA_SC(64, 128)
  CPA_SC(128, 16) CPA_SC(128, 32) CPA_SC(128, 64) CPA_SC(128, 128)
#undef CPA_SC
  return -1;
}

cudaError_t launch_pool_q(const __nv_bfloat16* q, const Geo& g, __nv_bfloat16* qbar, int* mstar_key,
                          unsigned* tables_done, bool after_append, cudaStream_t st, int* launches) {
  // x = nqb: padding blocks (they return at once when Rpad == R). PDL only right after k_append (whose
  // pdl_wait orders it after everything before): then q, qbar and the counters are safe to touch early.
  ++*launches;
  return launch_ex(k_pool_q, dim3(g.nqb + (g.Rpad > g.R ? 1 : 0), g.B, (g.Hq * g.d + kSlabT * 8 - 1) / (kSlabT * 8)),
                   dim3(kPoolParts * kSlabT), 0, st,
                   after_append && use_pdl(g), q, g, qbar, mstar_key, tables_done);
}

template <int D, int BS>
static cudaError_t launch_scores_t(const CUtensorMap& tq, const CUtensorMap& tk, const int32_t* pt,
                                   const Geo& g, float* scores, int* mstar_key, int num_sms,
                                   cudaStream_t st) {
  using Cfg = ScoreCfg<D, BS>;
  auto kern = k_block_scores<D, BS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
  if (e != cudaSuccess) return e;
  const int units = g.B * g.Gn * (g.Rpad / 128);
  int splits = num_sms / units;
  if (splits < 1) splits = 1;
  if (splits > g.nkvb) splits = g.nkvb;
  const int ppc = (g.nkvb + splits - 1) / splits;
  splits = (g.nkvb + ppc - 1) / ppc;
  return launch_ex(kern, dim3(splits, g.Rpad / 128, g.B * g.Gn), dim3(192), Cfg::kSmem, st, use_pdl(g), tq, tk, pt, g,
                   ppc, scores, mstar_key);
}

cudaError_t launch_block_scores(const CUtensorMap& tq, const CUtensorMap& tk, const int32_t* pt,
                                const Geo& g, float* scores, int* mstar_key, int num_sms,
                                cudaStream_t st, int* launches) {
  ++*launches;
#define CPA_SC(DD, BB) \
  if (g.d == DD && g.bs == BB) return launch_scores_t<DD, BB>(tq, tk, pt, g, scores, mstar_key, num_sms, st);
  CPA_SC(64, 16) CPA_SC(64, 32) CPA_SC(64, 64) CPA_SC(64, 128)
  CPA_SC(128, 16) CPA_SC(128, 32) CPA_SC(128, 64) CPA_SC(128, 128)
#undef CPA_SC
  return cudaErrorInvalidValue;
}

}  // namespace cpa
