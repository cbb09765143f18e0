// attention.cu -- §8 row a6: zero-copy paged attention over the tabled KV blocks, tcgen05/TMEM.
//
// each (batch b, execution group g) attends only to the blocks
// T[b,g] listed in kv_indices, read in place from the paged cache; causal masking is done in
// ABSOLUTE positions (query p at P+p sees keys t <= P+p) so the fully-open current chunk keeps
// causal semantics.  Value:
//   O[b,p,h] = sum_{t in A(p)} softmax_t(scale q_p.k_t) v_t,  A(p) = {t : t/bs in T[b,h/E], t <= P+p}.
//
// CTA = (b, g, 128-token q-tile, pair of query heads of g) -> NT=2 Q tiles of 128 rows that
// share every K/V page (GQA packing). Warp roles:
//   warps 0-3  softmax for tile 0 (one TMEM lane = one query row per thread)
//   warps 4-7  softmax for tile 1
//   warps 8-9  V converter: each landed bf16 V tile -> fp16 in place (P.V runs in fp16, DESIGN K3)
//   warp  10   TMA producer: kv_indices -> page_table -> cp.async.bulk.tensor K/V pages
//   warp  11   TMEM allocator + single-thread tcgen05.mma issuer
// Each page is processed as SPB sub-blocks of SB = min(bs, 64) keys. TMEM (512 columns):
//   S_t^0 [t*128, +64)  S_t^1 [t*128+64, +64)  O_t [NT*128 + t*128, +d)      (P_t aliases S_t^b)
// S is double-buffered per tile, so the tensor core computes S_t(u+1) while the softmax of
// S_t(u) runs; the softmax is the only serial link (S_t(u) -> P_t(u) -> PV_t(u)).
// MMA order per sub-block u: PV_0(u), S_0(u+2), PV_1(u), S_1(u+2). Online softmax in the log2
// domain with lazy O rescaling (only when the running max grows by > 8, so P <= 256).
#include "common.cuh"
#include "geo.cuh"
#include "out_store.cuh"

namespace cpa {

#ifdef CPA_TRACE
__device__ long long g_trace[16][2048];
#define TRACE(e, i) \
  do { if (blockIdx.x == 0 && (i) < 2048) g_trace[e][i] = clock64(); } while (0)
#else
#define TRACE(e, i) do {} while (0)
#endif

template <int D, int BS, int NT>
struct AttnCfg {
  static constexpr int kAtoms = D / 64;
  static constexpr int SB = BS < 64 ? BS : 64;      // keys per sub-block (one S MMA, one softmax step)
  static constexpr int SPB = BS / SB;               // sub-blocks per page
  static constexpr int kQBytes = 128 * D * 2;
  static constexpr int kKVBytes = BS * D * 2;
  static constexpr int kKStages = (BS * D >= 128 * 128) ? 3 : 4;
  static constexpr int kVStages = (BS * D >= 128 * 128) ? 2 : 4;
  static constexpr int kSoftmaxWarps = 4 * NT;
  static constexpr int kConvWarps = 2;             // bf16 -> fp16 in-place conversion of V tiles
  static constexpr int kThreads = (kSoftmaxWarps + kConvWarps + 2) * 32;
  static constexpr int kTmemCols = NT == 2 ? 512 : 256;
  static constexpr int kOCol0 = NT * 128;          // O_t at kOCol0 + t*128; S_t^b at t*128 + b*64
  static constexpr int kMaxList = NT == 1 ? 4096 : 0;  // block-sparse mode: the CTA's block list
  static constexpr int kSmem = NT * kQBytes + (kKStages + kVStages) * kKVBytes + 1024 + 512 + 4 * kMaxList;
  static_assert(kSmem <= 232448, "shared memory budget");
};

template <int D, int BS, int NT, bool PF16>
__global__ void __launch_bounds__(AttnCfg<D, BS, NT>::kThreads, 1)
    k_paged_attn(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, Geo g, AttnArgs args) {
  using Cfg = AttnCfg<D, BS, NT>;
  constexpr int SB = Cfg::SB, SPB = Cfg::SPB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + NT * Cfg::kQBytes;
  uint8_t* sV = sK + Cfg::kKStages * Cfg::kKVBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + Cfg::kVStages * Cfg::kKVBytes);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + Cfg::kKStages;
  uint64_t* v_full = k_empty + Cfg::kKStages;
  uint64_t* v_empty = v_full + Cfg::kVStages;
  uint64_t* v_ready = v_empty + Cfg::kVStages;  // [kVStages] V tile converted to fp16
  uint64_t* s_full = v_ready + Cfg::kVStages;   // [NT][2]
  uint64_t* p_full = s_full + 2 * NT;           // [NT][2] (per S buffer: the softmax may run 2 ahead)
  uint64_t* pv_done = p_full + 2 * NT;          // [NT]
  uint64_t* o_full = pv_done + NT;              // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);
  int* n_blocks_s = reinterpret_cast<int*>(tmem_slot + 1);
  int* row_start_s = n_blocks_s + 1;
  int* blist = row_start_s + 1;  // [Cfg::kMaxList]

  // ---- tile coordinates (heaviest q-tiles first)
  const int HP = g.E / NT;                     // head groups of NT per execution group
  const int nqt = (g.C + 127) / 128;
  const int per_qt = g.B * g.Gn * HP;
  const int qt = nqt - 1 - (int)blockIdx.x / per_qt;
  int rem = (int)blockIdx.x % per_qt;
  const int hp = rem % HP;
  rem /= HP;
  const int grp = rem % g.Gn;
  const int b = rem / g.Gn;
  const int p0 = qt * 128;
  const int h0 = grp * g.E + hp * NT;
  const int kvh = group_kv_head(g, grp);

  const uint32_t warp = warp_id(), lane = lane_id();
  constexpr uint32_t kConvWarp0 = Cfg::kSoftmaxWarps;
  constexpr uint32_t kTmaWarp = kConvWarp0 + Cfg::kConvWarps, kMmaWarp = kTmaWarp + 1;

  if (warp == kTmaWarp && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(q_full, 1);
    for (int s = 0; s < Cfg::kKStages; ++s) { mbar_init(k_full + s, 1); mbar_init(k_empty + s, 1); }
    for (int s = 0; s < Cfg::kVStages; ++s) {
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
      mbar_init(v_ready + s, Cfg::kConvWarps);
    }
    for (int t = 0; t < NT; ++t) {
      mbar_init(s_full + 2 * t, 1);
      mbar_init(s_full + 2 * t + 1, 1);
      mbar_init(p_full + 2 * t, 4);
      mbar_init(p_full + 2 * t + 1, 4);
      mbar_init(pv_done + t, 1);
    }
    mbar_init(o_full, 1);
    fence_barrier_init();
    // number of table entries this q-tile can see: ascending j with j*bs <= P + last query
    const int last_abs = g.P + min(p0 + 127, g.C - 1);
    const int jmax = last_abs / g.bs;
    const int r = b * g.Gn + grp;
    int start = 0, n = jmax + 1;
    if (args.indptr != nullptr) {
      start = args.indptr[r];
      const int end = args.indptr[r + 1];
      int lo = start, hi = end;  // first index with kv_indices > jmax
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (args.indices[mid] <= jmax) lo = mid + 1; else hi = mid;
      }
      n = lo - start;
    }
    *n_blocks_s = n;
    *row_start_s = start;
  }
  if constexpr (Cfg::kMaxList > 0) {
    // block-sparse execution: this CTA's tile (b, h0, q-block qt) runs
    // the blocks set in its own 2D mask row, interpreted here: warp-wide popc + exclusive scan of the
    // row's words (bits j <= jmax only), ascending block ids into shared memory.
    if (warp == kTmaWarp && args.mask != nullptr) {
      const int jmax = (g.P + min(p0 + 127, g.C - 1)) / g.bs;
      const int wmax = jmax >> 5;
      const uint32_t* mrow = args.mask + ((long long)(b * g.Hq + h0) * g.nqb + qt) * g.nwords;
      int base = 0;
      for (int w0 = 0; w0 <= wmax; w0 += 32) {
        const int w = w0 + (int)lane;
        uint32_t bits = 0;
        if (w <= wmax) {
          bits = __ldg(mrow + w);
          if (w == wmax && (jmax & 31) != 31) bits &= (2u << (jmax & 31)) - 1u;
        }
        const int c = __popc(bits);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if ((int)lane >= o) incl += y;
        }
        int pos = base + incl - c;
        while (bits) {
          blist[pos++] = w * 32 + __ffs(bits) - 1;
          bits &= bits - 1u;
        }
        base += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) {
        *n_blocks_s = base;
        *row_start_s = 0;
      }
    }
  }
  if (warp == kMmaWarp) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int N = *n_blocks_s;          // pages
  const int U = N * SPB;              // sub-blocks
  const int row_start = *row_start_s;
  // logical KV block of the CTA's n-th list entry
  auto block_of = [&](int n) -> int {
    if constexpr (Cfg::kMaxList > 0)
      if (args.mask != nullptr) return blist[n];
    return args.indptr != nullptr ? __ldg(args.indices + row_start + n) : n;
  };

  // TMA and MMA roles run on all 32 lanes with warp-uniform control flow (so descriptors and
  // coordinates live in uniform registers); one elected lane issues each TMA / tcgen05 instruction.
  if (warp == kTmaWarp) {
    if (N > 0) {  // ------------------------------------------------------------ TMA producer
      if (elect_one()) {
        mbar_expect_tx(q_full, NT * Cfg::kQBytes);
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int a = 0; a < Cfg::kAtoms; ++a)
            tma_load_4d(sQ + t * Cfg::kQBytes + a * 128 * 128, &tm_q, q_full, 64 * a, h0 + t, p0, b);
      }
      __syncwarp();
      const int32_t* ptab = args.page_table + (long long)b * g.maxb;
      for (int n = 0; n < N; ++n) {
        const int j = block_of(n);
        const int page = __ldg(ptab + j);
        const int ks = n % Cfg::kKStages, vs = n % Cfg::kVStages;
        mbar_wait(k_empty + ks, ((n / Cfg::kKStages) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(k_full + ks, Cfg::kKVBytes);
#pragma unroll
          for (int a = 0; a < Cfg::kAtoms; ++a)
            tma_load_4d(sK + ks * Cfg::kKVBytes + a * BS * 128, &tm_k, k_full + ks, 64 * a, 0, kvh, page);
        }
        __syncwarp();
        mbar_wait(v_empty + vs, ((n / Cfg::kVStages) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(v_full + vs, Cfg::kKVBytes);
#pragma unroll
          for (int a = 0; a < Cfg::kAtoms; ++a)
            tma_load_4d(sV + vs * Cfg::kKVBytes + a * BS * 128, &tm_v, v_full + vs, 64 * a, 0, kvh, page);
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    if (N > 0) {  // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, SB, 0, 0);
      // P (A, TMEM) and V (B, smem) are fp16 unless CPA_F_P_BF16: a/b formats [7,10)/[10,13) = 0 (f16)
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, 0, 1) & ~(PF16 ? ((7u << 7) | (7u << 10)) : 0u);
      const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
      // S_t(u) = Q_t K_(u)^T over SB keys into S_t^{u%2}; commit -> s_full[t][u%2]
      auto issue_s = [&](int t, int u) {
        const int n = u / SPB, h = u % SPB;
        const uint32_t d_tm = tmem + t * 128 + (u & 1) * 64;
        const uint32_t kb = k_base + (n % Cfg::kKStages) * Cfg::kKVBytes + h * SB * 128;
        if (elect_one()) {
#pragma unroll
          for (int a = 0; a < Cfg::kAtoms; ++a)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ad = umma_desc_sw128(q_base + t * Cfg::kQBytes + a * 128 * 128 + kk * 32, 16, 1024);
              const uint64_t bd = umma_desc_sw128(kb + a * BS * 128 + kk * 32, 16, 1024);
              mma_ss(d_tm, ad, bd, idesc_s, (a | kk) != 0);
            }
          tc_commit(s_full + 2 * t + (u & 1));
        }
        __syncwarp();
      };
      // O_t += P_t(u) V_(u): A = P in TMEM (fp16 pairs over S_t^{u%2}), B = V rows of the sub-block
      auto issue_pv = [&](int t, int u) {
        const int n = u / SPB, h = u % SPB;
        const uint32_t d_tm = tmem + Cfg::kOCol0 + t * 128;
        const uint32_t p_tm = tmem + t * 128 + (u & 1) * 64;
        const uint32_t vb = v_base + (n % Cfg::kVStages) * Cfg::kKVBytes + h * SB * 128;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < SB / 16; ++kk) {
            const uint64_t bd = umma_desc_sw128(vb + kk * 16 * 128, BS * 128, 1024);
            mma_ts(d_tm, p_tm + kk * 8, bd, idesc_o, (u > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(pv_done + t);
        }
        __syncwarp();
      };
      auto commit1 = [&](uint64_t* bar) {
        if (elect_one()) tc_commit(bar);
        __syncwarp();
      };
      auto wait_k = [&](int u) {  // first sub-block of a page: its K must have landed
        if (u % SPB == 0) {
          const int n = u / SPB;
          mbar_wait(k_full + n % Cfg::kKStages, (n / Cfg::kKStages) & 1);
          tc_fence_after();
        }
      };
      auto release_k = [&](int u) {  // after the last S of a page (both tiles) was issued
        if (u % SPB == SPB - 1) commit1(k_empty + (u / SPB) % Cfg::kKStages);
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int u = 0; u < 2 && u < U; ++u) {
        wait_k(u);
#pragma unroll
        for (int t = 0; t < NT; ++t) issue_s(t, u);
        release_k(u);
      }
      for (int u = 0; u < U; ++u) {
        const int n = u / SPB;
        if (u % SPB == 0) {
          mbar_wait(v_ready + n % Cfg::kVStages, (n / Cfg::kVStages) & 1);
          if (lane == 0) TRACE(1, n);
        }
        const bool more = u + 2 < U;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          mbar_wait(p_full + 2 * t + (u & 1), (u >> 1) & 1);
          if (lane == 0) TRACE(2, 2 * u + t);
          tc_fence_after();
          issue_pv(t, u);
          if (more) {
            if (t == 0) wait_k(u + 2);
            issue_s(t, u + 2);
          }
          if (lane == 0) TRACE(3, 2 * u + t);
        }
        if (u % SPB == SPB - 1) commit1(v_empty + n % Cfg::kVStages);
        if (more) release_k(u + 2);
      }
      commit1(o_full);
    }
  } else if (warp >= kConvWarp0) {  // --------------------------------------- V bf16 -> fp16
    // P is rounded to fp16 (2^-11) instead of bf16 (2^-8); tcgen05 kind::f16 needs A and B of one
    // type, so each landed V tile is converted in place (same swizzled layout: elementwise).
    const int ct = (warp - kConvWarp0) * 32 + lane;
    for (int n = 0; n < N; ++n) {
      const int vs = n % Cfg::kVStages;
      mbar_wait(v_full + vs, (n / Cfg::kVStages) & 1);
      if (PF16 && !(g.flags & (1u << 12))) {  // CPA_F_V_F16: the pool already holds fp16 V
        uint4* tile = reinterpret_cast<uint4*>(sV + vs * Cfg::kKVBytes);
#pragma unroll 4
        for (int x = ct; x < Cfg::kKVBytes / 16; x += Cfg::kConvWarps * 32) {
          uint4 w = tile[x];
          w.x = bf16x2_to_f16x2(w.x);
          w.y = bf16x2_to_f16x2(w.y);
          w.z = bf16x2_to_f16x2(w.z);
          w.w = bf16x2_to_f16x2(w.w);
          tile[x] = w;
        }
        fence_proxy_async_smem();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(v_ready + vs);
    }
  } else {  // ------------------------------------------------------------------ softmax / epilogue
    const int t = warp / 4;           // Q tile of this warpgroup
    const int quarter = warp & 3;     // TMEM lane quarter
    const int row = quarter * 32 + lane;
    const int p = p0 + row;           // chunk position of this thread's query row
    const int h = h0 + t;
    const int lim = min(g.P + p, g.L - 1);  // last visible absolute key
    const float sl2 = g.scale * 1.4426950408889634f;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t o_tm = tmem + lane_off + Cfg::kOCol0 + t * 128;
    constexpr int CH = SB >= 32 ? 32 : SB;
    constexpr int NCH = SB / CH;
    float m_run = -INFINITY, l_run = 0.f;
    int j = 0;
    for (int u = 0; u < U; ++u) {
      if (u % SPB == 0) j = block_of(u / SPB);
      const uint32_t s_tm = tmem + lane_off + t * 128 + (u & 1) * 64;
      if (row == 0) TRACE(4, 2 * u + t);
      mbar_wait(s_full + 2 * t + (u & 1), (u >> 1) & 1);
      if (row == 0) TRACE(5, 2 * u + t);
      tc_fence_after();
      uint32_t sv[NCH][CH];
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        if constexpr (CH == 32) tmem_ld32(s_tm + k * CH, sv[k]);
        else tmem_ld16(s_tm + k * CH, sv[k]);
      }
      tmem_wait_ld();
      const int tbase = j * g.bs + (u % SPB) * SB;
      if (tbase + SB - 1 > g.P + p0) {  // sub-block crosses the causal diagonal of this tile
#pragma unroll
        for (int k = 0; k < NCH; ++k)
#pragma unroll
          for (int c = 0; c < CH; ++c)
            if (tbase + k * CH + c > lim) sv[k][c] = __float_as_uint(-INFINITY);
      }
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int k = 0; k < NCH; ++k)
#pragma unroll
        for (int c = 0; c < CH; c += 8)
#pragma unroll
          for (int w4 = 0; w4 < 4; ++w4)
            m4[w4] = fmax3(m4[w4], __uint_as_float(sv[k][c + 2 * w4]), __uint_as_float(sv[k][c + 2 * w4 + 1]));
      const float m_blk = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * sl2;
      float f = 1.f;
      const bool rescale = m_blk > m_run + 8.0f;  // lazy rescale (first sub-block always lands here)
      if (rescale) {
        if (u > 0) f = fast_exp2(m_run - m_blk);
        m_run = m_blk;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      if (row == 0) TRACE(11, 2 * u + t);
      // P = exp2(s*sl2 - m): packed f32x2 FFMA; pairs selected by use_poly_exp go through a degree-3
      // polynomial on the FMA pipe (MUFU offload), the rest through MUFU.EX2; 4 independent f32x2
      // partial sums; each chunk is packed (fp16) and stored over S in TMEM.
      float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        uint32_t pk[CH / 2];
#pragma unroll
        for (int q2 = 0; q2 < CH / 2; ++q2) {
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
        if constexpr (CH == 32) tmem_st16(s_tm + k * CH / 2, *reinterpret_cast<uint32_t(*)[16]>(pk));
        else tmem_st8(s_tm + k * CH / 2, *reinterpret_cast<uint32_t(*)[8]>(pk));
      }
      const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
      l_run = l_run * f + ((a01.x + a01.y) + (a23.x + a23.y));
      if (row == 0) TRACE(12, 2 * u + t);
      // tcgen05.ld/st are warp-collective: rescale O when any row of the warp needs it (f = 1 else),
      // after PV_t(u-1) has completed and before PV_t(u) is issued (it waits on p_full below).
      if (__any_sync(0xffffffffu, rescale && u > 0)) {
        mbar_wait(pv_done + t, (u - 1) & 1);
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
      if (lane == 0) mbar_arrive(p_full + 2 * t + (u & 1));
      if (row == 0) TRACE(6, 2 * u + t);
    }
    // ---- epilogue: O = O_acc / l
    const bool store = p < g.C;
    const float inv_l = (U > 0 && l_run > 0.f) ? 1.0f / l_run : 0.f;
    if (U > 0) {
      mbar_wait(o_full, 0);
      tc_fence_after();
    }
    const long long obase = (long long)b * args.o_bstride + (long long)p * args.o_stride + (long long)h * D;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t o[32];
      if (U > 0) {
        tmem_ld32(o_tm + c0, o);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = 0u;
      }
      float v[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = __uint_as_float(o[c]) * inv_l;
      if (store) store_o_row32(args, obase + c0, v);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
}

// ---------------------------------------------------------------- launcher
template <int D, int BS, int NT, bool PF16>
static cudaError_t launch_attn_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                                 const Geo& g, const AttnArgs& a, cudaStream_t st) {
  using Cfg = AttnCfg<D, BS, NT>;
  auto kern = k_paged_attn<D, BS, NT, PF16>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
  if (e != cudaSuccess) return e;
  const int nqt = (g.C + 127) / 128;
  const int grid = nqt * g.B * g.Gn * (g.E / NT);
  kern<<<grid, Cfg::kThreads, Cfg::kSmem, st>>>(tq, tk, tv, g, a);
  return cudaGetLastError();
}

cudaError_t launch_paged_attention(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                                   const Geo& g, const AttnArgs& a, cudaStream_t st, int* launches) {
  ++*launches;
  const bool pair = (g.E % 2) == 0 && a.mask == nullptr;  // block-sparse: one head per CTA
#define CPA_AT(DD, BB)                                                        \
  if (g.d == DD && g.bs == BB) {                                              \
    if (g.flags & (1u << 8))                                                  \
      return pair ? launch_attn_t<DD, BB, 2, false>(tq, tk, tv, g, a, st)     \
                  : launch_attn_t<DD, BB, 1, false>(tq, tk, tv, g, a, st);    \
    return pair ? launch_attn_t<DD, BB, 2, true>(tq, tk, tv, g, a, st)        \
                : launch_attn_t<DD, BB, 1, true>(tq, tk, tv, g, a, st);       \
  }
  CPA_AT(64, 16) CPA_AT(64, 32) CPA_AT(64, 64) CPA_AT(64, 128)
  CPA_AT(128, 16) CPA_AT(128, 32) CPA_AT(128, 64) CPA_AT(128, 128)
#undef CPA_AT
  return cudaErrorInvalidValue;
}

}  // namespace cpa

#ifdef CPA_TRACE
extern "C" __attribute__((visibility("default"))) int cpa_debug_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, cpa::g_trace, sizeof(cpa::g_trace));
}
#endif
