// attention.cu -- §8 row a6: zero-copy paged attention over the tabled KV blocks, tcgen05/TMEM.
//
// each (batch b, execution group g) attends only to the blocks
// T[b,g] listed in kv_indices, read in place from the paged cache; causal masking is done in
// ABSOLUTE positions (query p at P+p sees keys t <= P+p) so the fully-open current chunk keeps
// causal semantics.  Value:
//   O[b,p,h] = sum_{t in A(p)} softmax_t(scale q_p.k_t) v_t,  A(p) = {t : t/bs in T[b,h/E], t <= P+p}.
//
// CTA = (b, g, 128-token q-tile, pair of query heads of g) -> NT=2 Q tiles of 128 rows that
// share every K/V page (GQA packing), FA4-style ping-pong:
//   warps 0-3  softmax for tile 0 (one TMEM lane = one query row per thread)
//   warps 4-7  softmax for tile 1
//   warps 8-9  V converter: each landed bf16 V tile -> fp16 in place (P.V runs in fp16, DESIGN K3)
//   warp  10   TMA producer: kv_indices -> page_table -> cp.async.bulk.tensor K/V pages
//   warp  11   TMEM allocator + single-thread tcgen05.mma issuer
// TMEM columns: S0 [0,128) S1 [128,256) O0 [256,256+d) O1 [384,384+d); P_t (bf16) aliases S_t.
// MMA order per KV block n: PV0(n), S0(n+1), PV1(n), S1(n+1) -- softmax of one tile overlaps the
// tensor-core work of the other. Online softmax in the log2 domain with lazy rescaling of O
// (only when the running max grows by > 8, i.e. P <= 256, fp32 accumulators).
#include "common.cuh"
#include "geo.cuh"

namespace cpa {

template <int D, int BS, int NT>
struct AttnCfg {
  static constexpr int kAtoms = D / 64;
  static constexpr int kQBytes = 128 * D * 2;
  static constexpr int kKVBytes = BS * D * 2;
  static constexpr int kKStages = (BS * D >= 128 * 128) ? 3 : 4;
  static constexpr int kVStages = (BS * D >= 128 * 128) ? 2 : 4;
  static constexpr int kSoftmaxWarps = 4 * NT;
  static constexpr int kConvWarps = 2;             // bf16 -> fp16 in-place conversion of V tiles
  static constexpr int kThreads = (kSoftmaxWarps + kConvWarps + 2) * 32;
  static constexpr int kTmemCols = NT == 2 ? 512 : 256;
  static constexpr int kSCol0 = 0;                 // S_t at t*128
  static constexpr int kOCol0 = NT * 128;          // O_t at kOCol0 + t*128
  static constexpr int kSmem = NT * kQBytes + (kKStages + kVStages) * kKVBytes + 1024 + 512;
  static_assert(kSmem <= 232448, "shared memory budget");
};

struct AttnArgs {
  const int32_t* page_table;
  const int32_t* indptr;   // nullptr => dense (all blocks)
  const int32_t* indices;
  void* out;
  int out_f32;
};

template <int D, int BS, int NT>
__global__ void __launch_bounds__(AttnCfg<D, BS, NT>::kThreads, 1)
    k_paged_attn(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, Geo g, AttnArgs args) {
  using Cfg = AttnCfg<D, BS, NT>;
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
  uint64_t* s_full = v_ready + Cfg::kVStages;   // [NT]
  uint64_t* p_full = s_full + NT;               // [NT]
  uint64_t* o_full = p_full + NT;               // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);
  int* n_blocks_s = reinterpret_cast<int*>(tmem_slot + 1);
  int* row_start_s = n_blocks_s + 1;

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
  const bool p_bf16 = (g.flags & (1u << 8)) != 0;  // ablation: bf16 P with the bf16 V as stored

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
    for (int t = 0; t < NT; ++t) { mbar_init(s_full + t, 1); mbar_init(p_full + t, 4); }
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
  if (warp == kMmaWarp) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int N = *n_blocks_s;
  const int row_start = *row_start_s;

  if (warp == kTmaWarp) {
    if (lane == 0 && N > 0) {  // ------------------------------------------------ TMA producer
      mbar_expect_tx(q_full, NT * Cfg::kQBytes);
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int a = 0; a < Cfg::kAtoms; ++a)
          tma_load_4d(sQ + t * Cfg::kQBytes + a * 128 * 128, &tm_q, q_full, 64 * a, h0 + t, p0, b);
      const int32_t* ptab = args.page_table + (long long)b * g.maxb;
      for (int n = 0; n < N; ++n) {
        const int j = args.indptr != nullptr ? __ldg(args.indices + row_start + n) : n;
        const int page = __ldg(ptab + j);
        const int ks = n % Cfg::kKStages, vs = n % Cfg::kVStages;
        mbar_wait(k_empty + ks, ((n / Cfg::kKStages) & 1) ^ 1);
        mbar_expect_tx(k_full + ks, Cfg::kKVBytes);
#pragma unroll
        for (int a = 0; a < Cfg::kAtoms; ++a)
          tma_load_4d(sK + ks * Cfg::kKVBytes + a * BS * 128, &tm_k, k_full + ks, 64 * a, 0, kvh, page);
        mbar_wait(v_empty + vs, ((n / Cfg::kVStages) & 1) ^ 1);
        mbar_expect_tx(v_full + vs, Cfg::kKVBytes);
#pragma unroll
        for (int a = 0; a < Cfg::kAtoms; ++a)
          tma_load_4d(sV + vs * Cfg::kKVBytes + a * BS * 128, &tm_v, v_full + vs, 64 * a, 0, kvh, page);
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0 && N > 0) {  // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, BS, 0, 0);
      // P (A, TMEM) and V (B, smem) are fp16 unless CPA_F_P_BF16: a/b formats [7,10)/[10,13) = 0 (f16)
      const uint32_t idesc_o = umma_idesc_bf16(128, D, 0, 1) & ~(p_bf16 ? 0u : ((7u << 7) | (7u << 10)));
      const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
      auto issue_s = [&](int t, int ks) {
        const uint32_t d_tm = tmem + Cfg::kSCol0 + t * 128;
#pragma unroll
        for (int a = 0; a < Cfg::kAtoms; ++a)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = umma_desc_sw128(q_base + t * Cfg::kQBytes + a * 128 * 128 + kk * 32, 16, 1024);
            const uint64_t bd = umma_desc_sw128(k_base + ks * Cfg::kKVBytes + a * BS * 128 + kk * 32, 16, 1024);
            mma_ss(d_tm, ad, bd, idesc_s, (a | kk) != 0);
          }
      };
      auto issue_pv = [&](int t, int vs, int n) {
        const uint32_t d_tm = tmem + Cfg::kOCol0 + t * 128;
        const uint32_t p_tm = tmem + Cfg::kSCol0 + t * 128;
#pragma unroll
        for (int kk = 0; kk < BS / 16; ++kk) {
          const uint64_t bd = umma_desc_sw128(v_base + vs * Cfg::kKVBytes + kk * 16 * 128, BS * 128, 1024);
          mma_ts(d_tm, p_tm + kk * 8, bd, idesc_o, (n > 0 || kk > 0) ? 1u : 0u);
        }
      };
      mbar_wait(q_full, 0);
      mbar_wait(k_full + 0, 0);
      tc_fence_after();
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        issue_s(t, 0);
        tc_commit(s_full + t);
      }
      tc_commit(k_empty + 0);
      for (int n = 0; n < N; ++n) {
        const int vs = n % Cfg::kVStages;
        const int ks1 = (n + 1) % Cfg::kKStages;
        const bool more = n + 1 < N;
        mbar_wait(v_ready + vs, (n / Cfg::kVStages) & 1);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          mbar_wait(p_full + t, n & 1);
          tc_fence_after();
          issue_pv(t, vs, n);
          if (more) {
            if (t == 0) {
              mbar_wait(k_full + ks1, ((n + 1) / Cfg::kKStages) & 1);
              tc_fence_after();
            }
            issue_s(t, ks1);
            tc_commit(s_full + t);
          }
        }
        tc_commit(v_empty + vs);
        if (more) tc_commit(k_empty + ks1);
      }
      tc_commit(o_full);
    }
  } else if (warp >= kConvWarp0) {  // --------------------------------------- V bf16 -> fp16
    // P is rounded to fp16 (2^-11) instead of bf16 (2^-8); tcgen05 kind::f16 needs A and B of one
    // type, so each landed V tile is converted in place (same swizzled layout: elementwise).
    const int ct = (warp - kConvWarp0) * 32 + lane;
    for (int n = 0; n < N; ++n) {
      const int vs = n % Cfg::kVStages;
      mbar_wait(v_full + vs, (n / Cfg::kVStages) & 1);
      if (!p_bf16) {
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
    const uint32_t s_tm = tmem + lane_off + Cfg::kSCol0 + t * 128;
    const uint32_t o_tm = tmem + lane_off + Cfg::kOCol0 + t * 128;
    float m_run = -INFINITY, l_run = 0.f;
    for (int n = 0; n < N; ++n) {
      const int j = args.indptr != nullptr ? __ldg(args.indices + row_start + n) : n;
      mbar_wait(s_full + t, n & 1);
      tc_fence_after();
      uint32_t s[BS];
      if constexpr (BS >= 32) {
#pragma unroll
        for (int c0 = 0; c0 < BS; c0 += 32) tmem_ld32(s_tm + c0, *reinterpret_cast<uint32_t(*)[32]>(s + c0));
      } else {
        tmem_ld16(s_tm, *reinterpret_cast<uint32_t(*)[16]>(s));
      }
      tmem_wait_ld();
      const int tbase = j * g.bs;
      if (tbase + BS - 1 > g.P + p0) {  // block crosses the causal diagonal of this tile
#pragma unroll
        for (int c = 0; c < BS; ++c)
          if (tbase + c > lim) s[c] = __float_as_uint(-INFINITY);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < BS; ++c) mx = fmaxf(mx, __uint_as_float(s[c]));
      const float m_blk = mx * sl2;
      float f = 1.f;
      const bool rescale = m_blk > m_run + 8.0f;  // lazy rescale (first block always lands here)
      if (rescale) {
        if (n > 0) f = fast_exp2(m_run - m_blk);
        m_run = m_blk;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      float lsum = 0.f;
      uint32_t pk[BS / 2];
#pragma unroll
      for (int c = 0; c < BS; c += 2) {
        const float e0 = fast_exp2(fmaf(__uint_as_float(s[c]), sl2, -m_use));
        const float e1 = fast_exp2(fmaf(__uint_as_float(s[c + 1]), sl2, -m_use));
        lsum += e0 + e1;
        pk[c / 2] = p_bf16 ? pack_bf16x2(e0, e1) : pack_f16x2(e0, e1);
      }
      l_run = l_run * f + lsum;
      if constexpr (BS >= 32) {
#pragma unroll
        for (int c0 = 0; c0 < BS / 2; c0 += 16) tmem_st16(s_tm + c0, *reinterpret_cast<uint32_t(*)[16]>(pk + c0));
      } else {
        tmem_st8(s_tm, *reinterpret_cast<uint32_t(*)[8]>(pk));
      }
      // tcgen05.ld/st are warp-collective: rescale O when any row of the warp needs it (f = 1 else)
      if (__any_sync(0xffffffffu, rescale && n > 0)) {  // PV_t(n-1) complete (implied by s_full)
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
      if (lane == 0) mbar_arrive(p_full + t);
    }
    // ---- epilogue: O = O_acc / l
    const bool store = p < g.C;
    const float inv_l = (N > 0 && l_run > 0.f) ? 1.0f / l_run : 0.f;
    if (N > 0) {
      mbar_wait(o_full, 0);
      tc_fence_after();
    }
    const long long obase = ((long long)b * g.C + p) * g.q_stride + (long long)h * D;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t o[32];
      if (N > 0) {
        tmem_ld32(o_tm + c0, o);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = 0u;
      }
      if (store) {
        if (args.out_f32) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(args.out) + obase + c0);
#pragma unroll
          for (int c = 0; c < 32; c += 4)
            dst[c / 4] = make_float4(__uint_as_float(o[c]) * inv_l, __uint_as_float(o[c + 1]) * inv_l,
                                     __uint_as_float(o[c + 2]) * inv_l, __uint_as_float(o[c + 3]) * inv_l);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(args.out) + obase + c0);
#pragma unroll
          for (int c = 0; c < 32; c += 8)
            dst[c / 8] = make_uint4(pack_bf16x2(__uint_as_float(o[c]) * inv_l, __uint_as_float(o[c + 1]) * inv_l),
                                    pack_bf16x2(__uint_as_float(o[c + 2]) * inv_l, __uint_as_float(o[c + 3]) * inv_l),
                                    pack_bf16x2(__uint_as_float(o[c + 4]) * inv_l, __uint_as_float(o[c + 5]) * inv_l),
                                    pack_bf16x2(__uint_as_float(o[c + 6]) * inv_l, __uint_as_float(o[c + 7]) * inv_l));
        }
      }
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
template <int D, int BS, int NT>
static cudaError_t launch_attn_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                                 const Geo& g, const AttnArgs& a, cudaStream_t st) {
  using Cfg = AttnCfg<D, BS, NT>;
  auto kern = k_paged_attn<D, BS, NT>;
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
  const bool pair = (g.E % 2) == 0;
#define CPA_AT(DD, BB)                                                        \
  if (g.d == DD && g.bs == BB) {                                              \
    return pair ? launch_attn_t<DD, BB, 2>(tq, tk, tv, g, a, st)              \
                : launch_attn_t<DD, BB, 1>(tq, tk, tv, g, a, st);             \
  }
  CPA_AT(64, 16) CPA_AT(64, 32) CPA_AT(64, 64) CPA_AT(64, 128)
  CPA_AT(128, 16) CPA_AT(128, 32) CPA_AT(128, 64) CPA_AT(128, 128)
#undef CPA_AT
  return cudaErrorInvalidValue;
}

}  // namespace cpa
