// api.cu -- the C ABI of libcpa.so (include/cpa.h): validation, workspace carving, TMA tensor
// maps and the stream-ordered kernel sequence of one CompactAttention chunk step.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <mutex>

#include "../../include/cpa.h"
#include "common.cuh"
#include "geo.cuh"

namespace cpa {
cudaError_t launch_pool_q(const __nv_bfloat16* q, const Geo& g, __nv_bfloat16* qbar, int* mstar_key,
                          unsigned* tables_done, bool after_append, cudaStream_t st, int* launches);
cudaError_t launch_block_scores(const CUtensorMap& tq, const CUtensorMap& tk, const int32_t* pt,
                                const Geo& g, float* scores, int* mstar_key, int num_sms,
                                cudaStream_t st, int* launches);
cudaError_t launch_block_scores_exact(const CUtensorMap& tq, const CUtensorMap& tk, const int32_t* pt,
                                      const Geo& g, float* scores, int* mstar_key, int num_sms, cudaStream_t st,
                                      int* launches);
cudaError_t launch_tables(const float* scores, const int* mstar_key, const Geo& g,
                          const uint32_t* mask_in, uint32_t* mask_out, uint32_t* gwords,
                          int* dev_status, unsigned* done, int32_t* indptr, int32_t* indices, cudaStream_t st,
                          int* launches);
cudaError_t launch_paged_attention(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                                   const Geo& g, const AttnArgs& a, cudaStream_t st, int* launches);
bool attn_2cta_supported(const Geo& g);
bool attn_rs_supported(const Geo& g);
cudaError_t launch_paged_attention_rs(const CUtensorMap& tq, const CUtensorMap& tk_half, const CUtensorMap& tv,
                                      const Geo& g, const AttnArgs& a, cudaStream_t st, int* launches);
int attn_2cta_max_clusters(const Geo& g);
bool attn_ks4_supported(const Geo& g);
cudaError_t launch_paged_attention_ks4(const CUtensorMap& tq, const CUtensorMap& tk_half, const CUtensorMap& tv,
                                       const Geo& g, const AttnArgs& a, cudaStream_t st, int* launches);
cudaError_t launch_paged_attention_2cta(const CUtensorMap& tq, const CUtensorMap& tk_half, const CUtensorMap& tv,
                                        const Geo& g, const AttnArgs& a, const SkSched* sk, cudaStream_t st,
                                        int* launches);
cudaError_t launch_append(const void* kc, const void* vc, const cpa_kv_cache& c, const Geo& g,
                          long long page_stride, long long head_stride, int num_sms, cudaStream_t st, int* launches);
cudaError_t launch_gather_pages(const cpa_kv_cache& c, const int32_t* indptr, const int32_t* indices, const Geo& g,
                                long long ps, long long hs, void* ck, void* cv, int32_t* cpt, cudaStream_t st,
                                int* launches);
cudaError_t launch_expand_tables(const int32_t* indptr, const int32_t* indices, const Geo& g, uint32_t* mask,
                                 cudaStream_t st, int* launches);
cudaError_t launch_row_max(const int* mstar_key, const Geo& g, float* row_max, cudaStream_t st,
                           int* launches);
cudaError_t launch_peer_barrier(const PeerSig& s, cudaStream_t st, int* launches);
}  // namespace cpa

using namespace cpa;

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(CPA_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

// ---------------------------------------------------------------- device properties
struct DevInfo {
  int ok = -1;  // -1 unknown, 0 unsupported, 1 sm_100
  int num_sms = 0;
};
DevInfo g_dev[64];
std::mutex g_dev_mu;

int device_info(int* num_sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(CPA_ERR_UNSUPPORTED, "device index %d", dev);
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DevInfo& d = g_dev[dev];
  if (d.ok < 0) {
    int major = 0, minor = 0, sms = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    d.ok = (major == 10 && minor == 0) ? 1 : 0;
    d.num_sms = sms;
  }
  if (!d.ok) return fail(CPA_ERR_UNSUPPORTED, "libcpa needs an sm_100 (B200) device");
  *num_sms = d.num_sms;
  return CPA_OK;
}

// ---------------------------------------------------------------- TMA tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int make_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims,
             const cuuint64_t* strides_bytes, const cuuint32_t* box, const char* what) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(CPA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides_bytes,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CPA_ERR_CUDA, "cuTensorMapEncodeTiled(%s) failed: %d", what, (int)r);
  return CPA_OK;
}

// ---------------------------------------------------------------- validation -> Geo
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int make_geo(const cpa_params* p, Geo* g) {
  if (!p) return fail(CPA_ERR_NULL, "params is NULL");
  if (p->batch < 1 || p->num_q_heads < 1 || p->num_kv_heads < 1 || p->chunk_len < 1 || p->prefix_len < 0)
    return fail(CPA_ERR_SHAPE, "batch/heads/chunk_len must be >= 1 and prefix_len >= 0");
  if (p->num_q_heads % p->num_kv_heads)
    return fail(CPA_ERR_SHAPE, "num_q_heads %% num_kv_heads != 0");
  const int kvq = p->num_q_heads / p->num_kv_heads;
  const int E = p->exec_group_size ? p->exec_group_size : kvq;
  if (E < 1 || kvq % E) return fail(CPA_ERR_SHAPE, "exec_group_size must divide Hq/Hkv");
  if (p->head_dim != 64 && p->head_dim != 128) return fail(CPA_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  const int bs = p->block_size;
  if (bs != 16 && bs != 32 && bs != 64 && bs != 128)
    return fail(CPA_ERR_UNSUPPORTED, "block_size must be 16, 32, 64 or 128");
  if (p->prefix_len % bs) return fail(CPA_ERR_MISALIGNED, "prefix_len %% block_size != 0");
  if (!(p->alpha > 0.f && p->alpha <= 1.f)) return fail(CPA_ERR_ALPHA, "alpha must be in (0, 1]");
  if ((p->flags & CPA_F_V_F16) && (p->flags & CPA_F_P_BF16))
    return fail(CPA_ERR_UNSUPPORTED, "CPA_F_V_F16 needs fp16 P (not CPA_F_P_BF16)");
  const long long qs = p->q_token_stride ? p->q_token_stride : (long long)p->num_q_heads * p->head_dim;
  if (qs < (long long)p->num_q_heads * p->head_dim || qs % 8)
    return fail(CPA_ERR_MISALIGNED, "q_token_stride must be >= Hq*d and a multiple of 8");
  g->B = p->batch;
  g->Hq = p->num_q_heads;
  g->Hkv = p->num_kv_heads;
  g->d = p->head_dim;
  g->bs = bs;
  g->E = E;
  g->Gn = p->num_q_heads / E;
  g->C = p->chunk_len;
  g->P = p->prefix_len;
  g->L = g->P + g->C;
  g->nqb = (g->C + bs - 1) / bs;
  g->nkvb = (g->L + bs - 1) / bs;
  g->pb = g->P / bs;
  g->nwords = (g->nkvb + 31) / 32;
  g->R = E * g->nqb;
  g->Rpad = ((g->R + 127) / 128) * 128;
  g->maxb = 0;
  g->kv_per_q = kvq;
  g->scale = p->sm_scale > 0.f ? p->sm_scale : 1.0f / sqrtf((float)p->head_dim);
  g->ln_alpha = logf(p->alpha);
  g->flags = p->flags;
  g->q_stride = qs;
  g->b_stride = (long long)g->C * qs;
  return CPA_OK;
}

int check_cache(const cpa_kv_cache* c, Geo* g, long long* ps, long long* hs) {
  if (!c || !c->k_pages || !c->v_pages || !c->page_table) return fail(CPA_ERR_NULL, "cache pointers");
  if (!aligned16(c->k_pages) || !aligned16(c->v_pages)) return fail(CPA_ERR_MISALIGNED, "pages not 16B aligned");
  if (c->max_blocks_per_seq < g->nkvb)
    return fail(CPA_ERR_SHAPE, "max_blocks_per_seq %d < nkvb %d", c->max_blocks_per_seq, g->nkvb);
  if (c->num_pages < 1) return fail(CPA_ERR_SHAPE, "num_pages < 1");
  *hs = c->head_stride ? c->head_stride : (long long)g->bs * g->d;
  *ps = c->page_stride ? c->page_stride : (long long)g->Hkv * g->bs * g->d;
  if (*hs % 8 || *ps % 8) return fail(CPA_ERR_MISALIGNED, "page/head strides must be multiples of 8");
  g->maxb = c->max_blocks_per_seq;
  return CPA_OK;
}

// workspace carve-up
struct WS {
  __nv_bfloat16* qbar;
  float* scores;
  int* mstar_key;
  uint32_t* gwords;
  unsigned* done;  // k_mask_union's last-CTA counter
  size_t total;
};
size_t up256(size_t x) { return (x + 255) & ~size_t(255); }
WS carve(const Geo& g, void* base) {
  WS w;
  const uintptr_t p = reinterpret_cast<uintptr_t>(base);
  size_t off = 0;
  w.qbar = reinterpret_cast<__nv_bfloat16*>(p + off);
  off += up256((size_t)2 * g.B * g.Gn * g.Rpad * g.d * 2);
  w.scores = reinterpret_cast<float*>(p + off);
  off += up256((size_t)g.B * g.Gn * g.nkvb * g.Rpad * 4);
  w.mstar_key = reinterpret_cast<int*>(p + off);
  off += up256((size_t)g.B * g.Gn * g.Rpad * 4);
  w.gwords = reinterpret_cast<uint32_t*>(p + off);
  off += up256((size_t)g.B * g.Gn * g.nwords * 4);
  w.done = reinterpret_cast<unsigned*>(p + off);
  off += 256;
  w.total = off;
  return w;
}

// Persistent stream-K attention (attention_2cta.cu). Its workspace (schedule + partial slots) is
// carved from the start of ws: the chunk step runs the estimator first, so both stages share one
// buffer. kSkMaxClusters bounds the persistent grid (B200: 74 co-resident SM pairs).
// Policy: the per-unit grid already keeps every SM pair busy when the unit count fills whole waves
// (128K, one GPU: 512 units = 6.92 waves of 74, 98.8%); stream-K pays off when it does not (one KV
// group per GPU: 64 units on 74 pairs, 86%) and the (b, group) segments are few (every segment
// boundary costs partial outputs: 2 per cluster per segment).
constexpr int kSkMaxClusters = 80;
static_assert(kSkFixStride - 2 >= kSkMaxClusters, "fixup part list holds one part per cluster");
constexpr int kSkMaxSegments = 4;
int sk_units(const Geo& g) { return (g.C + 127) / 128 * g.B * g.Gn * (g.E / 2); }
int sk_segments(const Geo& g) { return g.B * g.Gn; }
bool sk_wanted(const Geo& g, int clusters) {
  if (g.flags & CPA_F_PERSIST) return sk_segments(g) <= kSkMaxSegments;
  // short KV (< 64K tokens): shares are too short to amortise the per-item epilogue (measured:
  // 32K, 2 KV groups, 8% slower than the per-unit grid; 128K, 1 KV group, 10% faster)
  if (sk_segments(g) > kSkMaxSegments || g.nkvb < 512) return false;
  const double waves = (double)sk_units(g) / clusters;
  return waves / ceil(waves) < 0.9;
}
size_t attn_ws_bytes(const Geo& g) {
  if (sk_segments(g) > kSkMaxSegments) return 0;
  const size_t U = (size_t)sk_units(g), slots = (size_t)kSkMaxClusters * sk_segments(g) * 2;
  return 4 * up256((U + 1) * 4) + up256(slots * 256 * g.d * 4) + up256(slots * 256 * 2 * 4) +
         up256((size_t)kSkMaxClusters * sk_segments(g) * kSkFixStride * 4);
}
SkSched carve_sk(const Geo& g, void* base, int clusters) {
  SkSched s;
  const size_t U = (size_t)sk_units(g);
  uint8_t* p = reinterpret_cast<uint8_t*>(base);
  s.pre = reinterpret_cast<int*>(p);
  p += up256((U + 1) * 4);
  s.len = reinterpret_cast<int*>(p);
  p += up256((U + 1) * 4);
  s.start = reinterpret_cast<int*>(p);
  p += up256((U + 1) * 4);
  s.nd = reinterpret_cast<int*>(p);
  p += up256((U + 1) * 4);
  const size_t slots = (size_t)kSkMaxClusters * sk_segments(g) * 2;
  s.part_o = reinterpret_cast<float*>(p);
  p += up256(slots * 256 * g.d * 4);
  s.part_ml = reinterpret_cast<float*>(p);
  p += up256(slots * 256 * 2 * 4);
  s.fix = reinterpret_cast<int*>(p);
  s.units = (int)U;
  s.clusters = clusters;
  s.segments = sk_segments(g);
  s.seg_units = (int)U / s.segments;
  return s;
}

int q_map(CUtensorMap* m, const void* q, const Geo& g) {
  cuuint64_t dims[4] = {(cuuint64_t)g.d, (cuuint64_t)g.Hq, (cuuint64_t)g.C, (cuuint64_t)g.B};
  cuuint64_t str[3] = {(cuuint64_t)g.d * 2, (cuuint64_t)g.q_stride * 2, (cuuint64_t)g.b_stride * 2};
  cuuint32_t box[4] = {64, 1, 128, 1};
  return make_map(m, q, 4, dims, str, box, "q");
}
int kv_map(CUtensorMap* m, const void* pages, const Geo& g, int num_pages, long long ps, long long hs,
           const char* what, int box_rows = 0) {
  cuuint64_t dims[4] = {(cuuint64_t)g.d, (cuuint64_t)g.bs, (cuuint64_t)g.Hkv, (cuuint64_t)num_pages};
  cuuint64_t str[3] = {(cuuint64_t)g.d * 2, (cuuint64_t)hs * 2, (cuuint64_t)ps * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)(box_rows ? box_rows : g.bs), 1, 1};
  return make_map(m, pages, 4, dims, str, box, what);
}

// ---------------------------------------------------------------- plans
// Every entry point validates and encodes its TMA descriptors (prep_*) BEFORE the first launch, so a
// synchronous validation error leaves every output (pages, tables, o) untouched (cpa.h conventions).
struct TablesPlan {
  CUtensorMap tq, tk, tqq;
  WS w;
  float* scores;
  bool mask_in, exact, scores_out;
  const void* q;
  const int32_t* page_table;
  cpa_tables t;
  int num_sms;
};

int prep_tables(const cpa_params* p, const Geo& g, const void* q, const cpa_kv_cache* c, long long ps,
                long long hs, const cpa_tables* out, void* ws, size_t ws_bytes, int num_sms, TablesPlan* tp) {
  if (!out || !out->kv_indptr || !out->kv_indices) return fail(CPA_ERR_NULL, "tables pointers");
  if (out->capacity < (long long)g.B * g.Gn * g.nkvb)
    return fail(CPA_ERR_CAPACITY, "capacity %lld < B*Gn*nkvb = %lld", (long long)out->capacity,
                (long long)g.B * g.Gn * g.nkvb);
  tp->mask_in = (p->flags & CPA_F_MASK_IN) != 0;
  tp->exact = (p->flags & CPA_F_EXACT_SCORES) != 0;
  tp->scores_out = (p->flags & CPA_F_SCORES_OUT) != 0;
  if (tp->mask_in && !out->mask_bits) return fail(CPA_ERR_NULL, "CPA_F_MASK_IN needs tables->mask_bits");
  if ((p->flags & CPA_F_MASK_OUT) && !out->mask_bits) return fail(CPA_ERR_NULL, "CPA_F_MASK_OUT needs mask_bits");
  if (tp->scores_out && (!out->scores || !out->row_max))
    return fail(CPA_ERR_NULL, "CPA_F_SCORES_OUT needs scores and row_max");
  tp->w = carve(g, ws);
  if (!ws || ws_bytes < tp->w.total) return fail(CPA_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, tp->w.total);
  tp->scores = tp->scores_out ? out->scores : tp->w.scores;
  tp->q = q;
  tp->page_table = c->page_table;
  tp->t = *out;
  tp->num_sms = num_sms;
  if (!tp->mask_in) {
    if (!q) return fail(CPA_ERR_NULL, "q is NULL");
    if (!aligned16(q)) return fail(CPA_ERR_MISALIGNED, "q not 16B aligned");
    cuuint64_t dims[2] = {(cuuint64_t)g.d, (cuuint64_t)2 * g.B * g.Gn * g.Rpad};
    cuuint64_t str[1] = {(cuuint64_t)g.d * 2};
    cuuint32_t box[2] = {64, 128};
    int s;
    if ((s = make_map(&tp->tq, tp->w.qbar, 2, dims, str, box, "qbar")) != CPA_OK) return s;
    if ((s = kv_map(&tp->tk, c->k_pages, g, c->num_pages, ps, hs, "k")) != CPA_OK) return s;
    if (tp->exact && (s = q_map(&tp->tqq, q, g)) != CPA_OK) return s;
  }
  return CPA_OK;
}

int run_tables(const Geo& g, const TablesPlan& tp, cudaStream_t st, bool after_append = false) {
  cudaError_t e;
  int* launches = &g_launches;
  if (!tp.mask_in) {
    if (tp.exact) {  // NEXT-1: SPEC's exact tile-max scorer (full QK^T)
      if ((e = launch_block_scores_exact(tp.tqq, tp.tk, tp.page_table, g, tp.scores, tp.w.mstar_key, tp.num_sms, st,
                                         launches)) != cudaSuccess)
        return cuda_fail(e, "block_scores_exact");
    } else {
      if ((e = launch_pool_q(reinterpret_cast<const __nv_bfloat16*>(tp.q), g, tp.w.qbar, tp.w.mstar_key, tp.w.done, after_append, st,
                             launches)) != cudaSuccess)
        return cuda_fail(e, "pool_q");
      if ((e = launch_block_scores(tp.tq, tp.tk, tp.page_table, g, tp.scores, tp.w.mstar_key, tp.num_sms, st,
                                   launches)) != cudaSuccess)
        return cuda_fail(e, "block_scores");
    }
    if (tp.scores_out) {
      if ((e = launch_row_max(tp.w.mstar_key, g, tp.t.row_max, st, launches)) != cudaSuccess)
        return cuda_fail(e, "row_max");
    }
  }
  if (tp.mask_in && tp.t.dev_status) {
    if ((e = cudaMemsetAsync(tp.t.dev_status, 0, sizeof(int), st)) != cudaSuccess) return cuda_fail(e, "memset");
  }
  // the pooled path's k_pool_q zeroes the tables counter; the other paths do it here
  if (tp.mask_in || tp.exact) {
    if ((e = cudaMemsetAsync(tp.w.done, 0, sizeof(unsigned), st)) != cudaSuccess) return cuda_fail(e, "memset");
  }
  e = launch_tables(tp.scores, tp.w.mstar_key, g, tp.mask_in ? tp.t.mask_bits : nullptr,
                    (!tp.mask_in && (g.flags & CPA_F_MASK_OUT)) ? tp.t.mask_bits : nullptr, tp.w.gwords,
                    tp.mask_in ? tp.t.dev_status : nullptr, tp.w.done, tp.t.kv_indptr, tp.t.kv_indices, st, launches);
  if (e != cudaSuccess) return cuda_fail(e, "tables");
  return CPA_OK;
}

// Output destinations of the attention epilogue (AttnArgs.outs): the call's own o, or the W gathered
// buffers of a peer exchange (cpa_chunk_step_peer).
struct OutSpec {
  int n;
  void* outs[kMaxOut];
  long long stride, bstride;  // elements between tokens / batch entries
};

struct AttnPlan {
  CUtensorMap tq, tk, tv, tkh;
  AttnArgs a;
  int kind;  // 0: 1-CTA kernel, 1: 2-CTA per-unit grid, 2: 2-CTA persistent stream-K grid, 3: row-split 2-CTA,
             // 4: 2-CTA, four key slices with a shared running max (attention_ks4.cu)
  SkSched sk;
};

int prep_attention(const cpa_params* p, const Geo& g, const void* q, const void* k_pages, const void* v_pages,
                   int num_pages, long long ps, long long hs, const int32_t* page_table, const int32_t* indptr,
                   const int32_t* indices, void* o, AttnPlan* ap, const uint32_t* mask = nullptr,
                   const OutSpec* os = nullptr, void* ws = nullptr, size_t ws_bytes = 0) {
  int s;
  if ((s = q_map(&ap->tq, q, g)) != CPA_OK) return s;
  if ((s = kv_map(&ap->tk, k_pages, g, num_pages, ps, hs, "k")) != CPA_OK) return s;
  if ((s = kv_map(&ap->tv, v_pages, g, num_pages, ps, hs, "v")) != CPA_OK) return s;
  AttnArgs& a = ap->a;
  a.page_table = page_table;
  a.indptr = indptr;
  a.indices = indices;
  a.mask = mask;
  a.out_f32 = (p->flags & CPA_F_OUT_F32) ? 1 : 0;
  for (int k = 0; k < kMaxOut; ++k) a.outs[k] = nullptr;
  if (os) {
    a.n_out = os->n;
    for (int k = 0; k < os->n; ++k) a.outs[k] = os->outs[k];
    a.o_stride = os->stride;
    a.o_bstride = os->bstride;
  } else {
    a.n_out = 1;
    a.outs[0] = o;
    a.o_stride = g.q_stride;
    a.o_bstride = g.b_stride;
  }
  ap->kind = 0;
  if (attn_2cta_supported(g) && !(p->flags & CPA_F_NO_2CTA) && mask == nullptr) {
    // half a page of keys per CTA of the pair
    if ((s = kv_map(&ap->tkh, k_pages, g, num_pages, ps, hs, "k_half", g.bs / 2)) != CPA_OK) return s;
    const int clusters = std::min(attn_2cta_max_clusters(g), kSkMaxClusters);
    // measured: on the sparse tables the per-unit grid is as fast (the chip is power-
    // bound, idle SM pairs are not lost time); on the dense baseline the persistent grid is 2-5% faster
    const bool auto_sk = indptr == nullptr && sk_wanted(g, clusters);
    ap->kind = 1;
    if (ws != nullptr && !(p->flags & CPA_F_NO_PERSIST) &&
        (auto_sk || ((p->flags & CPA_F_PERSIST) && sk_wanted(g, clusters)))) {
      if (ws_bytes < attn_ws_bytes(g)) return fail(CPA_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, attn_ws_bytes(g));
      ap->sk = carve_sk(g, ws, clusters);
      ap->kind = 2;
    }
    if (ap->kind == 1 && attn_rs_supported(g) && (p->flags & CPA_F_ATTN_RS)) ap->kind = 3;
    if (ap->kind == 1 && attn_ks4_supported(g) && (p->flags & CPA_F_ATTN_KS4)) ap->kind = 4;
  }
  return CPA_OK;
}

int run_attention(const Geo& g, const AttnPlan& ap, cudaStream_t st) {
  cudaError_t e;
  if (ap.kind == 0) e = launch_paged_attention(ap.tq, ap.tk, ap.tv, g, ap.a, st, &g_launches);
  else if (ap.kind == 3) e = launch_paged_attention_rs(ap.tq, ap.tkh, ap.tv, g, ap.a, st, &g_launches);
  else if (ap.kind == 4) e = launch_paged_attention_ks4(ap.tq, ap.tkh, ap.tv, g, ap.a, st, &g_launches);
  else e = launch_paged_attention_2cta(ap.tq, ap.tkh, ap.tv, g, ap.a, ap.kind == 2 ? &ap.sk : nullptr, st, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "paged_attention");
  return CPA_OK;
}

int attention_launch(const cpa_params* p, const Geo& g, const void* q, const void* k_pages, const void* v_pages,
                     int num_pages, long long ps, long long hs, const int32_t* page_table, const int32_t* indptr,
                     const int32_t* indices, void* o, cudaStream_t st, const uint32_t* mask = nullptr) {
  AttnPlan ap;
  int s;
  if ((s = prep_attention(p, g, q, k_pages, v_pages, num_pages, ps, hs, page_table, indptr, indices, o, &ap, mask)) !=
      CPA_OK)
    return s;
  return run_attention(g, ap, st);
}

int prep_attention_impl(const cpa_params* p, const Geo& g, const void* q, const cpa_kv_cache* c, long long ps,
                        long long hs, const cpa_tables* t, void* o, const OutSpec* os, void* ws, size_t ws_bytes,
                        AttnPlan* ap) {
  if (!q || (!o && !os)) return fail(CPA_ERR_NULL, "q/o is NULL");
  if (!aligned16(q) || (!os && !aligned16(o))) return fail(CPA_ERR_MISALIGNED, "q/o not 16B aligned");
  if (t && (!t->kv_indptr || !t->kv_indices)) return fail(CPA_ERR_NULL, "tables pointers");
  if (attn_2cta_supported(g) && !(p->flags & (CPA_F_NO_2CTA | CPA_F_NO_PERSIST)) && attn_ws_bytes(g) > 0 &&
      ws_bytes < attn_ws_bytes(g))
    return fail(CPA_ERR_WORKSPACE, "paged attention needs cpa_workspace_bytes() of workspace");
  return prep_attention(p, g, q, c->k_pages, c->v_pages, c->num_pages, ps, hs, c->page_table,
                        t ? t->kv_indptr : nullptr, t ? t->kv_indices : nullptr, o, ap, nullptr, os, ws, ws_bytes);
}

// append (optional) -> estimator + tables -> attention, the body of cpa_chunk_step(_peer). Everything
// is validated and planned before the append's launch (cpa.h: a failing call leaves outputs untouched).
int chunk_step_impl(const cpa_params* p, const void* q, const void* k_chunk, const void* v_chunk,
                    const cpa_kv_cache* cache, cpa_tables* tables, void* o, void* ws, size_t ws_bytes,
                    cudaStream_t st, const OutSpec* os, bool with_attention = true) {
  Geo g;
  int s, sms;
  long long ps, hs;
  if ((s = make_geo(p, &g)) != CPA_OK) return s;
  if ((s = check_cache(cache, &g, &ps, &hs)) != CPA_OK) return s;
  if ((s = device_info(&sms)) != CPA_OK) return s;
  if ((k_chunk == nullptr) != (v_chunk == nullptr)) return fail(CPA_ERR_NULL, "k_chunk/v_chunk: both or neither");
  if (!q || (with_attention && !o && !os)) return fail(CPA_ERR_NULL, "q/o is NULL");
  if (!tables) return fail(CPA_ERR_NULL, "tables is NULL");
  if (k_chunk && (!aligned16(k_chunk) || !aligned16(v_chunk)))
    return fail(CPA_ERR_MISALIGNED, "k/v chunk not 16B aligned");
  TablesPlan tp;
  AttnPlan ap;
  if ((s = prep_tables(p, g, q, cache, ps, hs, tables, ws, ws_bytes, sms, &tp)) != CPA_OK) return s;
  if (with_attention && (s = prep_attention_impl(p, g, q, cache, ps, hs, tables, o, os, ws, ws_bytes, &ap)) != CPA_OK)
    return s;
  if (k_chunk) {
    cudaError_t e = launch_append(k_chunk, v_chunk, *cache, g, ps, hs, sms, st, &g_launches);
    if (e != cudaSuccess) return cuda_fail(e, "append");
  }
  if ((s = run_tables(g, tp, st, k_chunk != nullptr)) != CPA_OK) return s;
  return with_attention ? run_attention(g, ap, st) : CPA_OK;
}

int check_peers(const cpa_peer_out* pr) {
  if (!pr || !pr->peer_signal) return fail(CPA_ERR_NULL, "peers / peer_signal is NULL");
  if (pr->world < 1 || pr->world > CPA_MAX_PEERS || pr->rank < 0 || pr->rank >= pr->world)
    return fail(CPA_ERR_SHAPE, "world %d / rank %d out of range (world <= %d)", pr->world, pr->rank, CPA_MAX_PEERS);
  for (int w = 0; w < pr->world; ++w) {
    if (!pr->peer_signal[w]) return fail(CPA_ERR_NULL, "peer_signal[%d] is NULL", w);
    if (reinterpret_cast<uintptr_t>(pr->peer_signal[w]) & 3u) return fail(CPA_ERR_MISALIGNED, "peer_signal[%d]", w);
  }
  return CPA_OK;
}

int peer_barrier_impl(const cpa_peer_out* pr, cudaStream_t st) {
  PeerSig sg;
  for (int w = 0; w < kMaxOut; ++w) sg.pads[w] = w < pr->world ? pr->peer_signal[w] : nullptr;
  sg.world = pr->world;
  sg.rank = pr->rank;
  sg.epoch = pr->epoch;
  sg.status = pr->dev_status;
  sg.timeout_ns = (unsigned long long)(pr->timeout_ms ? pr->timeout_ms : 10000u) * 1000000ull;
  cudaError_t e = launch_peer_barrier(sg, st, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "peer_barrier");
  return CPA_OK;
}

// NEXT-3 copy ablation: compact pool [B*Gn*nkvb pages] of K and of V + per-row page tables
size_t copy_ws_bytes(const Geo& g) {
  const size_t pages = (size_t)g.B * g.Gn * g.nkvb;
  return 2 * up256(pages * g.bs * g.d * 2) + up256(pages * 4);
}

}  // namespace

extern "C" {

size_t cpa_workspace_bytes(const cpa_params* p) {
  Geo g;
  if (make_geo(p, &g) != CPA_OK) return 0;
  return std::max(carve(g, nullptr).total, attn_ws_bytes(g));
}

int cpa_build_tables(const cpa_params* p, const void* q, const cpa_kv_cache* cache, cpa_tables* out,
                     void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  Geo g;
  int s, sms;
  long long ps, hs;
  if ((s = make_geo(p, &g)) != CPA_OK) return s;
  if ((s = check_cache(cache, &g, &ps, &hs)) != CPA_OK) return s;
  if ((s = device_info(&sms)) != CPA_OK) return s;
  TablesPlan tp;
  if ((s = prep_tables(p, g, q, cache, ps, hs, out, ws, ws_bytes, sms, &tp)) != CPA_OK) return s;
  return run_tables(g, tp, (cudaStream_t)stream);
}

int cpa_paged_attention(const cpa_params* p, const void* q, const cpa_kv_cache* cache, const cpa_tables* tables,
                        void* o, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  Geo g;
  int s, sms;
  long long ps, hs;
  if ((s = make_geo(p, &g)) != CPA_OK) return s;
  if ((s = check_cache(cache, &g, &ps, &hs)) != CPA_OK) return s;
  if ((s = device_info(&sms)) != CPA_OK) return s;
  AttnPlan ap;
  if ((s = prep_attention_impl(p, g, q, cache, ps, hs, tables, o, nullptr, ws, ws_bytes, &ap)) != CPA_OK) return s;
  return run_attention(g, ap, (cudaStream_t)stream);
}

int cpa_append_kv(const cpa_params* p, const void* k_chunk, const void* v_chunk, const cpa_kv_cache* cache,
                  void* stream) {
  g_launches = 0;
  Geo g;
  int s, sms;
  long long ps, hs;
  if ((s = make_geo(p, &g)) != CPA_OK) return s;
  if ((s = check_cache(cache, &g, &ps, &hs)) != CPA_OK) return s;
  if ((s = device_info(&sms)) != CPA_OK) return s;
  if (!k_chunk || !v_chunk) return fail(CPA_ERR_NULL, "k_chunk/v_chunk NULL");
  if (!aligned16(k_chunk) || !aligned16(v_chunk)) return fail(CPA_ERR_MISALIGNED, "k/v chunk not 16B aligned");
  cudaError_t e = launch_append(k_chunk, v_chunk, *cache, g, ps, hs, sms, (cudaStream_t)stream, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "append");
  return CPA_OK;
}

int cpa_prepare_chunk(const cpa_params* p, const void* q, const void* k_chunk, const void* v_chunk,
                      const cpa_kv_cache* cache, cpa_tables* tables, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  return chunk_step_impl(p, q, k_chunk, v_chunk, cache, tables, nullptr, ws, ws_bytes, (cudaStream_t)stream, nullptr,
                         false);
}

int cpa_chunk_step(const cpa_params* p, const void* q, const void* k_chunk, const void* v_chunk,
                   const cpa_kv_cache* cache, cpa_tables* tables, void* o, void* ws, size_t ws_bytes,
                   void* stream) {
  g_launches = 0;
  return chunk_step_impl(p, q, k_chunk, v_chunk, cache, tables, o, ws, ws_bytes, (cudaStream_t)stream, nullptr);
}

}  // extern "C"

namespace {
// OutSpec of a peer exchange: this rank's head slice of every rank's gathered buffer, own buffer first,
// then the peers in rotated order (spreads the NVLink load).
int peer_outspec(const cpa_params* p, const Geo& g, const cpa_peer_out* peers, OutSpec* os) {
  int s;
  if ((s = check_peers(peers)) != CPA_OK) return s;
  if (!peers->peer_out) return fail(CPA_ERR_NULL, "peer_out is NULL");
  const int W = peers->world;
  const long long row = (long long)W * g.Hq * g.d;
  os->n = W;
  os->stride = peers->out_token_stride ? peers->out_token_stride : row;
  if (os->stride < row || os->stride % 8)
    return fail(CPA_ERR_SHAPE, "out_token_stride must be >= W*Hq*d, multiple of 8");
  os->bstride = (long long)g.C * os->stride;
  const size_t esz = (p->flags & CPA_F_OUT_F32) ? 4 : 2;
  for (int k = 0; k < W; ++k) {
    const int w = (peers->rank + k) % W;
    if (!peers->peer_out[w]) return fail(CPA_ERR_NULL, "peer_out[%d] is NULL", w);
    if (!aligned16(peers->peer_out[w])) return fail(CPA_ERR_MISALIGNED, "peer_out[%d] not 16B aligned", w);
    os->outs[k] = reinterpret_cast<uint8_t*>(peers->peer_out[w]) + (size_t)peers->rank * g.Hq * g.d * esz;
  }
  return CPA_OK;
}
}  // namespace

extern "C" {

int cpa_chunk_step_peer(const cpa_params* p, const void* q, const void* k_chunk, const void* v_chunk,
                        const cpa_kv_cache* cache, cpa_tables* tables, const cpa_peer_out* peers, void* ws,
                        size_t ws_bytes, void* stream) {
  g_launches = 0;
  Geo g;
  int s;
  OutSpec os;
  if ((s = make_geo(p, &g)) != CPA_OK) return s;
  if ((s = peer_outspec(p, g, peers, &os)) != CPA_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = chunk_step_impl(p, q, k_chunk, v_chunk, cache, tables, nullptr, ws, ws_bytes, st, &os)) != CPA_OK)
    return s;
  return peer_barrier_impl(peers, st);
}

int cpa_paged_attention_peer(const cpa_params* p, const void* q, const cpa_kv_cache* cache, const cpa_tables* tables,
                             const cpa_peer_out* peers, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  Geo g;
  int s, sms;
  long long ps, hs;
  OutSpec os;
  if ((s = make_geo(p, &g)) != CPA_OK) return s;
  if ((s = peer_outspec(p, g, peers, &os)) != CPA_OK) return s;
  if ((s = check_cache(cache, &g, &ps, &hs)) != CPA_OK) return s;
  if ((s = device_info(&sms)) != CPA_OK) return s;
  AttnPlan ap;
  if ((s = prep_attention_impl(p, g, q, cache, ps, hs, tables, nullptr, &os, ws, ws_bytes, &ap)) != CPA_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = run_attention(g, ap, st)) != CPA_OK) return s;
  return peer_barrier_impl(peers, st);
}

int cpa_peer_barrier(const cpa_peer_out* peers, void* stream) {
  g_launches = 0;
  int s, sms;
  if ((s = check_peers(peers)) != CPA_OK) return s;
  if ((s = device_info(&sms)) != CPA_OK) return s;
  return peer_barrier_impl(peers, (cudaStream_t)stream);
}

size_t cpa_copy_workspace_bytes(const cpa_params* p) {
  Geo g;
  if (make_geo(p, &g) != CPA_OK) return 0;
  return copy_ws_bytes(g);
}

int cpa_paged_attention_copy(const cpa_params* p, const void* q, const cpa_kv_cache* cache, const cpa_tables* t,
                             void* o, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  Geo g;
  int s, sms;
  long long ps, hs;
  if ((s = make_geo(p, &g)) != CPA_OK) return s;
  if ((s = check_cache(cache, &g, &ps, &hs)) != CPA_OK) return s;
  if ((s = device_info(&sms)) != CPA_OK) return s;
  if (!q || !o || !t || !t->kv_indptr || !t->kv_indices) return fail(CPA_ERR_NULL, "q/o/tables NULL");
  if (!ws || ws_bytes < copy_ws_bytes(g)) return fail(CPA_ERR_WORKSPACE, "copy workspace too small");
  const size_t pages = (size_t)g.B * g.Gn * g.nkvb;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  void* ck = base;
  void* cv = base + up256(pages * g.bs * g.d * 2);
  int32_t* cpt = reinterpret_cast<int32_t*>(base + 2 * up256(pages * g.bs * g.d * 2));
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = launch_gather_pages(*cache, t->kv_indptr, t->kv_indices, g, ps, hs, ck, cv, cpt, st, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "gather_pages");
  // per batch entry: pseudo-batch over the Gn execution groups (one KV head each, its own page list)
  for (int b = 0; b < g.B; ++b) {
    Geo gb = g;
    gb.B = g.Gn;
    gb.Hq = g.E;
    gb.Hkv = 1;
    gb.Gn = 1;
    gb.kv_per_q = g.E;
    gb.b_stride = (long long)g.E * g.d;  // next group's heads
    gb.maxb = g.nkvb;
    gb.nwords = g.nwords;
    const size_t off = (size_t)b * g.b_stride * 2;
    const void* qb = reinterpret_cast<const uint8_t*>(q) + off;
    void* ob = reinterpret_cast<uint8_t*>(o) + off * ((p->flags & CPA_F_OUT_F32) ? 2 : 1);
    if ((s = attention_launch(p, gb, qb, ck, cv, (int)pages, (long long)g.bs * g.d, (long long)g.bs * g.d,
                              cpt + (size_t)b * g.Gn * g.nkvb, t->kv_indptr + (size_t)b * g.Gn, t->kv_indices, ob,
                              st)) != CPA_OK)
      return s;
  }
  return CPA_OK;
}

int cpa_block_sparse_attention(const cpa_params* p, const void* q, const cpa_kv_cache* cache, const uint32_t* mask,
                               void* o, void* ws, size_t ws_bytes, void* stream) {
  (void)ws;
  (void)ws_bytes;
  g_launches = 0;
  Geo g;
  int s, sms;
  long long ps, hs;
  if ((s = make_geo(p, &g)) != CPA_OK) return s;
  if ((s = check_cache(cache, &g, &ps, &hs)) != CPA_OK) return s;
  if ((s = device_info(&sms)) != CPA_OK) return s;
  if (!q || !o || !mask) return fail(CPA_ERR_NULL, "q/o/mask is NULL");
  if (!aligned16(q) || !aligned16(o)) return fail(CPA_ERR_MISALIGNED, "q/o not 16B aligned");
  if (g.bs != 128) return fail(CPA_ERR_UNSUPPORTED, "block-sparse execution needs block_size 128");
  if (g.nkvb > 4096) return fail(CPA_ERR_UNSUPPORTED, "block-sparse execution needs nkvb <= 4096");
  return attention_launch(p, g, q, cache->k_pages, cache->v_pages, cache->num_pages, ps, hs, cache->page_table,
                          nullptr, nullptr, o, (cudaStream_t)stream, mask);
}

int cpa_expand_tables(const cpa_params* p, const cpa_tables* t, uint32_t* mask, void* stream) {
  g_launches = 0;
  Geo g;
  int s, sms;
  if ((s = make_geo(p, &g)) != CPA_OK) return s;
  if ((s = device_info(&sms)) != CPA_OK) return s;
  if (!t || !t->kv_indptr || !t->kv_indices || !mask) return fail(CPA_ERR_NULL, "tables/mask is NULL");
  cudaError_t e = launch_expand_tables(t->kv_indptr, t->kv_indices, g, mask, (cudaStream_t)stream, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "expand_tables");
  return CPA_OK;
}

const char* cpa_status_string(int status) {
  switch (status) {
    case CPA_OK: return "CPA_OK";
    case CPA_ERR_NULL: return "CPA_ERR_NULL";
    case CPA_ERR_SHAPE: return "CPA_ERR_SHAPE";
    case CPA_ERR_UNSUPPORTED: return "CPA_ERR_UNSUPPORTED";
    case CPA_ERR_MISALIGNED: return "CPA_ERR_MISALIGNED";
    case CPA_ERR_ALPHA: return "CPA_ERR_ALPHA";
    case CPA_ERR_WORKSPACE: return "CPA_ERR_WORKSPACE";
    case CPA_ERR_CAPACITY: return "CPA_ERR_CAPACITY";
    case CPA_ERR_CUDA: return "CPA_ERR_CUDA";
    default: return "CPA_ERR_UNKNOWN";
  }
}
const char* cpa_last_error(void) { return g_err; }
int cpa_version(void) { return CPA_VERSION; }
int cpa_last_launch_count(void) { return g_launches; }

}  // extern "C"
