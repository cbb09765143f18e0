// append.cu -- §8 row a0 (optional): write the chunk's K/V tokens [P, P+C) into their pages
// (SPEC.md:130-138 append_chunk). Plus the small row-max export used by CPA_F_SCORES_OUT.
#include "../../include/cpa.h"
#include "common.cuh"
#include "geo.cuh"
#include "launch.cuh"

namespace cpa {

// One warp per chunk token (b, c): the token's page is looked up once, then the warp copies its
// Hkv*d/8 16-byte vectors of K and of V (source [B, C, Hkv, d] contiguous, so every warp request is
// 512 contiguous bytes; each (head, token) row of d elements lands contiguous in its page slot). All
// loads of a token are issued before its stores (4 x 2 vectors per lane in flight for d=128, Hkv=8).
// Grid: at most 4 resident 8-warp CTAs per SM (half the threads: k_pool_q runs alongside under PDL),
// grid-stride over tokens.
constexpr int kAppendUnroll = 4;
__global__ void __launch_bounds__(256) k_append(const uint4* __restrict__ kc, const uint4* __restrict__ vc,
                                                uint4* __restrict__ kp, uint4* __restrict__ vp,
                                                const int32_t* __restrict__ pt, Geo g, long long ps, long long hs) {
  const int lane = threadIdx.x & 31;
  const int vshift = g.d == 128 ? 4 : 3;  // 16-byte vectors per (token, head) row: d/8
  const int per_tok = g.Hkv << vshift;
  const long long ntok = (long long)g.B * g.C;
  const long long hs16 = hs >> 3, ps16 = ps >> 3;
  const bool f16 = (g.flags & CPA_F_V_F16) != 0;
  const long long wstride = ((long long)gridDim.x * blockDim.x) >> 5;
  pdl_wait();     // the pages may still be read by the previous kernel (e.g. the last step's attention)
  pdl_trigger();  // pool_q (next) does not read the pages: let it run alongside
  for (long long tok = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; tok < ntok; tok += wstride) {
    const int b = (int)(tok / g.C);
    const int t = g.P + (int)(tok - (long long)b * g.C);
    const int j = t / g.bs;
    const int page = __ldg(pt + (long long)b * g.maxb + j);
    const long long dst0 = (long long)page * ps16 + (long long)(t - j * g.bs) * (g.d >> 3);
    const uint4* ks = kc + tok * per_tok;
    const uint4* vs = vc + tok * per_tok;
    for (int x0 = 0; x0 < per_tok; x0 += 32 * kAppendUnroll) {
      uint4 kr[kAppendUnroll], vr[kAppendUnroll];
#pragma unroll
      for (int u = 0; u < kAppendUnroll; ++u) {
        const int x = x0 + u * 32 + lane;
        if (x < per_tok) {
          kr[u] = __ldcs(ks + x);  // read once: evict-first
          vr[u] = __ldcs(vs + x);
        }
      }
#pragma unroll
      for (int u = 0; u < kAppendUnroll; ++u) {
        const int x = x0 + u * 32 + lane;
        if (x < per_tok) {
          const long long dst = dst0 + (long long)(x >> vshift) * hs16 + (x & ((1 << vshift) - 1));
          kp[dst] = kr[u];
          uint4 w = vr[u];
          if (f16) {  // V pool in fp16 (exact for bf16 values in fp16's normal range, saturating beyond)
            w.x = bf16x2_to_f16x2(w.x);
            w.y = bf16x2_to_f16x2(w.y);
            w.z = bf16x2_to_f16x2(w.z);
            w.w = bf16x2_to_f16x2(w.w);
          }
          vp[dst] = w;
        }
      }
    }
  }
}

cudaError_t launch_append(const void* kc, const void* vc, const cpa_kv_cache& c, const Geo& g, long long ps,
                          long long hs, int num_sms, cudaStream_t st, int* launches) {
  const long long ntok = (long long)g.B * g.C;
  const long long need = (ntok + 7) / 8;         // 8 tokens (warps) per CTA
  const long long cap = (long long)num_sms * 4;  // 4 resident 256-thread CTAs per SM (room for pool_q)
  const int blocks = (int)(need < cap ? need : cap);
  ++*launches;
  return launch_ex(k_append, dim3(blocks), dim3(256), 0, st, use_pdl(g), reinterpret_cast<const uint4*>(kc),
                   reinterpret_cast<const uint4*>(vc), reinterpret_cast<uint4*>(c.k_pages),
                   reinterpret_cast<uint4*>(c.v_pages), c.page_table, g, ps, hs);
}

// NEXT-3 "copy" execution ablation: gather the tabled K/V pages of every
// (b, g) row into a compact pool (slot e = the row's CSR entry) and write the row's page table
// cpt[r][j] = e. grid (nkvb, B*Gn), 256 threads; CTA (x, r) copies entry indptr[r] + x if it exists.
__global__ void __launch_bounds__(256) k_gather_pages(const uint4* __restrict__ kp, const uint4* __restrict__ vp,
                                                      const int32_t* __restrict__ pt, const int32_t* __restrict__ indptr,
                                                      const int32_t* __restrict__ indices, Geo g, long long ps,
                                                      long long hs, uint4* __restrict__ ck, uint4* __restrict__ cv,
                                                      int32_t* __restrict__ cpt) {
  const int x = blockIdx.x, r = blockIdx.y;
  const int beg = __ldg(indptr + r), len = __ldg(indptr + r + 1) - beg;
  if (x >= len) return;
  const int e = beg + x, j = __ldg(indices + e);
  const int b = r / g.Gn, grp = r % g.Gn;
  const int page = __ldg(pt + (long long)b * g.maxb + j);
  const long long src = ((long long)page * ps + (long long)group_kv_head(g, grp) * hs) / 8;
  const int nvec = g.bs * g.d / 8;
  for (int t = threadIdx.x; t < nvec; t += blockDim.x) {
    ck[(long long)e * nvec + t] = kp[src + t];
    cv[(long long)e * nvec + t] = vp[src + t];
  }
  if (threadIdx.x == 0) cpt[(long long)r * g.nkvb + j] = e;
}

cudaError_t launch_gather_pages(const cpa_kv_cache& c, const int32_t* indptr, const int32_t* indices, const Geo& g,
                                long long ps, long long hs, void* ck, void* cv, int32_t* cpt, cudaStream_t st,
                                int* launches) {
  k_gather_pages<<<dim3(g.nkvb, g.B * g.Gn), 256, 0, st>>>(
      reinterpret_cast<const uint4*>(c.k_pages), reinterpret_cast<const uint4*>(c.v_pages), c.page_table, indptr,
      indices, g, ps, hs, reinterpret_cast<uint4*>(ck), reinterpret_cast<uint4*>(cv), cpt);
  ++*launches;
  return cudaGetLastError();
}

__global__ void k_row_max(const int* __restrict__ key, long long n, float* __restrict__ out) {
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x)
    out[x] = key_float(key[x]);
}

cudaError_t launch_row_max(const int* mstar_key, const Geo& g, float* row_max, cudaStream_t st, int* launches) {
  const long long n = (long long)g.B * g.Gn * g.Rpad;
  k_row_max<<<(int)((n + 255) / 256), 256, 0, st>>>(mstar_key, n, row_max);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace cpa
