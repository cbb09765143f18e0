// append.cu -- §8 row a0 (optional): write the chunk's K/V tokens [P, P+C) into their pages
// (SPEC.md:130-138 append_chunk). Plus the small row-max export used by CPA_F_SCORES_OUT.
#include "../../include/cpa.h"
#include "common.cuh"
#include "geo.cuh"

namespace cpa {

// grid (C, Hkv, B), block d/8 threads: one 16-byte vector per thread for K and for V.
__global__ void k_append(const uint4* __restrict__ kc, const uint4* __restrict__ vc, uint4* __restrict__ kp,
                         uint4* __restrict__ vp, const int32_t* __restrict__ pt, Geo g, long long ps,
                         long long hs) {
  const int c = blockIdx.x, h = blockIdx.y, b = blockIdx.z, e = threadIdx.x;  // e: 8-element vector
  const int t = g.P + c, j = t / g.bs, slot = t % g.bs;
  const int page = __ldg(pt + (long long)b * g.maxb + j);
  const long long src = (((long long)b * g.C + c) * g.Hkv + h) * (g.d / 8) + e;
  const long long dst = ((long long)page * ps + (long long)h * hs + (long long)slot * g.d) / 8 + e;
  kp[dst] = kc[src];
  vp[dst] = vc[src];
}

cudaError_t launch_append(const void* kc, const void* vc, const cpa_kv_cache& c, const Geo& g, long long ps,
                          long long hs, cudaStream_t st, int* launches) {
  k_append<<<dim3(g.C, g.Hkv, g.B), g.d / 8, 0, st>>>(
      reinterpret_cast<const uint4*>(kc), reinterpret_cast<const uint4*>(vc),
      reinterpret_cast<uint4*>(c.k_pages), reinterpret_cast<uint4*>(c.v_pages),
      c.page_table, g, ps, hs);
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
