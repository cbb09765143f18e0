// Per-element cost of the softmax inner loop (per SMSP) for different MUFU/polynomial splits.
#include <cstdio>
#include <cstdint>
#include "../../paper_2605_16839_b200/csrc/common.cuh"
using namespace cpa;
template <int MASK>
__device__ __forceinline__ bool polyq(int q2) { return ((MASK >> (q2 & 7)) & 1) != 0; }
template <int MASK>
__global__ void __launch_bounds__(256) k(float* out, long long* cyc, int iters) {
  uint32_t sv[64];
  for (int i = 0; i < 64; ++i) sv[i] = __float_as_uint((threadIdx.x * 0.001f + i * 0.01f) - 3.0f);
  float l = 0.f, m = 0.5f;
  uint32_t ok = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
    for (int q2 = 0; q2 < 32; ++q2) {
      float2 x = ffma2(make_float2(__uint_as_float(sv[2 * q2]), __uint_as_float(sv[2 * q2 + 1])), 1.1f, -m);
      float2 e;
      if (polyq<MASK>(q2)) e = exp2_poly2(x);
      else { e.x = fast_exp2(x.x); e.y = fast_exp2(x.y); }
      acc[q2 & 3] = fadd2(acc[q2 & 3], e);
      ok ^= pack_f16x2(e.x, e.y);
    }
    l += acc[0].x + acc[1].y + acc[2].x + acc[3].y;
    m += 1e-7f;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + ok;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MASK> void run(float* o, long long* c, const char* name) {
  int iters = 2000;
  k<MASK><<<148, 256>>>(o, c, iters); cudaDeviceSynchronize();
  k<MASK><<<148, 256>>>(o, c, iters); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  // 8 warps/SM = 2 per SMSP; elements per SMSP per iteration = 2 warps * 32 lanes * 64
  printf("%-10s cycles/iter=%.1f  -> SMSP cycles per 128x128 tile-quarter (4096 el/SMSP): %.0f\n", name,
         (double)h / iters, (double)h / iters / (2 * 32 * 64) * 4096);
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 1 << 22); cudaMalloc(&c, 1 << 16);
  run<0x00>(o, c, "mufu-only"); run<0x12>(o, c, "poly 1/4"); run<0x52>(o, c, "poly 3/8");
  run<0x5A>(o, c, "poly 1/2"); run<0xFF>(o, c, "poly all");
  return 0;
}
