// TMEM load/store throughput microbenchmark (sm_100a).
#include <cstdio>
#include <cstdint>
#include "../../paper_2605_16839_b200/csrc/common.cuh"
using namespace cpa;
template <int MODE, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k(long long* cyc, int iters, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp / 4) * 64;
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = threadIdx.x + i;
  float acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {  // 4 back-to-back x32 loads, one wait
      uint32_t a[32], b[32], c[32], d[32];
      tmem_ld32(tm, a); tmem_ld32(tm + 32, b); tmem_ld32(tm + 128, c); tmem_ld32(tm + 160, d);
      tmem_wait_ld();
      acc += __uint_as_float(a[5]) + __uint_as_float(b[3]) + __uint_as_float(c[7]) + __uint_as_float(d[9]) + __uint_as_float(a[30]) + __uint_as_float(d[31]);
    } else if (MODE == 1) {  // x16 stores
      uint32_t (&s)[16] = *reinterpret_cast<uint32_t(*)[16]>(v);
      tmem_st16(tm, s); tmem_st16(tm + 16, s); tmem_st16(tm + 32, s); tmem_st16(tm + 48, s);
      tmem_wait_st();
    } else {  // single x32 load + wait (latency)
      uint32_t a[32];
      tmem_ld32(tm + (it & 3) * 32, a);
      tmem_wait_ld();
      acc += __uint_as_float(a[7]) + __uint_as_float(a[31]);
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(slot); }
}
template <int MODE, int WARPS> void run(long long* c, float* s) {
  int iters = 2000;
  k<MODE, WARPS><<<148, WARPS * 32>>>(c, iters, s); cudaDeviceSynchronize();
  k<MODE, WARPS><<<148, WARPS * 32>>>(c, iters, s); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double per_it = (double)h / iters;
  double bytes = MODE == 0 ? WARPS * 32 * 4 * 128.0 : MODE == 1 ? WARPS * 32 * 4 * 64.0 : WARPS * 32 * 4 * 32.0;
  printf("mode=%d warps=%2d cycles/iter=%.1f  bytes/iter/SM=%.0f  => %.1f B/cycle/SM  err=%s\n", MODE, WARPS, per_it,
         bytes, bytes / per_it, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* c; float* s; cudaMalloc(&c, 1 << 16); cudaMalloc(&s, 1 << 22);
  run<0, 4>(c, s); run<0, 8>(c, s); run<1, 4>(c, s); run<1, 8>(c, s); run<2, 4>(c, s); run<2, 8>(c, s);
  return 0;
}
