// Does tcgen05.ld/st .16x256b work at a lane base of 16 within a warp's 32-lane sub-partition, so that
// the two softmax warps of one SMSP (warps w and w+4) can own rows [32q, 32q+16) and [32q+16, 32q+32)?
// Writes row*1000+col with 32x32b stores, reads back with 16x256b at lane base 32q + 16*(w/4); then the
// reverse (16x256b stores, 32x32b loads). Prints the mismatch counts (expect 0 0).
#include <cstdint>
#include <cstdio>
#include "../../paper_2605_16839_b200/csrc/common.cuh"
using namespace cpa;

__device__ __forceinline__ void ld16x256(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
}
__device__ __forceinline__ void st16x256(uint32_t taddr, const uint32_t (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
}

__global__ void __launch_bounds__(256) k(int* bad) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31, q = warp & 3, half = warp >> 2;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  // phase 1: warps 0-3 write rows 32q+lane, cols [0,64) with 32x32b
  if (warp < 4) {
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t v[16];
      for (int c = 0; c < 16; ++c) v[c] = (32 * q + lane) * 1000 + c0 + c;
      tmem_st16(tm + ((uint32_t)(32 * q) << 16) + c0, v);
    }
    tmem_wait_st();
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  // phase 2: all 8 warps read their 16-lane half with 16x256b, cols [0, 64)
  int nbad = 0;
  const int base = 32 * q + 16 * half;
  for (int c0 = 0; c0 < 64; c0 += 8) {
    uint32_t r[4];
    ld16x256(tm + ((uint32_t)base << 16) + c0, r);
    tmem_wait_ld();
    const int t0 = lane & 3, t1 = lane >> 2;
    const int rows[2] = {base + t1, base + t1 + 8};
    for (int k2 = 0; k2 < 4; ++k2) {
      const uint32_t want = rows[k2 >> 1] * 1000 + c0 + 2 * t0 + (k2 & 1);
      if (r[k2] != want) ++nbad;
    }
  }
  atomicAdd(bad, nbad);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  // phase 3: 8 warps write cols [64, 128) of their half with 16x256b; warps 0-3 read back with 32x32b
  for (int c0 = 64; c0 < 128; c0 += 8) {
    const int t0 = lane & 3, t1 = lane >> 2;
    uint32_t r[4];
    for (int k2 = 0; k2 < 4; ++k2) r[k2] = (base + t1 + 8 * (k2 >> 1)) * 1000 + c0 + 2 * t0 + (k2 & 1);
    st16x256(tm + ((uint32_t)base << 16) + c0, r);
  }
  tmem_wait_st();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp < 4) {
    int nb = 0;
    for (int c0 = 64; c0 < 128; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(tm + ((uint32_t)(32 * q) << 16) + c0, v);
      tmem_wait_ld();
      for (int c = 0; c < 16; ++c)
        if (v[c] != (uint32_t)((32 * q + lane) * 1000 + c0 + c)) ++nb;
    }
    atomicAdd(bad + 1, nb);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

int main() {
  int* bad;
  cudaMalloc(&bad, 8);
  cudaMemset(bad, 0, 8);
  k<<<1, 256>>>(bad);
  cudaError_t e = cudaDeviceSynchronize();
  int h[2] = {-1, -1};
  cudaMemcpy(h, bad, 8, cudaMemcpyDeviceToHost);
  printf("16x256b at lane base +16: load mismatches %d, store mismatches %d (%s)\n", h[0], h[1], cudaGetErrorString(e));
  return 0;
}
