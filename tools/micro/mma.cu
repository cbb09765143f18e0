// tcgen05.mma throughput: SS (A,B smem) vs TS (A TMEM) for M=128, K=16, N in {64,128,256}.
#include <cstdio>
#include <cstdint>
#include "../../paper_2605_16839_b200/csrc/common.cuh"
using namespace cpa;
template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t a = smem_u32(base), b = smem_u32(base + 32768);
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
  long long t0 = clock64();
  if (warp == 0) {
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = umma_desc_sw128(b + (kk & 3) * 32, 16, 1024);
          if (TS) mma_ts(tm + 256, tm + 384 + kk * 8, bd, idesc, 1);
          else mma_ss(tm + 256, umma_desc_sw128(a + (kk & 3) * 32, 16, 1024), bd, idesc, 1);
        }
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}
template <int N, bool TS> void run(long long* c) {
  int iters = 1000;
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k<N, TS><<<148, 128, 70000>>>(c, iters); cudaDeviceSynchronize();
  k<N, TS><<<148, 128, 70000>>>(c, iters); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (iters * 8.0);
  double ideal = 128.0 * N / 256.0;
  printf("N=%3d %s: %.1f cycles/MMA (ideal %.0f) -> %.0f%% ; err=%s\n", N, TS ? "TS" : "SS", per, ideal, 100 * ideal / per,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* c; cudaMalloc(&c, 1 << 16);
  run<64, false>(c); run<128, false>(c); run<256, false>(c);
  run<64, true>(c); run<128, true>(c); run<256, true>(c);
  return 0;
}
