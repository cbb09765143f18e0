// tcgen05 (cta_group::2, M=256 N=128 K=16, SS) throughput while other warps of the same SMs run
// softmax-like ALU / MUFU work: does CUDA-core activity slow the tensor pipe?
//   mode 0: other warps idle; 1: MUFU.EX2 stream; 2: FFMA2 stream; 3: softmax mix (FFMA2 + EX2 + FMNMX3
//   + F2FP); 4: TMEM load / store stream (columns the MMA does not touch)
// One cluster per SM pair on all 148 SMs; prints cycles per MMA (issuing warp, leader CTA of cluster 0).
#include <cstdio>
#include <cstdint>
#include "../../paper_2605_16839_b200/csrc/common.cuh"
using namespace cpa;

constexpr int kWorkWarps = 8;
constexpr int kMmas = 8192;

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * (2 + kWorkWarps), 1)
    k(long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t done_bar;
  __shared__ volatile int stop;
  const uint32_t warp = warp_id(), lane = lane_id(), cta = cluster_ctarank();
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { stop = 0; mbar_init(&done_bar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  if (warp == 1) tmem_alloc2<512>(&slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
  constexpr uint32_t idesc = umma_idesc_bf16(256, 128, 0, 0);
  if (warp == 0) {
    if (cta == 0) {
      const long long t0 = clock64();
      for (int it = 0; it < kMmas; it += 8) {
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma2_ss(tm, umma_desc_sw128(a + (kk & 3) * 32, 16, 1024), umma_desc_sw128(b + (kk & 3) * 32, 16, 1024),
                    idesc, 1);
        }
        __syncwarp();
      }
      const long long t_issued = clock64();
      if (elect_one()) tc_commit2(&done_bar);
      __syncwarp();
      mbar_wait(&done_bar, 0);
      const long long t1 = clock64();
      if (lane == 0 && blockIdx.x == 0) { out[MODE] = t1 - t0; out[5] = t_issued - t0; }
      // issue-queue probe (mode 0 only, after the stream drained): cycles to issue 1, 2, 4, 8, 16, 32
      // back-to-back MMAs (returns once the last is accepted), then until they complete
      if (MODE == 0) {
        int ph = 1;
        for (int q = 0; q < 6; ++q) {
          const int cnt = 1 << q;
          const long long s0 = clock64();
          if (elect_one()) {
            for (int i = 0; i < cnt; ++i)
              mma2_ss(tm, umma_desc_sw128(a, 16, 1024), umma_desc_sw128(b, 16, 1024), idesc, 1);
          }
          __syncwarp();
          const long long s1 = clock64();
          if (elect_one()) tc_commit2(&done_bar);
          __syncwarp();
          mbar_wait(&done_bar, ph);
          ph ^= 1;
          const long long s2 = clock64();
          if (lane == 0 && blockIdx.x == 0) { out[8 + 2 * q] = s1 - s0; out[9 + 2 * q] = s2 - s0; }
        }
      }
    } else {
      mbar_wait(&done_bar, 0);  // the peer's completion arrives here too (multicast commit)
      if (MODE == 0)
        for (int q = 0, ph = 1; q < 6; ++q, ph ^= 1) mbar_wait(&done_bar, ph);
    }
    if (lane == 0) stop = 1;
  } else if (warp >= 2) {
    float acc = (float)threadIdx.x * 1e-3f;
    float2 f2 = make_float2(acc, acc + 1.f);
    uint32_t pk = 0;
    uint32_t r[32];
    const uint32_t tcol = tm + ((uint32_t)(((warp - 2) & 3) * 32) << 16) + 256 + ((warp - 2) >> 2) * 64;
    while (!stop) {
#pragma unroll 4
      for (int i = 0; i < 64; ++i) {
        if (MODE == 1) { acc = fast_exp2(acc * 0.999f - 0.5f); }
        if (MODE == 2) { f2 = ffma2(f2, 0.999f, 0.37f); }
        if (MODE == 3) {
          float2 x = ffma2(f2, 0.999f, -0.37f);
          float e0 = fast_exp2(x.x), e1 = fast_exp2(x.y);
          acc = fmax3(acc, e0, e1);
          pk ^= pack_f16x2(e0, e1);
          f2 = make_float2(e1, e0);
        }
      }
      if (MODE == 4) {
        tmem_ld32(tcol, r);
        tmem_wait_ld();
        tmem_st16(tcol, *reinterpret_cast<uint32_t(*)[16]>(r));
        tmem_wait_st();
      }
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc + f2.x + f2.y + (float)pk + (MODE == 4 ? __uint_as_float(r[3]) : 0.f);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) { tc_fence_after(); tmem_dealloc2<512>(tm); }
}

template <int MODE>
void run(long long* d_out, float* sink, int sms) {
  auto kern = k<MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 + 1024);
  kern<<<sms, 32 * (2 + kWorkWarps), 49152 + 1024>>>(d_out, sink);
  cudaDeviceSynchronize();
  kern<<<sms, 32 * (2 + kWorkWarps), 49152 + 1024>>>(d_out, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[24];
  cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
  const char* names[] = {"idle", "MUFU.EX2 stream", "FFMA2 stream", "softmax mix", "TMEM ld/st stream"};
  printf("mode %d (%-17s): %.1f cycles per M=256 N=128 K=16 MMA (ideal 64), issue loop %.1f cycles per MMA  %s\n",
         MODE, names[MODE], (double)h[MODE] / kMmas, (double)h[5] / kMmas, cudaGetErrorString(e));
  if (MODE == 0)
    for (int q = 0; q < 6; ++q)
      printf("  %2d back-to-back MMAs: issue returns after %lld cycles, complete after %lld\n", 1 << q, h[8 + 2 * q],
             h[9 + 2 * q]);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 24 * 8);
  cudaMalloc(&sink, (size_t)sms * 1024 * sizeof(float));
  run<0>(d_out, sink, sms);
  run<1>(d_out, sink, sms);
  run<2>(d_out, sink, sms);
  run<3>(d_out, sink, sms);
  run<4>(d_out, sink, sms);
  return 0;
}
