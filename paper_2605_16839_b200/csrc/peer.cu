// peer.cu -- §8(e): completion barrier of the fused head-output all-gather over NVLink peer memory.
//
// The chunk step shards by execution group (every table is per (b, g)), so rank r
// of W computes the heads of its KV groups and its attention epilogue stores each O tile straight
// into every rank's gathered [B, C, Hq_total, d] buffer (out_store.cuh). What is left of the
// all-gather is this barrier: rank r tells every peer "my slice of your buffer is written" and
// waits until every peer has told it the same, after which its own gathered buffer is complete.
//
// Signal pads: rank w owns u32 pad[W] (mapped into every rank); slot pad_w[r] is written only by
// rank r, with strictly increasing epochs, so no reset is needed between calls. The epoch is kept on
// the device (epoch = 1 + the last one this rank posted, read from its own pad's slot r), so a
// captured CUDA graph of the step replays with fresh epochs; a nonzero host epoch overrides it.
#include "common.cuh"
#include "geo.cuh"

namespace cpa {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One warp; lane w < W signals peer w and then waits for peer w's signal. The stores of the
// preceding attention kernel (same stream) are ordered before the release by the system-scope fence.
__global__ void __launch_bounds__(32) k_peer_barrier(PeerSig s) {
  const int w = threadIdx.x;
  uint32_t epoch = s.epoch;
  if (epoch == 0) {  // device-side epoch: every lane reads it before lane `rank` posts the new one
    epoch = __shfl_sync(0xffffffffu, w == 0 ? ld_acquire_sys(s.pads[s.rank] + s.rank) : 0u, 0) + 1u;
  }
  if (w >= s.world) return;
  __threadfence_system();
  st_release_sys(s.pads[w] + s.rank, epoch);
  const uint32_t* mine = s.pads[s.rank] + w;
  const unsigned long long t0 = global_ns();
  while ((int)(ld_acquire_sys(mine) - epoch) < 0) {
    if (global_ns() - t0 > s.timeout_ns) {  // a peer never arrived: report, do not hang the GPU
      if (s.status) atomicCAS(s.status, 0, 1 + w);
      break;
    }
    __nanosleep(64);
  }
}

cudaError_t launch_peer_barrier(const PeerSig& s, cudaStream_t st, int* launches) {
  ++*launches;
  k_peer_barrier<<<1, 32, 0, st>>>(s);
  return cudaGetLastError();
}

}  // namespace cpa
