// launch.cuh -- kernel launch with optional programmatic dependent launch (PDL).
//
// The chunk step is a chain append -> pool_q -> block_scores -> mask_union -> attention in one
// stream. With PDL each kernel may be scheduled while its predecessor is still running: it triggers
// its dependents early (pdl_trigger) and calls pdl_wait() before touching anything a predecessor
// writes or reads, so launch latency and prologues (barrier init, TMEM alloc, descriptor prefetch)
// overlap the predecessor's tail, and pool_q overlaps the append outright (it does not read its
// output; it waits at its end so that its completion still implies the append's).
#pragma once
#include <cuda_runtime.h>

#include "geo.cuh"

namespace cpa {

constexpr uint32_t kFlagNoPdl = 8192u;  // CPA_F_NO_PDL
inline bool use_pdl(const Geo& g) { return (g.flags & kFlagNoPdl) == 0; }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace cpa
