// out_store.cuh -- epilogue store of normalised O rows to every destination of AttnArgs.
// With a peer exchange the same 32 values go to each rank's gathered buffer over NVLink (P2P
// stores), so the head all-gather is done tile by tile inside the attention kernel.
#pragma once
#include "common.cuh"
#include "geo.cuh"

namespace cpa {

// v[0..32) are output columns [off, off+32) of one (b, p, h) row (elements, from each outs[k]).
CPA_DEV void store_o_row32(const AttnArgs& a, long long off, const float (&v)[32]) {
  if (a.out_f32) {
#pragma unroll
    for (int k = 0; k < kMaxOut; ++k) {
      if (k < a.n_out) {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.outs[k]) + off);
#pragma unroll
        for (int c = 0; c < 32; c += 4) dst[c / 4] = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
      }
    }
  } else {
    uint4 w[4];
#pragma unroll
    for (int c = 0; c < 32; c += 8)
      w[c / 8] = make_uint4(pack_bf16x2(v[c], v[c + 1]), pack_bf16x2(v[c + 2], v[c + 3]),
                            pack_bf16x2(v[c + 4], v[c + 5]), pack_bf16x2(v[c + 6], v[c + 7]));
#pragma unroll
    for (int k = 0; k < kMaxOut; ++k) {
      if (k < a.n_out) {
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.outs[k]) + off);
#pragma unroll
        for (int c = 0; c < 4; ++c) dst[c] = w[c];
      }
    }
  }
}

}  // namespace cpa
