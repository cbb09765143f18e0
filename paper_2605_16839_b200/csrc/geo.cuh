// geo.cuh -- chunk geometry passed by value to every libcpa kernel.
#pragma once
#include <stdint.h>

namespace cpa {

struct Geo {
  int B, Hq, Hkv, d, bs, E, Gn, C, P, L;
  int nqb, nkvb, pb, nwords;
  int R, Rpad;       // estimator rows per group: R = E*nqb, Rpad = 128*ceil(R/128)
  int maxb;          // page_table row length
  int kv_per_q;      // Hq/Hkv
  float scale;       // softmax / score scale
  float ln_alpha;
  uint32_t flags;
  long long q_stride;  // elements between tokens of q / o
  long long b_stride;  // elements between batch entries of q / o (C*q_stride; other for pseudo-batches)
};

// KV head of execution group g: its query heads [g*E, (g+1)*E) all read KV head (g*E)/(Hq/Hkv).
__host__ __device__ inline int group_kv_head(const Geo& g, int grp) {
  return (grp * g.E) / g.kv_per_q;
}

// Arguments of the paged-attention kernels. Block list of a CTA, in priority order:
//   mask    != nullptr: the set bits of its per-(b, h, q-block) 2D mask row (block-sparse execution,
//                       1-CTA kernel only; mask layout [B, Hq, nqb, nwords] u32, LSB-first);
//   indptr  != nullptr: its CSR table row b*Gn + g (zero-copy paged execution);
//   else               every block (dense baseline).
// Output: the normalised O tile of every CTA is stored to each of outs[0 .. n_out): outs[0] is the
// call's own output; with a peer exchange (cpa_chunk_step_peer) outs[k] is rank (rank+k) % W's
// gathered buffer, already offset to this rank's head slice and mapped into this process (P2P over
// NVLink), so the all-gather of the head outputs happens in the epilogue, tile by tile.
constexpr int kMaxOut = 8;
struct AttnArgs {
  const int32_t* page_table;
  const int32_t* indptr;
  const int32_t* indices;
  const uint32_t* mask;
  int out_f32;
  int n_out;             // >= 1
  long long o_stride;    // elements between tokens of every output
  long long o_bstride;   // elements between batch entries of every output
  void* outs[kMaxOut];
};

// Stream-K schedule of the persistent 2-CTA attention (attention_2cta.cu), in the call's workspace.
// Unit u = (b, group, q-tile, head pair) in the non-persistent cluster order; its visible table
// prefix is entries [start[u], start[u] + len[u]) of kv_indices, the first nd[u] of them fully
// visible; pre[] = exclusive prefix sum of len (pre[units] = total pages). Segment s = the seg_units
// units of one (b, group) row; cluster c processes the c-th of `clusters` equal page shares of every
// segment, in segment order. A unit cut by a share boundary leaves partials in
// part_o [clusters][segments][2][256][d] fp32 / part_ml [...][256][2] (slot 0: the share's first
// item, slot 1: its last).
struct SkSched {
  int* pre;
  int* len;
  int* start;
  int* nd;
  float* part_o;
  float* part_ml;
  int* fix;  // per share (c, s): [0] = #parts (0: nothing to merge here), [1] = unit, [2..] part slots
  int units, clusters, segments, seg_units;
};
constexpr int kSkFixStride = 2 + 80;  // ints per share in SkSched::fix (<= 80 clusters)

// Arguments of the peer completion barrier (peer.cu).
struct PeerSig {
  uint32_t* pads[kMaxOut];  // pads[w]: rank w's signal pad u32[W], mapped into this process
  int world, rank;
  uint32_t epoch;
  int* status;              // optional: 1 + the peer that did not arrive within the timeout
  unsigned long long timeout_ns;
};

}  // namespace cpa
