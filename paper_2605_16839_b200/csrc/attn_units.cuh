// attn_units.cuh -- work units of the 2-CTA attention kernels (attention_2cta.cu, attention_ks4.cu):
// u = (b, execution group, 128-token q-tile, head pair), heaviest q-tile first within a group, and the
// unit's visible prefix of its CSR table row (ascending logical block ids).
#pragma once
#include "common.cuh"
#include "geo.cuh"

namespace cpa {

// Coordinates of work unit u (cluster order of the non-persistent grid).
struct Unit {
  int b, grp, qt, hp;
};
__device__ __forceinline__ Unit unit_coords(const Geo& g, int u) {
  const int HP = g.E / 2, nqt = (g.C + 127) / 128;
  Unit r;
  r.hp = u % HP;
  r.qt = nqt - 1 - (u / HP) % nqt;
  const int bg = u / (HP * nqt);
  r.grp = bg % g.Gn;
  r.b = bg / g.Gn;
  return r;
}

// Visible table prefix of unit u: first entry `start`, `n` entries with block <= the tile's last
// query position, of which the first `nd` are fully visible to every row (no causal mask).
__device__ __forceinline__ void unit_table(const Geo& g, const AttnArgs& args, int u, int* start, int* n, int* nd) {
  const Unit c = unit_coords(g, u);
  const int p0 = c.qt * 128;
  const int jmax = (g.P + min(p0 + 127, g.C - 1)) / g.bs;
  const int jfull = (g.P + p0 + 1) / g.bs - 1;  // last block with j*bs + bs - 1 <= P + p0
  if (args.indptr == nullptr) {
    *start = 0;
    *n = jmax + 1;
    *nd = min(jfull + 1, jmax + 1);
    return;
  }
  const int r = c.b * g.Gn + c.grp;
  const int s = args.indptr[r];
  int lo = s, hi = args.indptr[r + 1];  // first index with kv_indices > jmax
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (args.indices[mid] <= jmax) lo = mid + 1; else hi = mid;
  }
  const int e = lo;
  lo = s;
  hi = e;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (args.indices[mid] <= jfull) lo = mid + 1; else hi = mid;
  }
  *start = s;
  *n = e - s;
  *nd = lo - s;
}

// Number of entries <= key of the ascending list a[0, n), by a whole warp: a 32-ary search, i.e.
// ceil(log32 n) rounds of dependent loads (2 for n <= 1024) instead of a lane's log2(n) chain (each
// step an L2 round trip that the cluster's prologue would otherwise wait on).
__device__ __forceinline__ int warp_count_le(const int32_t* __restrict__ a, int n, int key) {
  const int lane = (int)lane_id();
  int lo = 0, hi = n;  // the count c satisfies lo <= c <= hi
  while (lo < hi) {
    const int step = (hi - lo + 31) >> 5;
    const int pos = lo + (lane + 1) * step - 1;
    const bool le = pos < hi && __ldg(a + pos) <= key;
    const int k = __popc(__ballot_sync(0xffffffffu, le));  // probes <= key (they ascend)
    const int nlo = lo + k * step;
    hi = min(hi, nlo + step - 1);
    lo = nlo;
  }
  return lo;
}

// unit_table by the whole warp (same results): the visible prefix and its fully visible part.
__device__ __forceinline__ void unit_table_warp(const Geo& g, const AttnArgs& args, int u, int* start, int* n,
                                                int* nd) {
  const Unit c = unit_coords(g, u);
  const int p0 = c.qt * 128;
  const int jmax = (g.P + min(p0 + 127, g.C - 1)) / g.bs;
  const int jfull = (g.P + p0 + 1) / g.bs - 1;
  if (args.indptr == nullptr) {
    *start = 0;
    *n = jmax + 1;
    *nd = min(jfull + 1, jmax + 1);
    return;
  }
  const int r = c.b * g.Gn + c.grp;
  const int s = __ldg(args.indptr + r), len = __ldg(args.indptr + r + 1) - s;
  *start = s;
  // Fast path: a row ending with exactly the chunk's blocks pb .. nkvb-1 (always so on the estimator
  // path: they are forced) has both counts in closed form (jmax >= pb, jfull >= pb - 1).
  // Checked with two parallel loads (first and last tail entry; the row is strictly ascending), since a
  // caller's MASK_IN tables may lack chunk blocks; otherwise the 32-ary searches.
  const int nch = g.nkvb - g.pb;
  if (nch > 0 && len >= nch) {
    const int v = lane_id() < 2 ? __ldg(args.indices + s + (lane_id() == 0 ? len - nch : len - 1)) : 0;
    const int first = __shfl_sync(0xffffffffu, v, 0), last = __shfl_sync(0xffffffffu, v, 1);
    if (first == g.pb && last == g.nkvb - 1) {
      const int prefix = len - nch;
      *n = prefix + (jmax - g.pb + 1);
      *nd = min(*n, prefix + max(0, jfull - g.pb + 1));
      return;
    }
  }
  *n = warp_count_le(args.indices + s, len, jmax);
  *nd = warp_count_le(args.indices + s, *n, jfull);
}

}  // namespace cpa
