// tables.cu -- §8 rows a3/a4/a5: threshold -> 2D mask -> Q-block union -> intra-group union
// -> CSR block tables, integer work with warp ballots / popc and a block prefix sum.
//
// a3  M[b,h,i,j] = causal && (m - m* >= ln(alpha) || j >= pb || (SINK && j == 0))
//     (PAPER.md:174, 538 fully-open chunk)
// a4  G[b,g,j]   = OR_{h in H(g)} OR_i M[b,h,i,j]
// a5  T[b,g]     = {j | G[b,g,j]}, CSR rows r = b*Gn + g, ascending j (
//                  SPEC.md:305-311, 343)
#include "common.cuh"
#include "geo.cuh"
#include "launch.cuh"

namespace cpa {

// Exclusive-scan CSR of the G words (row-major over r = b*Gn + g, then word) by one CTA of any
// multiple-of-32 size: per tile of blockDim words a block-wide scan of the popcounts with a running
// carry, then every word scatters its set bits (ascending j within a row). gwords is read with
// .cg loads: other CTAs of the same grid wrote it.
__device__ void csr_block(const uint32_t* gwords, const Geo& g, int32_t* indptr, int32_t* indices) {
  __shared__ int warp_sums[32];
  __shared__ int carry_s;
  const int nrows = g.B * g.Gn;
  const int total = nrows * g.nwords;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (int base = 0; base < total; base += blockDim.x) {
    const int x = base + tid;
    const uint32_t word = x < total ? __ldcg(gwords + x) : 0u;
    const int cnt = __popc(word);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int v = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (lane < nw) warp_sums[lane] = v;  // inclusive prefix of warp totals
    }
    __syncthreads();
    const int carry = carry_s;
    const int excl = carry + (wid > 0 ? warp_sums[wid - 1] : 0) + incl - cnt;
    if (x < total) {
      const int row = x / g.nwords, wi = x % g.nwords;
      if (wi == 0) indptr[row] = excl;
      uint32_t rem = word;
      int pos = excl;
      while (rem) {
        const int bit = __ffs(rem) - 1;
        rem &= rem - 1;
        indices[pos++] = wi * 32 + bit;
      }
    }
    __syncthreads();
    if (tid == blockDim.x - 1) carry_s = carry + warp_sums[nw - 1];
    __syncthreads();
  }
  if (tid == 0) indptr[nrows] = carry_s;
}

// One CTA per (word w of 32 kv blocks, execution group bg). Thread t handles estimator rows
// r = t, t+blockDim, ... (r = hl*nqb + i). Each row forms its 32-bit mask word, the CTA ORs the
// words of all its rows (Q-block union and intra-group union in one reduction). The CSR tables are
// built by k_csr (next kernel, one 1024-thread CTA, PDL-overlapped with this one).
__global__ void __launch_bounds__(128)
    k_mask_union(const float* __restrict__ scores, const int* __restrict__ mstar_key, Geo g,
                 const uint32_t* __restrict__ mask_in, uint32_t* __restrict__ mask_out,
                 uint32_t* __restrict__ gwords, int* __restrict__ dev_status, unsigned* __restrict__ done,
                 int32_t* __restrict__ indptr, int32_t* __restrict__ indices) {
  const int w = blockIdx.x, bg = blockIdx.y;
  const int b = bg / g.Gn, grp = bg % g.Gn;
  const bool sink = (g.flags & 1u) != 0;
  pdl_wait();     // scores / row max (block_scores) or mask_in complete
  pdl_trigger();  // the attention may start its prologue (it waits for this grid before the tables)
  const int jbase = w * 32;
  // valid kv blocks of this word: j < nkvb
  const int nvalid = min(32, g.nkvb - jbase);
  const uint32_t in_range = nvalid >= 32 ? 0xffffffffu : ((1u << nvalid) - 1u);
  uint32_t acc = 0;
  for (int r = threadIdx.x; r < g.R; r += blockDim.x) {
    const int hl = r / g.nqb, i = r % g.nqb, h = grp * g.E + hl;
    const long long mw = (((long long)b * g.Hq + h) * g.nqb + i) * g.nwords + w;
    uint32_t bits;
    if (mask_in != nullptr) {
      bits = __ldg(mask_in + mw) & in_range;
    } else {
      const float mstar = key_float(__ldg(mstar_key + (long long)bg * g.Rpad + r));
      const int jmax = g.pb + i;  // causal-valid blocks j <= pb + i
      // all 32 loads first (each a coalesced 128 B warp request), then the threshold
      float mv[32];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const int j = jbase + jj;
        mv[jj] = (j <= jmax && j < g.nkvb) ? __ldg(scores + ((long long)bg * g.nkvb + j) * g.Rpad + r) : -INFINITY;
      }
      bits = 0;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const int j = jbase + jj;
        const bool valid = j <= jmax && j < g.nkvb;
        const bool keep = (mv[jj] - mstar >= g.ln_alpha) || (j >= g.pb) || (sink && j == 0);
        bits |= (uint32_t)(valid && keep) << jj;
      }
      if (mask_out != nullptr) mask_out[mw] = bits;
    }
    acc |= bits;
  }
  acc = __reduce_or_sync(0xffffffffu, acc);
  __shared__ uint32_t red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t word = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) word |= red[k];
    gwords[(long long)bg * g.nwords + w] = word;
    if (mask_in != nullptr && dev_status != nullptr) {
      // open-chunk rule: every chunk block [pb, nkvb) must be present
      uint32_t need = 0;
      for (int jj = 0; jj < nvalid; ++jj)
        if (jbase + jj >= g.pb) need |= 1u << jj;
      if ((word & need) != need) atomicCAS(dev_status, 0, 1 + bg);
    }
  }
}

// a5: CSR of the G words, one CTA (csr_block), after k_mask_union (PDL: resident early, waits for it).
__global__ void __launch_bounds__(1024) k_csr(const uint32_t* __restrict__ gwords, Geo g, int32_t* __restrict__ indptr,
                                              int32_t* __restrict__ indices) {
  pdl_wait();
  pdl_trigger();
  csr_block(gwords, g, indptr, indices);
}

cudaError_t launch_tables(const float* scores, const int* mstar_key, const Geo& g,
                          const uint32_t* mask_in, uint32_t* mask_out, uint32_t* gwords,
                          int* dev_status, unsigned* done, int32_t* indptr, int32_t* indices, cudaStream_t st,
                          int* launches) {
  (void)done;
  *launches += 2;
  cudaError_t e = launch_ex(k_mask_union, dim3(g.nwords, g.B * g.Gn), dim3(128), 0, st, use_pdl(g), scores, mstar_key,
                            g, mask_in, mask_out, gwords, dev_status, done, indptr, indices);
  if (e != cudaSuccess) return e;
  return launch_ex(k_csr, dim3(1), dim3(1024), 0, st, use_pdl(g), (const uint32_t*)gwords, g, indptr, indices);
}

// Fig. 7(c) ablation ("the same unioned block mask"; SPEC.md:447 q-uniform expansion):
// Mq[b,h,i,j] = [j in T[b, h/E]] && j <= jmax(i), the table row of h's execution group repeated over
// every q-block i and cut to the causal-valid tiles. One CTA per (q-block i, b*Hq + h), word-wise
// OR in shared memory.
__global__ void __launch_bounds__(128)
    k_expand_tables(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices, Geo g,
                    uint32_t* __restrict__ mask) {
  extern __shared__ uint32_t words[];
  const int i = blockIdx.x, bh = blockIdx.y;
  const int b = bh / g.Hq, h = bh % g.Hq;
  const int r = b * g.Gn + h / g.E;
  const int jmax = (g.P + min((i + 1) * g.bs, g.C) - 1) / g.bs;
  for (int w = threadIdx.x; w < g.nwords; w += blockDim.x) words[w] = 0u;
  __syncthreads();
  const int end = indptr[r + 1];
  for (int k = indptr[r] + threadIdx.x; k < end; k += blockDim.x) {
    const int j = indices[k];
    if (j <= jmax) atomicOr(&words[j >> 5], 1u << (j & 31));
  }
  __syncthreads();
  uint32_t* dst = mask + ((long long)bh * g.nqb + i) * g.nwords;
  for (int w = threadIdx.x; w < g.nwords; w += blockDim.x) dst[w] = words[w];
}

cudaError_t launch_expand_tables(const int32_t* indptr, const int32_t* indices, const Geo& g, uint32_t* mask,
                                 cudaStream_t st, int* launches) {
  k_expand_tables<<<dim3(g.nqb, g.B * g.Hq), 128, g.nwords * 4, st>>>(indptr, indices, g, mask);
  *launches += 1;
  return cudaGetLastError();
}

}  // namespace cpa
