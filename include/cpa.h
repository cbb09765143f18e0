/*
 * cpa.h -- C ABI of libcpa.so, the B200 (sm_100a) chunked-prefill hot path of
 * CompactAttention (arXiv 2605.16839, "Block-Union KV Selection").
 *
 * One chunk step = three stages (§3.1):
 *   (1) pattern search: per (batch b, query head h, q-block i, kv-block j) block mask
 *       M[b,h,i,j] from a max-threshold estimator over the accumulated KV cache
 *       (keep rule SPEC.md:220-238, pooled-query variant SPEC.md:269);
 *   (2) selection: Q-block union  Mbar[b,h,j] = OR_i M[b,h,i,j]
 *                  intra-group union G[b,g,j] = OR_{h in H(g)} Mbar[b,h,j]
 *                  table T[b,g] = {j | G[b,g,j] = 1} as CSR kv_indptr/kv_indices
 *                  (PAPER.md:206, 533-534);
 *   (3) execution: causal attention of the whole chunk over only the tabled blocks,
 *       read in place from the paged KV cache.
 *
 * Conventions (all entry points):
 *   - Host-callable, stream-ordered on `stream` (a cudaStream_t passed as void*; NULL =
 *     legacy default stream). They never synchronize, never allocate or free device
 *     memory and keep no pointer after they return. Re-entrant.
 *   - Every pointer argument is a DEVICE pointer owned by the caller unless stated.
 *   - Synchronous validation errors are returned as a cpa_status and leave every output
 *     untouched; cpa_last_error() (thread-local) gives the detail. Asynchronous CUDA
 *     faults surface on a later CUDA call (standard CUDA semantics).
 *   - Inputs are bf16. Non-finite inputs are undefined behaviour.
 *   - No CPU fallback exists: without an sm_100a device every call returns
 *     CPA_ERR_CUDA / CPA_ERR_UNSUPPORTED.
 *
 * Notation: B batch, Hq query heads, Hkv KV heads,
 *   E = exec_group_size query heads per execution group ("a KV group by default",
 *   PAPER.md:203; 4 under sub-KV-group union), Gn = Hq/E groups,
 *   d head_dim, bs block_size (= page size = q-block size),
 *   C chunk_len, P prefix_len (tokens already cached; P % bs == 0), L = P + C,
 *   nqb = ceil(C/bs), nkvb = ceil(L/bs), pb = P/bs, nwords = ceil(nkvb/32).
 *   Query position p in [0,C) sits at absolute position P+p and may attend to
 *   absolute positions t <= P+p.
 */
#ifndef CPA_H_
#define CPA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CPA_VERSION 1

#if defined(__GNUC__)
#define CPA_API __attribute__((visibility("default")))
#else
#define CPA_API
#endif

typedef enum {
  CPA_OK = 0,
  CPA_ERR_NULL = 1,        /* a required pointer is NULL */
  CPA_ERR_SHAPE = 2,       /* Hq % Hkv, E does not divide Hq/Hkv, C < 1, nkvb > max_blocks_per_seq,
                              B < 1 (SPEC.md:52, 134 shape errors) */
  CPA_ERR_UNSUPPORTED = 3, /* head_dim not in {64,128}; block_size not in {16,32,64,128};
                              no sm_100 device */
  CPA_ERR_MISALIGNED = 4,  /* P % bs != 0 (SPEC.md:167 uniform prefix, R8);
                              a pointer not 16-byte aligned; a stride not a multiple of 8 */
  CPA_ERR_ALPHA = 5,       /* alpha not in (0, 1] */
  CPA_ERR_WORKSPACE = 6,   /* ws == NULL or ws_bytes < cpa_workspace_bytes() */
  CPA_ERR_CAPACITY = 7,    /* tables->capacity < B*Gn*nkvb */
  CPA_ERR_CUDA = 8         /* a CUDA runtime/driver call failed (see cpa_last_error) */
} cpa_status;

/* flags */
enum {
  CPA_F_SINK = 1u,        /* always keep kv-block 0 (default on in the binding) */
  CPA_F_MASK_IN = 2u,     /* skip the estimator: M is read from tables->mask_bits */
  CPA_F_MASK_OUT = 4u,    /* also write M to tables->mask_bits */
  CPA_F_SCORES_OUT = 8u,  /* also write block scores / row max to tables->scores / ->row_max */
  CPA_F_OUT_F32 = 16u,    /* O is fp32 instead of bf16 (parity/debug) */
  CPA_F_EXACT_SCORES = 32u, /* SPEC.md:223 exact tile-max scorer (full QK^T, max over every causal
                               (p, t) pair of the tile) instead of the pooled-query estimator */
  CPA_F_P_BF16 = 256u,    /* ablation: round softmax P to bf16 instead of fp16 before P.V (K3) */
  CPA_F_NO_2CTA = 512u,   /* ablation: single-CTA attention kernel instead of the cta_group::2 pair */
  CPA_F_NO_PERSIST = 1024u, /* ablation: one cluster per work unit instead of the persistent stream-K grid */
  CPA_F_PERSIST = 2048u,  /* ablation / tests: persistent stream-K grid whenever B*Gn <= 4 */
  CPA_F_V_F16 = 4096u,    /* the V pool holds fp16 (cpa_append_kv converts the bf16 chunk; exact for bf16
                             values in fp16's normal range, i.e. the conversion the attention kernels
                             otherwise do per page; |v| > 65504 saturates to +-65504, |v| < 2^-14 becomes
                             an fp16 subnormal): the attention kernels skip their V conversion.
                             Incompatible with CPA_F_P_BF16. The bf16-pool path converts V per page with
                             the same saturating rounding (P.V runs in fp16 either way, K3). */
  CPA_F_NO_PDL = 8192u,   /* ablation: launch the step's kernels without programmatic dependent launch */
  CPA_F_ATTN_RS = 16384u, /* ablation: row-split 2-CTA attention (one O, three S buffers; d=128, bs=128)
                             instead of the key-split one (two O accumulators, two S buffers) */
  CPA_F_ATTN_KS4 = 65536u /* 2-CTA attention with four key slices sharing one running max (one O, three S
                             buffers; d=128, bs=128, CPA_F_V_F16, per-unit grid) */
};

typedef struct {
  int32_t batch;           /* B >= 1 */
  int32_t num_q_heads;     /* Hq (heads present in q/o for this call) */
  int32_t num_kv_heads;    /* Hkv (heads present in the cache for this call) */
  int32_t head_dim;        /* d in {64, 128} */
  int32_t block_size;      /* bs in {16, 32, 64, 128}; page size == selection block size */
  int32_t exec_group_size; /* E; 0 => Hq/Hkv. Must divide Hq/Hkv. */
  int32_t chunk_len;       /* C >= 1; the last chunk of a prompt may be shorter */
  int32_t prefix_len;      /* P >= 0, P % bs == 0 */
  float alpha;             /* keep threshold in (0,1]; paper's CA-FP uses 0.06 */
  float sm_scale;          /* logit scale; 0 => 1/sqrt(d) */
  uint32_t flags;          /* CPA_F_* */
  int64_t q_token_stride;  /* elements between consecutive tokens of q / o; 0 => Hq*d.
                              Lets a rank pass a head slice of a larger [B,C,Hq_total,d] tensor. */
} cpa_params;

/* Paged KV cache (PAPER.md:237-249 KV-head-major pages).
 * Element (physical page pg, kv head h, token slot t, dim e) of K (resp. V) lives at
 *   k_pages + pg*page_stride + h*head_stride + t*head_dim + e      (bf16 elements)
 * so every (page, kv head) is one contiguous [bs, d] region. A pool laid out
 * [num_pages, Hkv, bs, d] has head_stride = bs*d, page_stride = Hkv*bs*d; the paper's
 * per-sequence [B, Hkv, L, d] layout is page = b*nblocks + j, head_stride = L*d,
 * page_stride = bs*d.  Logical block j of sequence b is page page_table[b*max_blocks_per_seq + j].
 * Slots past the end of the sequence in its last page must be finite (pools are
 * zero-initialised by the caller; SURVEY §7 hard part 7). */
typedef struct {
  void* k_pages;                /* bf16 (written only by cpa_append_kv / cpa_chunk_step append) */
  void* v_pages;                /* bf16, or fp16 with CPA_F_V_F16 (same layout) */
  int64_t page_stride;          /* elements; 0 => Hkv*bs*d */
  int64_t head_stride;          /* elements; 0 => bs*d */
  const int32_t* page_table;    /* int32 [B, max_blocks_per_seq], device */
  int32_t max_blocks_per_seq;
  int32_t num_pages;            /* pages addressable from k_pages / v_pages */
} cpa_kv_cache;

/* Per-chunk block tables (CSR over pseudo-rows r = b*Gn + g).
 * kv_indices holds LOGICAL block ids j, ascending within a row; the chunk blocks [pb, nkvb)
 * are always present (fully-open current chunk), so no row is empty. */
typedef struct {
  int32_t* kv_indptr;    /* int32 [B*Gn + 1] (out of cpa_build_tables, in of cpa_paged_attention) */
  int32_t* kv_indices;   /* int32 [capacity] */
  int64_t capacity;      /* >= B*Gn*nkvb */
  uint32_t* mask_bits;   /* optional u32 [B, Hq, nqb, nwords]; bit (j%32) of word j/32 is M[b,h,i,j].
                            Input with CPA_F_MASK_IN, output with CPA_F_MASK_OUT. */
  float* scores;         /* optional fp32 [B, Gn, nkvb, Rpad] (CPA_F_SCORES_OUT): block score
                            m[b, g*E + r/nqb, r%nqb, j] at row r < E*nqb; -inf where j > pb + i.
                            Rpad = 128*ceil(E*nqb/128). */
  float* row_max;        /* optional fp32 [B, Gn, Rpad] (CPA_F_SCORES_OUT): m*[b,h,i] = max_j m */
  int32_t* dev_status;   /* optional int32[1]: with CPA_F_MASK_IN, set to 1 + r for a row r whose
                            mask lacks a chunk block (open-chunk violation); 0 otherwise */
} cpa_tables;

/* Device workspace needed by cpa_build_tables / cpa_paged_attention / cpa_chunk_step (the estimator
 * scratch and the attention's stream-K schedule + partial-output slots share one buffer). */
CPA_API size_t cpa_workspace_bytes(const cpa_params* p);

/* Stages (1)+(2): estimator -> M -> Q-block union -> intra-group union -> CSR tables.
 *   q:     bf16 [B, C, Hq, d] (token stride p->q_token_stride), the chunk's queries.
 *   cache: K pages must already contain tokens [0, L) of every sequence.
 *   out:   kv_indptr / kv_indices written (plus mask_bits / scores per flags).
 * Estimator: qbar[b,h,i] = mean of the valid queries of q-block i;
 *   m[b,h,i,j] = max over keys t of block j with t <= P + last query of block i of
 *   sm_scale * qbar . k_t;  m* = max_j m;  M = causal && (m - m* >= ln(alpha) ||
 *   j >= pb || (SINK && j == 0)). */
CPA_API int cpa_build_tables(const cpa_params* p, const void* q, const cpa_kv_cache* cache,
                     cpa_tables* out, void* ws, size_t ws_bytes, void* stream);

/* Stage (3): O[b,p,h] = sum_{t in A(p)} softmax_t(sm_scale q_p . k_t) v_t with
 *   A(p) = { t : floor(t/bs) in T[b, h/E], t <= P + p }  (absolute coordinates).
 *   tables == NULL => dense causal chunk attention over every block [0, nkvb) (the baseline).
 *   o: bf16 (or fp32 with CPA_F_OUT_F32) [B, C, Hq, d], token stride p->q_token_stride.
 *   ws: >= cpa_workspace_bytes(p) (CPA_ERR_WORKSPACE otherwise). The cta_group::2 path runs one
 *   cluster per work unit (b, group, 128-token q-tile, head pair), or a persistent grid of one cluster
 *   per co-resident SM pair, each taking an equal contiguous share of every (b, group) row's
 *   (unit, page) work, with units cut by a share boundary merged in a fixup kernel. The persistent
 *   grid is chosen for the dense baseline (tables == NULL) when the units do not fill whole waves,
 *   there are at most 4 (b, group) rows and at least 512 KV blocks (measured faster there only);
 *   CPA_F_PERSIST (at most 4 rows) / CPA_F_NO_PERSIST force either grid. */
CPA_API int cpa_paged_attention(const cpa_params* p, const void* q, const cpa_kv_cache* cache,
                        const cpa_tables* tables, void* o, void* ws, size_t ws_bytes,
                        void* stream);

/* One whole chunk step: optional append of the chunk's K/V into the pages
 * (k_chunk/v_chunk bf16 [B, C, Hkv, d], token slots [P, P+C); NULL => already resident),
 * then cpa_build_tables, then cpa_paged_attention over the built tables. */
CPA_API int cpa_chunk_step(const cpa_params* p, const void* q, const void* k_chunk, const void* v_chunk,
                   const cpa_kv_cache* cache, cpa_tables* tables, void* o, void* ws,
                   size_t ws_bytes, void* stream);

/* Append only (SPEC.md:130-138 append_chunk): write k_chunk/v_chunk [B, C, Hkv, d] into
 * token slots [P, P+C) of each sequence's pages. K/V pools are written in place. */
CPA_API int cpa_append_kv(const cpa_params* p, const void* k_chunk, const void* v_chunk,
                  const cpa_kv_cache* cache, void* stream);

/* The first half of cpa_chunk_step: optional append of the chunk's K/V, then the estimator and the
 * tables (rows a0-a5), i.e. cpa_append_kv + cpa_build_tables as one call, so the append and the query
 * pooling may overlap (programmatic dependent launch). cpa_chunk_step == cpa_prepare_chunk followed by
 * cpa_paged_attention over the tables. Arguments and errors as cpa_chunk_step (no o). */
CPA_API int cpa_prepare_chunk(const cpa_params* p, const void* q, const void* k_chunk, const void* v_chunk,
                              const cpa_kv_cache* cache, cpa_tables* tables, void* ws, size_t ws_bytes,
                              void* stream);

/* ---- Multi-GPU: head-group sharding with the output all-gather fused into the attention epilogue.
 * The chunk step shards by execution group with no data-path exchange: every table is per (b, g)
 * (PAPER.md:203-209), so rank r of W owns KV heads [r*Hkv/W, (r+1)*Hkv/W) and their query heads (the
 * attention half of the paper's tensor-parallel setting). The only exchange is the
 * all-gather of the head outputs, which cpa_chunk_step_peer performs inside the attention kernel: each
 * normalised O tile is stored to every rank's gathered buffer through NVLink peer mappings (P2P stores),
 * then a one-warp barrier signals every peer and waits for every peer's signal.
 *
 * Buffers (all DEVICE pointers mapped into the calling process, e.g. CUDA IPC / torch symmetric
 * memory; none is allocated or retained by libcpa):
 *   peer_out[w]:    rank w's gathered output [B, C, W*Hq, d] (Hq = this call's p->num_q_heads, the same
 *                   on every rank), bf16 (fp32 with CPA_F_OUT_F32), token stride out_token_stride
 *                   (0 => W*Hq*d elements). Rank r writes heads [r*Hq, (r+1)*Hq) of every peer_out[w].
 *   peer_signal[w]: rank w's signal pad, uint32 [W], zero-initialised once before the first call.
 *                   Slot w' of rank w's pad is written only by rank w'.
 * epoch: 0 (default) => kept on the device: each call posts 1 + the last epoch this rank posted (read
 *   from its own pad), so the calls stay matched across ranks and a captured CUDA graph of the step
 *   replays correctly; nonzero => that epoch, strictly increasing across calls. The call returns
 *   (stream order) after every rank has posted the epoch, i.e. after every peer_out[rank] is complete.
 * Reuse: a rank must not read its peer_out buffer for call k+1's purposes before that call's barrier,
 *   and must have finished reading call k's contents before ANY rank starts call k+1 (alternate two
 *   buffer sets, or call cpa_peer_barrier with a fresh epoch first).
 * dev_status (optional int32[1]): set to 1 + w if peer w did not post within timeout_ms (0 => 10000);
 *   the barrier then stops waiting instead of hanging the GPU. */
#define CPA_MAX_PEERS 8
typedef struct {
  int32_t world;                  /* W in [1, CPA_MAX_PEERS] */
  int32_t rank;                   /* r in [0, W) */
  void* const* peer_out;          /* HOST array [W] of device pointers (see above) */
  int64_t out_token_stride;       /* elements; 0 => W*Hq*d */
  uint32_t* const* peer_signal;   /* HOST array [W] of device pointers */
  uint32_t epoch;                 /* 0 => device-side epochs (see above) */
  uint32_t timeout_ms;            /* 0 => 10000 */
  int32_t* dev_status;            /* optional */
} cpa_peer_out;

/* cpa_chunk_step with the head-output all-gather fused in (see above): optional append, tables,
 * attention whose epilogue writes every peer_out[w] at this rank's head slice, then the barrier.
 * p describes this rank's shard (Hq, Hkv = its own heads); q / k_chunk / v_chunk / cache / tables as in
 * cpa_chunk_step. Errors: CPA_ERR_NULL (missing peer arrays/pointers), CPA_ERR_SHAPE (W or rank out of
 * range, out_token_stride < W*Hq*d), CPA_ERR_MISALIGNED (a peer pointer not 16B aligned). */
CPA_API int cpa_chunk_step_peer(const cpa_params* p, const void* q, const void* k_chunk, const void* v_chunk,
                                const cpa_kv_cache* cache, cpa_tables* tables, const cpa_peer_out* peers,
                                void* ws, size_t ws_bytes, void* stream);

/* The attention stage alone with the fused all-gather: cpa_paged_attention over `tables` (NULL =>
 * dense) whose epilogue writes every peer_out[w] at this rank's head slice, then the barrier; i.e. the
 * last two stages of cpa_chunk_step_peer, for callers that run append / cpa_build_tables separately
 * (bench.py times the attention kernel inside the step this way). Errors as cpa_chunk_step_peer. */
CPA_API int cpa_paged_attention_peer(const cpa_params* p, const void* q, const cpa_kv_cache* cache,
                                     const cpa_tables* tables, const cpa_peer_out* peers, void* ws,
                                     size_t ws_bytes, void* stream);

/* The barrier alone (signal every peer with `epoch`, wait for all); peer_out is not used. */
CPA_API int cpa_peer_barrier(const cpa_peer_out* peers, void* stream);

/* NEXT-3 execution ablation only ("CompactAttention-FP (Copy)"): gather the
 * tabled K/V pages of every (b, g) row into a compact pool in `ws` (an explicit KV copy, exactly what
 * the zero-copy path avoids), then run the same attention kernel over the compact pool through a
 * per-row page table; causal masking stays in absolute positions (logical block ids are kept).
 * Output equals cpa_paged_attention with the same tables. ws: cpa_copy_workspace_bytes(). */
CPA_API size_t cpa_copy_workspace_bytes(const cpa_params* p);
CPA_API int cpa_paged_attention_copy(const cpa_params* p, const void* q, const cpa_kv_cache* cache,
                                     const cpa_tables* tables, void* o, void* ws, size_t ws_bytes, void* stream);

/* NEXT-3 execution ablation only ("The block-sparse variant executes this mask directly
 * with a block-sparse kernel"; SPEC.md:440-449 exec_block_sparse). Each (b, h, q-block i) tile runs
 * over the KV blocks set in ITS OWN row of the 2D mask, one query head per CTA (no GQA sharing of the
 * K/V tiles), the mask bits interpreted inside the kernel:
 *   O[b,p,h] = sum_{t in A(p)} softmax_t(sm_scale q_p . k_t) v_t,
 *   A(p) = { t : mask[b, h, p/bs, t/bs] = 1, t <= P + p }.
 *   mask: u32 [B, Hq, nqb, nwords] device, layout of cpa_tables.mask_bits; bits j > pb + i are ignored.
 *   A row whose A(p) is empty (SPEC.md:445 calls it an error) yields O = 0 for those queries.
 * Requires block_size == 128 (one 128-query tile per q-block, FlashPrefill's block size)
 * and nkvb <= 4096; otherwise CPA_ERR_UNSUPPORTED. ws is unused (may be NULL). */
CPA_API int cpa_block_sparse_attention(const cpa_params* p, const void* q, const cpa_kv_cache* cache,
                                       const uint32_t* mask, void* o, void* ws, size_t ws_bytes, void* stream);

/* q-uniform expansion of tables into a 2D mask (the "same unioned block mask" of
 * PAPER.md:409): mask[b,h,i,j] = [j in T[b, h/E]] && j <= pb + i, written for every (b, h, i).
 * mask: u32 [B, Hq, nqb, nwords] device, overwritten. */
CPA_API int cpa_expand_tables(const cpa_params* p, const cpa_tables* tables, uint32_t* mask, void* stream);

CPA_API const char* cpa_status_string(int status);
CPA_API const char* cpa_last_error(void);  /* thread-local detail of the last failing call */
CPA_API int cpa_version(void);
/* Number of kernels the last successful call on this thread enqueued (for bench accounting). */
CPA_API int cpa_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CPA_H_ */
