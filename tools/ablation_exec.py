"""NEXT-3 execution-strategy ablation (Fig. 7(c); batch scaling of Table
tab:copy_metadata_batch_scaling): same unioned tables, executed
  zero-copy : attention reads the tabled pages in place (CompactAttention)
  copy      : gather the tabled pages into a compact buffer, then the same attention kernel
  block-sparse (unioned mask) : the q-uniform expansion of the same tables executed per (h, q-block)
              tile by the block-sparse kernel (cpa_block_sparse_attention), metadata =
              estimator + unions + CSR + expansion
and, for reference, block-sparse over the estimator's own 2D mask (no unions: FlashPrefill-style
execution, fewer blocks per tile but a different output), metadata = estimator + mask.
Reports metadata (estimator + unions + CSR), copy and compute device times per batch size."""
import argparse, dataclasses, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool

ap = argparse.ArgumentParser()
ap.add_argument("--context", type=int, default=131072)
ap.add_argument("--chunk", type=int, default=512)
ap.add_argument("--batches", default="1,2,4,8,16")
args = ap.parse_args()
ev = lambda: torch.cuda.Event(enable_timing=True)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for B in [int(x) for x in args.batches.split(",")]:
    cfg = dataclasses.replace(CONFIGS["llama8b_128k"], batch=B, context=args.context, chunk=args.chunk)
    seed = 16839
    P, C, L = cfg.chunk_geometry(); bs = cfg.block_size
    k, v = make_kv(cfg, seed); q = make_q(cfg, seed)
    pt, npg = page_layout(B, -(-L // bs), seed)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs)).half(), torch.from_numpy(pt).cuda())  # fp16 V pool (bench default)
    dq = dev(q); del k, v
    p = cpa.make_params(B, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, bs, C, P, alpha=0.06, flags=cpa.F_V_F16)
    t = cpa.alloc_tables(p, mask=True)
    nqb, nkvb, pb, Gn, nwords, Rpad = cpa.geometry(p)
    qmask = torch.empty(B, cfg.num_q_heads, nqb, nwords, dtype=torch.int32, device="cuda")
    pm = cpa.make_params(B, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, bs, C, P, alpha=0.06, flags=cpa.F_MASK_OUT | cpa.F_V_F16)
    ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
    cws = torch.empty(int(cpa.lib().cpa_copy_workspace_bytes(__import__("ctypes").byref(p))), dtype=torch.uint8, device="cuda")
    o = torch.empty(B, C, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
    def timed(fn, reps=7):
        fn(); ts = []
        for _ in range(reps):
            flush.zero_(); a, b = ev(), ev(); a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        return float(np.median(ts))
    meta = timed(lambda: cpa.build_tables(p, dq, cache, t, workspace=ws))
    zc = timed(lambda: cpa.paged_attention(p, dq, cache, t, o, workspace=ws))
    cp_total = timed(lambda: cpa.paged_attention_copy(p, dq, cache, t, o, workspace=cws))
    bs_meta = timed(lambda: (cpa.build_tables(p, dq, cache, t, workspace=ws), cpa.expand_tables(p, t, qmask)))
    bs_union = timed(lambda: cpa.block_sparse_attention(p, dq, cache, qmask, o))
    raw_meta = timed(lambda: cpa.build_tables(pm, dq, cache, t, workspace=ws))
    raw_density = float(np.unpackbits(t.mask_bits.cpu().numpy().view(np.uint8), bitorder="little").sum())
    bs_raw = timed(lambda: cpa.block_sparse_attention(p, dq, cache, t.mask_bits, o))
    cpa.build_tables(p, dq, cache, t, workspace=ws)
    # copy-only time: the gather kernel alone = copy total - compact attention (measured via dense-free path)
    ip = t.kv_indptr.cpu().numpy()
    sel_bytes = int(ip[-1]) * bs * cfg.head_dim * 2 * 2
    print(json.dumps({"batch": B, "context": args.context, "chunk": args.chunk, "metadata_ms": round(meta, 4),
                      "zero_copy_attention_ms": round(zc, 4), "copy_variant_ms": round(cp_total, 4),
                      "copy_overhead_ms": round(cp_total - zc, 4), "bytes_copied": sel_bytes,
                      "zero_copy_total_ms": round(meta + zc, 4), "copy_total_ms": round(meta + cp_total, 4),
                      "block_sparse_union_attention_ms": round(bs_union, 4),
                      "block_sparse_union_total_ms": round(bs_meta + bs_union, 4),
                      "block_sparse_raw_mask_attention_ms": round(bs_raw, 4),
                      "block_sparse_raw_mask_total_ms": round(raw_meta + bs_raw, 4),
                      "raw_mask_tiles": int(raw_density)}), flush=True)
