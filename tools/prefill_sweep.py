"""NEXT-4 sweeps: whole chunked prefills through the C ABI.

For each (context, chunk) the prompt is prefilled chunk by chunk exactly as a serving engine would:
every chunk appends its K/V into the paged cache and runs the CompactAttention chunk step
(cpa_chunk_step: estimator -> tables -> paged attention over the tabled blocks); the dense baseline
runs append + dense paged attention (cpa_paged_attention with tables=NULL) on the same inputs. The
per-chunk device times (CUDA events) are summed over the whole prefill, mirroring the paper's
"attention latency" totals (tab:latency_h200 / tab:chunk_size_sensitivity), and the
alpha sweep (Fig. 7(b)) reports speedup vs the tabled density. One JSON line per point.

  python tools/prefill_sweep.py [--contexts 8192,32768,131072] [--chunks 1024,4096] [--alphas 0.06]
"""
import argparse
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool


def run(context, chunk, alpha, base="llama8b_128k", seed=16839, rho=0.30, variant="base"):
    cfg = dataclasses.replace(CONFIGS[base], context=context, chunk=chunk, name=f"{base}@{context}/{chunk}")
    bs, d = cfg.block_size, cfg.head_dim
    nkvb = -(-context // bs)
    k, v = make_kv(cfg, seed, rho, variant=variant)
    pt, npg = page_layout(cfg.batch, nkvb, seed)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    kp = torch.zeros(npg, cfg.num_kv_heads, bs, d, dtype=torch.bfloat16, device="cuda")
    vp = torch.zeros_like(kp, dtype=torch.float16)  # fp16 V pool (CPA_F_V_F16, bench default)
    cache = cpa.PagedKVCache(kp, vp, torch.from_numpy(pt).cuda())
    ev = lambda: torch.cuda.Event(enable_timing=True)
    tot_sparse = tot_dense = 0.0
    dens = []
    for t in range(cfg.num_chunks):
        P, C, L = cfg.chunk_geometry(t)
        q = dev(make_q(cfg, seed, chunk_index=t, variant=variant))
        kc = dev(k[:, :, P:L].transpose(0, 2, 1, 3))
        vc = dev(v[:, :, P:L].transpose(0, 2, 1, 3))
        p = cpa.make_params(cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, d, bs, C, P, alpha=alpha, flags=cpa.F_V_F16)
        tabs = cpa.alloc_tables(p)
        ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
        o = torch.empty(cfg.batch, C, cfg.num_q_heads, d, dtype=torch.bfloat16, device="cuda")
        cpa.append_kv(p, kc, vc, cache)  # warm-up (idempotent re-append below)
        cpa.chunk_step(p, q, cache, tabs, o, kc, vc, workspace=ws)
        a, b, c2 = ev(), ev(), ev()
        a.record()
        cpa.chunk_step(p, q, cache, tabs, o, kc, vc, workspace=ws)
        b.record()
        cpa.append_kv(p, kc, vc, cache)
        cpa.paged_attention(p, q, cache, None, o, workspace=ws)
        c2.record()
        torch.cuda.synchronize()
        tot_sparse += a.elapsed_time(b)
        tot_dense += b.elapsed_time(c2)
        ip = tabs.kv_indptr.cpu().numpy()
        pb = P // bs
        G = cfg.batch * (cfg.num_q_heads // cfg.group_size)
        if pb > 0:
            dens.append((ip[-1] - G * (-(-L // bs) - pb)) / (G * pb))
    return {"context": context, "chunk": chunk, "alpha": alpha, "rho": rho, "variant": variant, "chunks": cfg.num_chunks,
            "prefill_attention_ms_sparse": round(tot_sparse, 3), "prefill_attention_ms_dense": round(tot_dense, 3),
            "speedup": round(tot_dense / tot_sparse, 3),
            "final_chunk_prefix_density": round(float(dens[-1]), 4) if dens else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--contexts", default="8192,16384,32768,65536,131072")
    ap.add_argument("--chunks", default="4096")
    ap.add_argument("--alphas", default="0.06")
    ap.add_argument("--rho", type=float, default=0.30)
    ap.add_argument("--variant", default="base")
    args = ap.parse_args()
    for a in [float(x) for x in args.alphas.split(",")]:
        for c in [int(x) for x in args.chunks.split(",")]:
            for L in [int(x) for x in args.contexts.split(",")]:
                if L % c == 0:
                    print(json.dumps(run(L, c, a, rho=args.rho, variant=args.variant)), flush=True)


if __name__ == "__main__":
    main()
