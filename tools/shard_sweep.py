"""Per-GPU work of the KV-group-sharded chunk step, measured on ONE GPU (§8(e) evidence when no
multi-GPU box is available): rank 0's shard at W = 1, 2, 4, 8 (8/W KV groups, their query heads and
pages) runs the whole chunk step (append + estimator + tables + paged attention) exactly as that rank
would, timed with CUDA events after an L2 flush. The head-output all-gather is fused into the
attention epilogue (cpa_chunk_step_peer); its NVLink stores are not exercised here, so T_W is the
compute part of a rank's step and T_1 / (W T_W) an upper bound on the strong-scaling efficiency.

  python tools/shard_sweep.py [--config llama8b_128k] [--reps 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_16839_b200 as cpa
from paper_2605_16839_b200.shard import head_shard
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b_128k")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    seed = 16839 + list(CONFIGS).index(args.config)
    P, C, L = cfg.chunk_geometry()
    bs, d = cfg.block_size, cfg.head_dim
    nkvb = -(-L // bs)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    t1 = None
    for W in (1, 2, 4, 8):
        kvh, qh = head_shard(cfg.num_q_heads, cfg.num_kv_heads, W, 0)
        k, v = make_kv(cfg, seed, 0.30, kv_heads=kvh)
        q = dev(make_q(cfg, seed, q_heads=qh))
        pt, npg = page_layout(cfg.batch, nkvb, seed)
        # fp16 V pool, as bench.py (CPA_F_V_F16)
        cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs)).half(),
                                 torch.from_numpy(pt).cuda())
        kc, vc = dev(k[:, :, P:].transpose(0, 2, 1, 3)), dev(v[:, :, P:].transpose(0, 2, 1, 3))
        res = {}
        for name, extra in (("auto", 0), ("per_unit_grid", cpa.F_NO_PERSIST)):
            p = cpa.make_params(cfg.batch, len(qh), len(kvh), d, bs, C, P, alpha=0.06, flags=extra | cpa.F_V_F16)
            t = cpa.alloc_tables(p)
            ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
            o = torch.empty(cfg.batch, C, len(qh), d, dtype=torch.bfloat16, device="cuda")
            for _ in range(3):
                cpa.chunk_step(p, q, cache, t, o, kc, vc, workspace=ws)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()  # the step as bench.py times it: one graph replay
            with torch.cuda.graph(g):
                cpa.chunk_step(p, q, cache, t, o, kc, vc, workspace=ws)
            g.replay()
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                g.replay()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res[name] = float(np.median(ts))
            del g
        if t1 is None:
            t1 = res["auto"]
        print(json.dumps({"config": cfg.name, "W": W, "kv_groups_per_gpu": len(kvh), "step_ms": round(res["auto"], 4),
                          "step_ms_per_unit_grid": round(res["per_unit_grid"], 4),
                          "compute_scaling_bound": round(t1 / (W * res["auto"]), 3)}), flush=True)
        del k, v, q, cache, kc, vc
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
