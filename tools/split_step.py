"""One chunk step as two concurrent half-steps on one GPU: after the append, KV groups [0, Hkv/2) and
[Hkv/2, Hkv) each run estimator -> tables -> attention on their own stream (head slices of q / o and of
the page pool through the ABI's strides, their own tables and workspace), so one half's HBM-bound
estimator overlaps the other half's tensor-bound attention and both attention grids share the SMs.
Compared with the single-stream cpa_chunk_step (both replayed from CUDA graphs, L2 flushed).

  python tools/split_step.py [--config llama8b_128k] [--parts 2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b_128k")
    ap.add_argument("--parts", type=int, default=2)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    seed = 16839 + list(CONFIGS).index(args.config)
    P, C, L = cfg.chunk_geometry()
    bs, d, B, Hq, Hkv = cfg.block_size, cfg.head_dim, cfg.batch, cfg.num_q_heads, cfg.num_kv_heads
    E = Hq // Hkv
    nkvb = -(-L // bs)
    k, v = make_kv(cfg, seed)
    q = make_q(cfg, seed)
    pt, npg = page_layout(B, nkvb, seed)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    kp = dev(to_pool(k, pt, npg, bs))
    vp = dev(to_pool(v, pt, npg, bs)).half()
    ptab = torch.from_numpy(pt).cuda()
    dq = dev(q)
    kc, vc = dev(k[:, :, P:].transpose(0, 2, 1, 3)), dev(v[:, :, P:].transpose(0, 2, 1, 3))
    del k, v
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    o = torch.empty(B, C, Hq, d, dtype=torch.bfloat16, device="cuda")
    o2 = torch.empty_like(o)
    # full step
    p = cpa.make_params(B, Hq, Hkv, d, bs, C, P, alpha=0.06, flags=cpa.F_V_F16)
    cache = cpa.PagedKVCache(kp, vp, ptab)
    t = cpa.alloc_tables(p)
    ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
    # parts: KV heads [s*h, (s+1)*h) through the pool's strides, q / o head slices
    h = Hkv // args.parts
    parts = []
    for s in range(args.parts):
        ps = cpa.make_params(B, h * E, h, d, bs, C, P, alpha=0.06, flags=cpa.F_V_F16, q_token_stride=Hq * d)
        cs = cpa.PagedKVCache(kp[:, s * h:(s + 1) * h], vp[:, s * h:(s + 1) * h], ptab,
                              page_stride=Hkv * bs * d, head_stride=bs * d, num_pages=kp.shape[0])
        parts.append(dict(p=ps, cache=cs, t=cpa.alloc_tables(ps),
                          ws=torch.empty(cpa.workspace_bytes(ps), dtype=torch.uint8, device="cuda"),
                          q=dq[:, :, s * h * E:(s + 1) * h * E], o=o2[:, :, s * h * E:(s + 1) * h * E],
                          st=torch.cuda.Stream()))
    ev_app = torch.cuda.Event()
    ev_done = [torch.cuda.Event() for _ in parts]

    def full():
        cpa.chunk_step(p, dq, cache, t, o, kc, vc, workspace=ws)

    def split():
        main_st = torch.cuda.current_stream()  # the capture stream inside torch.cuda.graph
        cpa.append_kv(p, kc, vc, cache)
        ev_app.record(main_st)
        for x, e in zip(parts, ev_done):
            x["st"].wait_event(ev_app)
            cpa.build_tables(x["p"], x["q"], x["cache"], x["t"], workspace=x["ws"], stream=x["st"])
            cpa.paged_attention(x["p"], x["q"], x["cache"], x["t"], x["o"], workspace=x["ws"], stream=x["st"])
            e.record(x["st"])
        for e in ev_done:
            main_st.wait_event(e)

    res = {}
    for name, fn in (("full", full), ("split", split)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
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
    same = bool(torch.equal(o, o2))
    print(json.dumps({"config": cfg.name, "parts": args.parts, "full_ms": round(res["full"], 4),
                      "split_ms": round(res["split"], 4), "gain": round(res["full"] / res["split"], 3),
                      "outputs_identical": same}), flush=True)


if __name__ == "__main__":
    main()
