"""Whole chunked prefills, timed end to end on the device (first append to last attention), three ways:

  serial  -- cpa_chunk_step per chunk on one stream (append -> estimator -> tables -> attention);
  overlap -- a serving-engine schedule of the same calls on two streams: chunk t+1's append,
             estimator and tables (stream A) run while chunk t's attention (stream B) runs. Legal
             because chunk t+1 appends to pages chunk t's attention never reads, and its estimator
             only reads K of chunks <= t+1 (all appended on stream A before it); tables are double
             buffered and stream A waits for attention(t) before rebuilding tables[t % 2];
  dense   -- append + dense paged attention (tables = NULL) per chunk on one stream.
Each run starts from an empty (zeroed) cache; inputs of every chunk are device-resident beforehand.

  python tools/prefill_pipeline.py [--contexts 32768,65536,131072] [--chunk 4096]
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
from synth.workload import CONFIGS, make_kv, make_q, page_layout


def run(context, chunk, alpha=0.06, seed=16839, reps=3):
    cfg = dataclasses.replace(CONFIGS["llama8b_128k"], context=context, chunk=chunk,
                              name=f"llama8b@{context}/{chunk}")
    bs, d, B, Hq, Hkv = cfg.block_size, cfg.head_dim, cfg.batch, cfg.num_q_heads, cfg.num_kv_heads
    nkvb = -(-context // bs)
    k, v = make_kv(cfg, seed)
    pt, npg = page_layout(B, nkvb, seed)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    kp = torch.zeros(npg, Hkv, bs, d, dtype=torch.bfloat16, device="cuda")
    vp = torch.zeros(npg, Hkv, bs, d, dtype=torch.float16, device="cuda")  # fp16 V pool (CPA_F_V_F16)
    cache = cpa.PagedKVCache(kp, vp, torch.from_numpy(pt).cuda())
    chunks = []
    for t in range(cfg.num_chunks):
        P, C, L = cfg.chunk_geometry(t)
        p = cpa.make_params(B, Hq, Hkv, d, bs, C, P, alpha=alpha, flags=cpa.F_V_F16)
        chunks.append(dict(p=p, q=dev(make_q(cfg, seed, chunk_index=t)),
                           kc=dev(k[:, :, P:L].transpose(0, 2, 1, 3)), vc=dev(v[:, :, P:L].transpose(0, 2, 1, 3)),
                           o=torch.empty(B, C, Hq, d, dtype=torch.bfloat16, device="cuda")))
    del k, v
    last = chunks[-1]["p"]
    ws_a = torch.empty(cpa.workspace_bytes(last), dtype=torch.uint8, device="cuda")
    ws_b = torch.empty(cpa.workspace_bytes(last), dtype=torch.uint8, device="cuda")
    tabs = [cpa.alloc_tables(last), cpa.alloc_tables(last)]  # sized for the largest chunk
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()

    def serial():
        for c in chunks:
            cpa.chunk_step(c["p"], c["q"], cache, tabs[0], c["o"], c["kc"], c["vc"], workspace=ws_a, stream=sA)

    def dense():
        for c in chunks:
            cpa.append_kv(c["p"], c["kc"], c["vc"], cache, stream=sA)
            cpa.paged_attention(c["p"], c["q"], cache, None, c["o"], workspace=ws_a, stream=sA)

    def overlap():
        ready = [torch.cuda.Event() for _ in chunks]
        done = [torch.cuda.Event() for _ in chunks]
        for t, c in enumerate(chunks):
            if t >= 2:
                sA.wait_event(done[t - 2])  # attention(t-2) has finished reading tables[t % 2]
            cpa.append_kv(c["p"], c["kc"], c["vc"], cache, stream=sA)
            cpa.build_tables(c["p"], c["q"], cache, tabs[t % 2], workspace=ws_a, stream=sA)
            ready[t].record(sA)
            sB.wait_event(ready[t])
            cpa.paged_attention(c["p"], c["q"], cache, tabs[t % 2], c["o"], workspace=ws_b, stream=sB)
            done[t].record(sB)
        sA.wait_event(done[-1])

    res = {}
    outs = {}
    for name, fn in (("serial", serial), ("overlap", overlap), ("dense", dense)):
        ts = []
        for r in range(reps):
            kp.zero_()
            vp.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(sA)
            fn()
            b.record(sA)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[name] = float(np.median(ts))
        outs[name] = chunks[-1]["o"].clone()
    same = bool(torch.equal(outs["serial"], outs["overlap"]))
    return {"context": context, "chunk": chunk, "chunks": cfg.num_chunks,
            "prefill_ms_serial": round(res["serial"], 3), "prefill_ms_overlap": round(res["overlap"], 3),
            "prefill_ms_dense": round(res["dense"], 3),
            "speedup_serial": round(res["dense"] / res["serial"], 3),
            "speedup_overlap": round(res["dense"] / res["overlap"], 3),
            "final_chunk_output_identical_serial_vs_overlap": same}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--contexts", default="32768,65536,131072")
    ap.add_argument("--chunk", type=int, default=4096)
    args = ap.parse_args()
    for L in [int(x) for x in args.contexts.split(",")]:
        print(json.dumps(run(L, args.chunk)), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
