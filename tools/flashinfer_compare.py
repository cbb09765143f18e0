"""Comparator (bench-only, never in libcpa): FlashInfer paged prefill on the same B200, same pages.

SURVEY §8(d): (1) dense chunked-prefill paged attention through FlashInfer vs our dense kernel
(cpa_paged_attention, tables=NULL) -- a check on the baseline our speedups divide by; (2) the paper's
own execution recipe: one pseudo-request per (b, execution group) with num_kv_heads=1,
its query heads as qo heads and its tabled pages as the page list, vs our zero-copy table kernel.
Our pool [pages, Hkv, bs, d] is FlashInfer's HND layout as is; for the pseudo-batch it is viewed as
[pages*Hkv, 1, bs, d] (page p, head h -> page p*Hkv + h), still zero-copy. FlashInfer's causal mask
aligns each query to the END of its page list, which is right here only because every chunk block is
in every table and sorts last (the fully open chunk).

  python tools/flashinfer_compare.py [--config llama8b_128k] [--backends trtllm-gen,fa2,auto]
One JSON line per (backend, mode): ms (CUDA events, L2 flushed), max|d|/RMS vs our output.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool


def timed(fn, flush, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b_128k")
    ap.add_argument("--backends", default="trtllm-gen,fa2,auto")
    args = ap.parse_args()
    import flashinfer
    cfg = CONFIGS[args.config]
    seed = 16839 + list(CONFIGS).index(args.config)
    P, C, L = cfg.chunk_geometry()
    bs, d, Hq, Hkv, B = cfg.block_size, cfg.head_dim, cfg.num_q_heads, cfg.num_kv_heads, cfg.batch
    E = Hq // Hkv
    nkvb = -(-L // bs)
    k, v = make_kv(cfg, seed)
    q = make_q(cfg, seed)
    pt, npg = page_layout(B, nkvb, seed)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    kp, vp = dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs))
    cache = cpa.PagedKVCache(kp, vp, torch.from_numpy(pt).cuda())
    dq = dev(q)
    del k, v
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    p = cpa.make_params(B, Hq, Hkv, d, bs, C, P, alpha=0.06)
    ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
    tabs = cpa.alloc_tables(p)
    cpa.build_tables(p, dq, cache, tabs, workspace=ws)
    o_dense = torch.empty(B, C, Hq, d, dtype=torch.bfloat16, device="cuda")
    o_sparse = torch.empty_like(o_dense)
    ours = {"dense": timed(lambda: cpa.paged_attention(p, dq, cache, None, o_dense, workspace=ws), flush),
            "sparse": timed(lambda: cpa.paged_attention(p, dq, cache, tabs, o_sparse, workspace=ws), flush)}
    print(json.dumps({"impl": "libcpa", "config": cfg.name, **{f"{m}_ms": round(t, 4) for m, t in ours.items()}}),
          flush=True)
    ip = tabs.kv_indptr.cpu().numpy()
    ix = tabs.kv_indices.cpu().numpy()
    pt_t = torch.from_numpy(pt)
    last_len = L - (nkvb - 1) * bs
    fi_ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rms = lambda o: float(o.double().pow(2).mean().sqrt())
    for backend in args.backends.split(","):
        for mode in ("dense", "sparse"):
            rec = {"impl": "flashinfer", "backend": backend, "mode": mode, "config": cfg.name}
            try:
                t0 = time.time()
                if mode == "dense":  # B requests, Hkv heads, every page of the sequence
                    qo_indptr = torch.arange(B + 1, dtype=torch.int32) * C
                    kv_indptr = torch.arange(B + 1, dtype=torch.int32) * nkvb
                    kv_indices = pt_t[:, :nkvb].reshape(-1).to(torch.int32)
                    last = torch.full((B,), last_len, dtype=torch.int32)
                    qq = dq.reshape(B * C, Hq, d)
                    nq, nk, kvc = Hq, Hkv, (kp, vp)
                    seq_lens = torch.full((B,), L, dtype=torch.int32)
                    block_tables = pt_t[:, :nkvb].to(torch.int32)
                    ref = o_dense.reshape(B * C, Hq, d)
                else:  # pseudo-batch: one request per (b, group) with num_kv_heads = 1
                    Gn = Hq // E
                    rows = B * Gn
                    qo_indptr = torch.arange(rows + 1, dtype=torch.int32) * C
                    kv_indptr = torch.from_numpy(ip.astype(np.int32))
                    lst = []
                    for r in range(rows):
                        b, g = divmod(r, Gn)
                        kvh = g  # execution group = KV group: group g reads KV head g
                        js = ix[ip[r]:ip[r + 1]]
                        lst.append(pt[b, js].astype(np.int64) * Hkv + kvh)
                    kv_indices = torch.from_numpy(np.concatenate(lst).astype(np.int32))
                    last = torch.full((rows,), last_len, dtype=torch.int32)
                    # q of row (b, g): [C, E, d] -- heads g*E .. g*E+E-1 of batch b
                    qq = dq.reshape(B, C, Gn, E, d).permute(0, 2, 1, 3, 4).reshape(rows * C, E, d).contiguous()
                    nq, nk = E, 1
                    kvc = (kp.view(npg * Hkv, 1, bs, d), vp.view(npg * Hkv, 1, bs, d))
                    seq_lens = torch.from_numpy(((ip[1:] - ip[:-1]) * bs - (bs - last_len)).astype(np.int32))
                    mx = int((ip[1:] - ip[:-1]).max())
                    block_tables = torch.zeros(rows, mx, dtype=torch.int32)
                    for r in range(rows):
                        block_tables[r, :len(lst[r])] = torch.from_numpy(lst[r].astype(np.int32))
                    ref = o_sparse.reshape(B, C, Gn, E, d).permute(0, 2, 1, 3, 4).reshape(rows * C, E, d)
                w = flashinfer.BatchPrefillWithPagedKVCacheWrapper(fi_ws, kv_layout="HND", backend=backend)
                kw = dict(causal=True, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
                if backend == "trtllm-gen":
                    kw.update(seq_lens=seq_lens.cuda(), block_tables=block_tables.cuda(),
                              max_token_per_sequence=C)
                # indptr / last-page arrays on the host (FlashInfer's planner reads them there)
                w.plan(qo_indptr, kv_indptr, kv_indices.cuda(), last, nq, nk, d, bs, **kw)
                out = torch.empty_like(qq)
                w.run(qq, kvc, out=out)
                torch.cuda.synchronize()
                rec["setup_s"] = round(time.time() - t0, 1)
                rec["ms"] = round(timed(lambda: w.run(qq, kvc, out=out), flush), 4)
                rec["max_abs_diff_over_rms_vs_libcpa"] = round(float((out.float() - ref.float()).abs().max()) / rms(ref), 5)
                rec["libcpa_ms"] = round(ours[mode], 4)
            except Exception as ex:  # noqa: BLE001 -- report and go on
                rec["error"] = f"{type(ex).__name__}: {str(ex)[:300]}"
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
