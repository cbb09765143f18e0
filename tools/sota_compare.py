"""Comparator (bench-only, never in libcpa): the strongest dense attention kernels in this image on
the same B200 and the same 128K chunk, to calibrate what our dense / table kernel reaches.

  * FlashAttention-4 (CuTe-DSL, tcgen05; vendored in vllm as vllm.vllm_flash_attn.cute), paged with
    page_size 128 (its NHD layout [pages, 128, Hkv, d]: a permuted copy of our HND pool) and on a
    contiguous [B, L, Hkv, d] cache;
  * FlashInfer trtllm-gen context FMHA (the prebuilt Blackwell cubins of flashinfer_cubin) on our
    HND pool as is (page 128) and, if that kernel is missing, on re-paged copies (64 / 32).
Causal mask bottom-right aligned (query p sits at P + p), i.e. the dense chunked-prefill attention our
dense baseline computes. One JSON line per (impl, variant): ms (CUDA events, L2 flushed before every
rep), TFLOP/s on the exact causal FLOPs 4 d sum_p (P+p+1) per head, max|d|/RMS vs our dense output.

  python tools/sota_compare.py [--config llama8b_128k] [--reps 10]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool


def timed(fn, flush, reps):
    for _ in range(3):
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
    return float(np.median(ts)), float(np.min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b_128k")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--skip", default="")
    args = ap.parse_args()
    skip = set(args.skip.split(",")) if args.skip else set()
    cfg = CONFIGS[args.config]
    seed = 16839 + list(CONFIGS).index(args.config)
    P, C, L = cfg.chunk_geometry()
    bs, d, Hq, Hkv, B = cfg.block_size, cfg.head_dim, cfg.num_q_heads, cfg.num_kv_heads, cfg.batch
    nkvb = -(-L // bs)
    k, v = make_kv(cfg, seed)
    q = make_q(cfg, seed)
    pt, npg = page_layout(B, nkvb, seed)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    kp, vp = dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs))  # [pages, Hkv, bs, d]
    del k, v
    pt_d = torch.from_numpy(pt).cuda()
    cache = cpa.PagedKVCache(kp, vp, pt_d)
    dq = dev(q)  # [B, C, Hq, d]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    scale = 1.0 / math.sqrt(d)
    flops = 4.0 * d * Hq * B * sum(P + p + 1 for p in range(C))
    rms = lambda o: float(o.double().pow(2).mean().sqrt())

    p = cpa.make_params(B, Hq, Hkv, d, bs, C, P, alpha=0.06)
    ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
    o_dense = torch.empty(B, C, Hq, d, dtype=torch.bfloat16, device="cuda")
    med, mn = timed(lambda: cpa.paged_attention(p, dq, cache, None, o_dense, workspace=ws), flush, args.reps)
    ref = o_dense.float()
    ref_rms = rms(ref)
    print(json.dumps({"impl": "libcpa dense paged (bf16 V pool)", "config": cfg.name, "ms": round(med, 4),
                      "min_ms": round(mn, 4), "tflops": round(flops / med / 1e9, 1)}), flush=True)

    def report(name, fn, out_of):
        rec = {"impl": name, "config": cfg.name}
        try:
            t0 = time.time()
            o = fn()
            torch.cuda.synchronize()
            rec["setup_s"] = round(time.time() - t0, 1)
            med, mn = timed(fn, flush, args.reps)
            rec.update(ms=round(med, 4), min_ms=round(mn, 4), tflops=round(flops / med / 1e9, 1),
                       max_abs_diff_over_rms_vs_libcpa=round(float((out_of(o).float() - ref).abs().max()) / ref_rms, 5))
        except Exception as ex:  # noqa: BLE001 -- report and go on
            rec["error"] = f"{type(ex).__name__}: {str(ex)[:400]}"
        print(json.dumps(rec), flush=True)

    # ---- FlashAttention-4 (CuTe DSL) ----
    if "fa4" not in skip:
        try:
            from vllm.vllm_flash_attn.cute.interface import _flash_attn_fwd
            k_nhd = kp.permute(0, 2, 1, 3).contiguous()  # [pages, bs, Hkv, d]
            v_nhd = vp.permute(0, 2, 1, 3).contiguous()
            pt32 = pt_d[:, :nkvb].to(torch.int32).contiguous()
            out = torch.empty_like(dq)
            report("FA4 cute paged (page 128, NHD copy)",
                   lambda: _flash_attn_fwd(dq, k_nhd, v_nhd, page_table=pt32, softmax_scale=scale, causal=True,
                                           out=out)[0], lambda o: o)
            # contiguous cache [B, L, Hkv, d] gathered through the page table
            kc = k_nhd[pt_d[:, :nkvb].long()].reshape(B, nkvb * bs, Hkv, d)[:, :L].contiguous()
            vc = v_nhd[pt_d[:, :nkvb].long()].reshape(B, nkvb * bs, Hkv, d)[:, :L].contiguous()
            report("FA4 cute contiguous KV",
                   lambda: _flash_attn_fwd(dq, kc, vc, softmax_scale=scale, causal=True, out=out)[0], lambda o: o)
            del kc, vc, k_nhd, v_nhd
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"impl": "FA4 cute", "error": f"{type(ex).__name__}: {str(ex)[:400]}"}), flush=True)

    # ---- FlashInfer trtllm-gen context FMHA ----
    if "trtllm" not in skip:
        try:
            import flashinfer
            fi_ws = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")
            qq = dq.reshape(B * C, Hq, d)
            cum_q = torch.arange(B + 1, dtype=torch.int32, device="cuda") * C
            cum_kv = torch.arange(B + 1, dtype=torch.int32, device="cuda") * L
            seq_lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
            for page in (128, 64, 32):
                if page == bs:
                    kc_, vc_, bt = kp, vp, pt_d[:, :nkvb].to(torch.int32).contiguous()
                else:  # re-page: page j of size bs -> bs/page sub-pages (same tokens)
                    r = bs // page
                    kc_ = kp.reshape(npg, Hkv, r, page, d).permute(0, 2, 1, 3, 4).reshape(npg * r, Hkv, page, d).contiguous()
                    vc_ = vp.reshape(npg, Hkv, r, page, d).permute(0, 2, 1, 3, 4).reshape(npg * r, Hkv, page, d).contiguous()
                    bt = (pt_d[:, :nkvb].long()[:, :, None] * r + torch.arange(r, device="cuda")).reshape(B, -1)
                    bt = bt.to(torch.int32).contiguous()
                out = torch.empty_like(qq)
                report(f"FlashInfer trtllm-gen context (page {page}, HND)",
                       lambda: flashinfer.prefill.trtllm_batch_context_with_kv_cache(
                           qq, (kc_, vc_), fi_ws, bt, seq_lens, C, L, scale, 1.0, B, cum_q, cum_kv, out=out,
                           kv_layout="HND", causal=True),
                       lambda o: o.reshape(B, C, Hq, d))
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"impl": "trtllm-gen", "error": f"{type(ex).__name__}: {str(ex)[:400]}"}), flush=True)


if __name__ == "__main__":
    main()
