"""NEXT-4 alpha sweep on a graded-needle workload (the accuracy/speed trade-off shape of Fig. 7(b),
PAPER.md:389, 402-405, with a synthetic accuracy proxy since RULER is out of scope).

Final chunk of a long context (default 128K, LLaMA-8B shape), needles with graded strengths
(synth.workload.make_kv(graded=True)). For each alpha:
  * CompactAttention chunk step (estimator -> unions -> tables -> zero-copy attention): device ms,
    tabled prefix density, relative output error ||O - O_dense|| / ||O_dense||;
  * block-sparse execution of the estimator's own 2D mask (FlashPrefill-style, no unions): device ms,
    executed prefix tile density, relative error;
against dense paged attention over the same cache. One JSON line per alpha.

  python tools/alpha_sweep.py [--context 131072] [--chunk 4096] [--alphas 0.005,0.01,...]
"""
import argparse, dataclasses, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool

ap = argparse.ArgumentParser()
ap.add_argument("--context", type=int, default=131072)
ap.add_argument("--chunk", type=int, default=4096)
ap.add_argument("--alphas", default="0.002,0.005,0.01,0.02,0.06,0.1,0.2,0.4,0.7")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

cfg = dataclasses.replace(CONFIGS["llama8b_128k"], context=args.context, chunk=args.chunk, name="graded")
seed = 16839
P, C, L = cfg.chunk_geometry()
bs, d, B, Hq = cfg.block_size, cfg.head_dim, cfg.batch, cfg.num_q_heads
k, v = make_kv(cfg, seed, graded=True)
q = make_q(cfg, seed)
pt, npg = page_layout(B, -(-L // bs), seed)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs)), torch.from_numpy(pt).cuda())
dq = dev(q)
del k, v
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)


def timed(fn):
    fn()
    ts = []
    for _ in range(args.reps):
        flush.zero_()
        a, b = ev(), ev()
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def rel(o, ref):
    return float((o.float() - ref).norm() / ref.norm())


p0 = cpa.make_params(B, Hq, cfg.num_kv_heads, d, bs, C, P, alpha=0.06)
ws = torch.empty(cpa.workspace_bytes(p0), dtype=torch.uint8, device="cuda")
o_dense = torch.empty(B, C, Hq, d, dtype=torch.bfloat16, device="cuda")
dense_ms = timed(lambda: cpa.paged_attention(p0, dq, cache, None, o_dense, workspace=ws))
ref = o_dense.float()
nqb, nkvb, pb, Gn, nwords, _ = cpa.geometry(p0)
for a in [float(x) for x in args.alphas.split(",")]:
    p = cpa.make_params(B, Hq, cfg.num_kv_heads, d, bs, C, P, alpha=a)
    pm = cpa.make_params(B, Hq, cfg.num_kv_heads, d, bs, C, P, alpha=a, flags=cpa.F_MASK_OUT)
    t = cpa.alloc_tables(p, mask=True)
    o = torch.empty_like(o_dense)
    ca_ms = timed(lambda: cpa.chunk_step(p, dq, cache, t, o, workspace=ws))
    ca_err = rel(o, ref)
    ip = t.kv_indptr.cpu().numpy()
    tab_density = (int(ip[-1]) - B * Gn * (nkvb - pb)) / (B * Gn * pb)
    meta_ms = timed(lambda: cpa.build_tables(pm, dq, cache, t, workspace=ws))
    bsp_ms = timed(lambda: cpa.block_sparse_attention(p, dq, cache, t.mask_bits, o))
    bsp_err = rel(o, ref)
    bits = np.unpackbits(t.mask_bits.cpu().numpy().view(np.uint8), bitorder="little").reshape(B, Hq, nqb, nwords * 32)
    raw_density = float(bits[..., :pb].mean())
    print(json.dumps({"alpha": a, "context": L, "chunk": C, "dense_ms": round(dense_ms, 4),
                      "ca_step_ms": round(ca_ms, 4), "ca_speedup": round(dense_ms / ca_ms, 3),
                      "ca_prefix_density": round(tab_density, 4), "ca_rel_err": round(ca_err, 5),
                      "block_sparse_step_ms": round(meta_ms + bsp_ms, 4),
                      "block_sparse_speedup": round(dense_ms / (meta_ms + bsp_ms), 3),
                      "block_sparse_prefix_density": round(raw_density, 4),
                      "block_sparse_rel_err": round(bsp_err, 5)}), flush=True)
