"""A/B microbenchmark of k_paged_attn variants on the 128K final chunk: libs x flag sets, interleaved
rounds (robust to clock drift), median of per-launch CUDA-event times."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool

cfg = CONFIGS[os.environ.get("CFG", "llama8b_128k")]
seed = 16839 + list(CONFIGS).index(cfg.name)
P, C, L = cfg.chunk_geometry(); bs = cfg.block_size
KVH = int(os.environ.get("KVH", cfg.num_kv_heads))  # < Hkv: one rank's KV-group shard (multi-GPU per-GPU work)
E_ = cfg.num_q_heads // cfg.num_kv_heads
k, v = make_kv(cfg, seed, kv_heads=range(KVH)); q = make_q(cfg, seed, q_heads=range(KVH * E_))
pt, npg = page_layout(cfg.batch, -(-L // bs), seed)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
VF16 = os.environ.get("V_F16", "1") == "1"  # default: the fp16 V pool of the product path (CPA_F_V_F16)
vpool = dev(to_pool(v, pt, npg, bs))
cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), vpool.half() if VF16 else vpool, torch.from_numpy(pt).cuda())
dq = dev(q); del k, v
p = cpa.make_params(cfg.batch, KVH * E_, KVH, cfg.head_dim, bs, C, P, alpha=0.06)
flag_sets = [int(x, 0) for x in os.environ.get("FLAGSETS", "0").split(",")]
rounds = int(os.environ.get("ROUNDS", "5"))
o = torch.empty(cfg.batch, C, KVH * E_, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
variants = [(pp, f) for pp in sys.argv[1:] for f in flag_sets]
libs = {}
import ctypes
tabs = None
times = {(v_, n_): [] for v_ in variants for n_ in ("sparse", "dense")}
ref = None
import random
rng = random.Random(0)
for r in range(rounds):
    order = list(variants)
    rng.shuffle(order)  # no variant always follows the same one (power / clock carry-over)
    for (path, fl) in order:
        cpa._lib = libs.get(path); cpa.LIB_PATH = path
        cpa.lib(); libs[path] = cpa._lib
        p.flags = (p.flags & 1) | fl | (cpa.F_V_F16 if VF16 else 0)
        if tabs is None:
            tabs = cpa.alloc_tables(p); cpa.build_tables(p, dq, cache, tabs)
        for name, tab in (("sparse", tabs),) + ((("dense", None),) if os.environ.get("DENSE", "1") == "1" else ()):
            cpa.paged_attention(p, dq, cache, tab, o)
            for _ in range(int(os.environ.get("REPS", "3"))):
                flush.zero_(); a = torch.cuda.Event(True); b = torch.cuda.Event(True)
                a.record(); cpa.paged_attention(p, dq, cache, tab, o); b.record(); torch.cuda.synchronize()
                times[((path, fl), name)].append(a.elapsed_time(b))
            if name == "sparse" and r == 0:
                if ref is None: ref = o.clone()
                print(json.dumps({"lib": os.path.basename(path), "flags": fl,
                                  "maxdiff_vs_first": float((o.float() - ref.float()).abs().max())}), flush=True)
for (path, fl) in variants:
    print(json.dumps({"lib": os.path.basename(path), "flags": fl,
                      "sparse_ms": round(float(np.median(times[((path, fl), "sparse")])), 4),
                      "sparse_mean_ms": round(float(np.mean(times[((path, fl), "sparse")])), 4),
                      "sparse_p25_ms": round(float(np.percentile(times[((path, fl), "sparse")], 25)), 4),
                      "sparse_min_ms": round(float(np.min(times[((path, fl), "sparse")])), 4),
                      "dense_ms": round(float(np.median(times[((path, fl), "dense")] or [0])), 4)}), flush=True)
