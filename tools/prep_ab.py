"""A/B of the chunk step's first half (cpa_prepare_chunk: append + pooled estimator + tables) across
libcpa builds: CUDA-graph replays, L2 flushed before each, interleaved rounds, median per variant.

  CFG=llama8b_128k KVH=8 ROUNDS=8 REPS=20 [FLAGSETS=0,32768] python tools/prep_ab.py a.so b.so
(variants = libs x extra flag sets)
"""
import os, sys, json, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool

cfg = CONFIGS[os.environ.get("CFG", "llama8b_128k")]
seed = 16839 + list(CONFIGS).index(cfg.name)
P, C, L = cfg.chunk_geometry(); bs = cfg.block_size
KVH = int(os.environ.get("KVH", cfg.num_kv_heads)); E_ = cfg.num_q_heads // cfg.num_kv_heads
k, v = make_kv(cfg, seed, kv_heads=range(KVH)); q = make_q(cfg, seed, q_heads=range(KVH * E_))
pt, npg = page_layout(cfg.batch, -(-L // bs), seed)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs)).half(), torch.from_numpy(pt).cuda())
kc = dev(k[:, :, P:].transpose(0, 2, 1, 3)); vc = dev(v[:, :, P:].transpose(0, 2, 1, 3)); dq = dev(q); del k, v
p = cpa.make_params(cfg.batch, KVH * E_, KVH, cfg.head_dim, bs, C, P, alpha=0.06, flags=cpa.F_V_F16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
libs, graphs, times, ref = {}, {}, {}, None
base_flags = p.flags
variants = [(lp, int(f, 0)) for lp in sys.argv[1:] for f in os.environ.get("FLAGSETS", "0").split(",")]
for path in variants:
    lp, fl = path
    p.flags = base_flags | fl
    if lp not in libs:
        cpa._lib = None; cpa.LIB_PATH = lp; libs[lp] = cpa.lib()
    cpa._lib = libs[lp]
    t = cpa.alloc_tables(p); ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
    for _ in range(2): cpa.prepare_chunk(p, dq, cache, t, kc, vc, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): cpa.prepare_chunk(p, dq, cache, t, kc, vc, workspace=ws)
    g.replay(); torch.cuda.synchronize()
    ip = t.kv_indptr.cpu().numpy(); ix = t.kv_indices.cpu().numpy()[: ip[-1]]
    if ref is None: ref = (ip, ix)
    assert np.array_equal(ip, ref[0]) and np.array_equal(ix, ref[1]), path
    graphs[path] = (g, t, ws); times[path] = []
rng = random.Random(0)
for r in range(int(os.environ.get("ROUNDS", "8"))):
    order = list(graphs); rng.shuffle(order)
    for path in order:
        g = graphs[path][0]
        for _ in range(int(os.environ.get("REPS", "20"))):
            flush.zero_(); a = torch.cuda.Event(True); b = torch.cuda.Event(True)
            a.record(); g.replay(); b.record(); torch.cuda.synchronize(); times[path].append(a.elapsed_time(b) * 1e3)
for path in graphs:
    ts = times[path]
    print(json.dumps({"lib": os.path.basename(path[0]), "flags": path[1], "cfg": cfg.name, "kv_heads": KVH, "prepare_us_median": round(float(np.median(ts)), 2),
                      "p25": round(float(np.percentile(ts, 25)), 2), "min": round(float(np.min(ts)), 2)}), flush=True)
