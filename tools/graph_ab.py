"""Chunk step launched directly vs replayed from a captured CUDA graph, on rank 0's shard at W=1..8
(KVH = 8/W KV groups): how much of the step is launch / inter-kernel gap rather than kernel time."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_16839_b200 as cpa
from paper_2605_16839_b200.shard import head_shard
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool
cfg = CONFIGS[os.environ.get("CFG", "llama8b_128k")]
seed = 16839 + list(CONFIGS).index(cfg.name)
P, C, L = cfg.chunk_geometry(); bs, d = cfg.block_size, cfg.head_dim
nkvb = -(-L // bs)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for W in (1, 8):
    kvh, qh = head_shard(cfg.num_q_heads, cfg.num_kv_heads, W, 0)
    k, v = make_kv(cfg, seed, 0.30, kv_heads=kvh); q = dev(make_q(cfg, seed, q_heads=qh))
    pt, npg = page_layout(cfg.batch, nkvb, seed)
    cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs)), torch.from_numpy(pt).cuda())
    kc, vc = dev(k[:, :, P:].transpose(0, 2, 1, 3)), dev(v[:, :, P:].transpose(0, 2, 1, 3))
    p = cpa.make_params(cfg.batch, len(qh), len(kvh), d, bs, C, P, alpha=0.06)
    t = cpa.alloc_tables(p); ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
    o = torch.empty(cfg.batch, C, len(qh), d, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    step = lambda: cpa.chunk_step(p, q, cache, t, o, kc, vc, workspace=ws, stream=s)
    with torch.cuda.stream(s):
        for _ in range(3): step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    torch.cuda.synchronize()
    res = {}
    for name, fn in (("direct", step), ("graph", g.replay)):
        ts = []
        for _ in range(15):
            flush.zero_(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                a.record(s); fn(); b.record(s)
            torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        res[name] = round(float(np.median(ts)), 4)
    # stage sums
    st = {}
    for name, fn in (("append", lambda: cpa.append_kv(p, kc, vc, cache, stream=s)),
                     ("tables", lambda: cpa.build_tables(p, q, cache, t, workspace=ws, stream=s)),
                     ("attention", lambda: cpa.paged_attention(p, q, cache, t, o, workspace=ws, stream=s))):
        ts = []
        for _ in range(15):
            flush.zero_(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); fn(); b.record(s); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        st[name] = round(float(np.median(ts)), 4)
    print(json.dumps({"W": W, **res, "stages": st, "stage_sum": round(sum(st.values()), 4)}), flush=True)
    del k, v, cache
    torch.cuda.empty_cache()
