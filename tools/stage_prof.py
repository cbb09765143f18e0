"""Per-kernel device times of one chunk step (torch.profiler / CUPTI), 128K config by default."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool
cfg = CONFIGS[os.environ.get("CFG", "llama8b_128k")]
seed = 16839 + list(CONFIGS).index(cfg.name)
P, C, L = cfg.chunk_geometry(); bs = cfg.block_size
k, v = make_kv(cfg, seed); q = make_q(cfg, seed)
pt, npg = page_layout(cfg.batch, -(-L // bs), seed)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs)), torch.from_numpy(pt).cuda())
kc = dev(k[:, :, P:].transpose(0, 2, 1, 3)); vc = dev(v[:, :, P:].transpose(0, 2, 1, 3))
dq = dev(q); del k, v
p = cpa.make_params(cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, bs, C, P, alpha=0.06)
t = cpa.alloc_tables(p)
ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
o = torch.empty(cfg.batch, C, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
for _ in range(3): cpa.chunk_step(p, dq, cache, t, o, kc, vc, workspace=ws)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        cpa.chunk_step(p, dq, cache, t, o, kc, vc, workspace=ws)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
