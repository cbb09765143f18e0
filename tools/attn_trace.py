"""Per-sub-block event trace of CTA 0 of k_paged_attn (build with -DCPA_TRACE)."""
import os, sys, ctypes, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
os.environ["CPA_LIB_PATH"] = sys.argv[1]
import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool
cfg = CONFIGS[os.environ.get("CFG", "llama8b_32k")]
seed = 16839 + list(CONFIGS).index(cfg.name)
P, C, L = cfg.chunk_geometry(); bs = cfg.block_size
k, v = make_kv(cfg, seed); q = make_q(cfg, seed)
pt, npg = page_layout(cfg.batch, -(-L // bs), seed)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs)), torch.from_numpy(pt).cuda())
dq = dev(q)
p = cpa.make_params(cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, bs, C, P, alpha=0.06)
o = torch.empty(cfg.batch, C, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
t = cpa.alloc_tables(p); cpa.build_tables(p, dq, cache, t)
for _ in range(3): cpa.paged_attention(p, dq, cache, t, o)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (16 * 2048))()
cpa.lib().cpa_debug_trace(buf)
tr = np.frombuffer(buf, dtype=np.int64).reshape(16, 2048)
U = int((tr[2, 0::2] > 0).sum())
print("sub-blocks", U)
d = lambda a, b: int(a - b)
per = [d(tr[2, 2*(u+1)], tr[2, 2*u]) for u in range(1, U - 1)]
print("median period per sub-block (cycles)", int(np.median(per)), "=> per 128-key page", 2 * int(np.median(per)))
for u in list(range(0, 4)) + list(range(U // 2, U // 2 + 4)):
    row = {"u": u, "period": d(tr[2, 2*(u+1)], tr[2, 2*u]) if u + 1 < U else 0,
           "mma_wait_p1": d(tr[2, 2*u+1], tr[3, 2*u]), "mma_pv0_s0": d(tr[3, 2*u], tr[2, 2*u]),
           "sm0_wait": d(tr[5, 2*u], tr[4, 2*u]), "sm0_ld_max": d(tr[11, 2*u], tr[5, 2*u]), "sm0_exp": d(tr[12, 2*u], tr[11, 2*u]),
           "sm0_tail": d(tr[6, 2*u], tr[12, 2*u]), "sm1_wait": d(tr[5, 2*u+1], tr[4, 2*u+1]),
           "sm1_work": d(tr[6, 2*u+1], tr[5, 2*u+1])}
    print(json.dumps(row))
