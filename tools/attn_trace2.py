"""Per-block event trace of cluster 0 (leader CTA) of k_paged_attn_2cta (build with -DCPA_TRACE)."""
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
VF16 = os.environ.get("V_F16", "1") == "1"  # fp16 V pool (product default)
vpool = dev(to_pool(v, pt, npg, bs))
cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), vpool.half() if VF16 else vpool, torch.from_numpy(pt).cuda())
dq = dev(q)
p = cpa.make_params(cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, bs, C, P, alpha=0.06,
                    flags=cpa.F_V_F16 if VF16 else 0)
o = torch.empty(cfg.batch, C, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
t = cpa.alloc_tables(p); cpa.build_tables(p, dq, cache, t)
for _ in range(3): cpa.paged_attention(p, dq, cache, t, o)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (32 * 2048))()
cpa.lib().cpa_debug_trace2(buf)
tr = np.frombuffer(buf, dtype=np.int64).reshape(32, 2048)
N = int((tr[2] > 0).sum())
d = lambda a, b: int(a - b)
per = [d(tr[2, n + 1], tr[2, n]) for n in range(2, N - 2)]
print("blocks", N, "median period per 128-key page (cycles)", int(np.median(per)))
for n in list(range(0, 4)) + list(range(N // 2, N // 2 + 4)):
    rec = {"n": n, "period": d(tr[2, n + 1], tr[2, n]) if n + 1 < N else 0,
           "mma_vready_wait": d(tr[1, n], tr[3, n - 1]) if n > 0 else 0, "mma_p_wait": d(tr[2, n], tr[1, n]),
           "mma_pv_issue": d(tr[9, n], tr[2, n]), "mma_k_wait": d(tr[10, n], tr[9, n]),
           "mma_s_issue": d(tr[3, n], tr[10, n]), "conv": d(tr[8, n], tr[7, n])}
    for w in (0, 1):  # both softmax WGs work on every page (key-column halves)
        o_ = 16 * w
        rec[f"wg{w}"] = {"wait": d(tr[5 + o_, n], tr[4 + o_, n]), "ld_max": d(tr[11 + o_, n], tr[5 + o_, n]),
                         "exp": d(tr[12 + o_, n], tr[11 + o_, n]), "tail": d(tr[6 + o_, n], tr[12 + o_, n])}
    print(json.dumps(rec))
# absolute timeline (cycles from the first listed event) of a few mid-kernel pages
b0 = N // 2
t0 = int(tr[5, b0])
for n in range(b0, b0 + 6):
    r = lambda e: int(tr[e, n]) - t0
    print(f"page {n}: wg0 stag_arrived {r(13):6d} wg1 top {r(20):6d} stag_passed {r(29):6d} | " + " | ".join(
        f"wg{w} s_ready {r(5 + 16*w):6d} max {r(11 + 16*w):6d} exp {r(12 + 16*w):6d} arrive {r(6 + 16*w):6d}"
        for w in (0, 1)) + f" || mma: p_seen {r(2):6d} pv_issued {r(9):6d} s(n+2)_issued {r(3):6d}")

# tensor-pipe completions observed by the idle converter warps (fp16 pool): per page, cycles from
# WG0's s_ready of that page
print("completions (relative to page 165's WG0 s_ready):")
for n in range(b0, b0 + 6):
    r = lambda e: int(tr[e, n]) - t0
    print(f"page {n}: K landed {r(31):6d} | S(n) done {r(14):6d} | PV(n,0) done {r(15):6d} | PV(n,1)+S(n+2) done {r(30):6d}"
          f" || mma: p_seen {r(2):6d} pv1_issued {r(9):6d} s(n+2)_issued {r(3):6d} | wg1 P arrive {r(22):6d}")
