"""Dense reference for the baseline kernel: torch SDPA (cuDNN / flash / efficient backends) on the
same 128K final chunk with CONTIGUOUS K/V (no paging), bottom-right causal alignment (query p at
absolute position P + p), GQA 32/8, bf16. Compared with cpa_paged_attention(tables=NULL)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.nn.attention import SDPBackend, sdpa_kernel
from torch.nn.attention.bias import causal_lower_right
import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool
cfg = CONFIGS[os.environ.get("CFG", "llama8b_128k")]
seed = 16839 + list(CONFIGS).index(cfg.name)
P, C, L = cfg.chunk_geometry(); bs, d, Hq, Hkv = cfg.block_size, cfg.head_dim, cfg.num_q_heads, cfg.num_kv_heads
k, v = make_kv(cfg, seed); q = make_q(cfg, seed)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
qt = dev(q).transpose(1, 2).contiguous()          # [B, Hq, C, d]
kt, vt = dev(k), dev(v)                            # [B, Hkv, L, d]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def timed(fn, reps=8):
    for _ in range(2): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        flush.zero_(); a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))
nkvb = -(-L // bs); pt, npg = page_layout(cfg.batch, nkvb, seed)
cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs)), torch.from_numpy(pt).cuda())
p = cpa.make_params(cfg.batch, Hq, Hkv, d, bs, C, P)
ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
o = torch.empty(cfg.batch, C, Hq, d, dtype=torch.bfloat16, device="cuda")
dq = dev(q)
t_ours = timed(lambda: cpa.paged_attention(p, dq, cache, None, o, workspace=ws))
ref = o.transpose(1, 2).float()
flops = 4 * d * Hq * (C * P + C * (C + 1) // 2)
print(json.dumps({"impl": "libcpa dense paged", "ms": round(t_ours, 4), "tflops": round(flops / t_ours / 1e9, 1)}), flush=True)
bias = causal_lower_right(C, L)
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    rec = {"impl": f"torch sdpa {name} (contiguous KV)"}
    try:
        with sdpa_kernel([be]):
            f = lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=bias, enable_gqa=True)
            out = f()
            t = timed(f)
        rec.update(ms=round(t, 4), tflops=round(flops / t / 1e9, 1),
                   max_abs_diff_over_rms_vs_libcpa=round(float((out.float() - ref).abs().max() / ref.pow(2).mean().sqrt()), 5))
    except Exception as ex:  # noqa: BLE001
        rec["error"] = f"{type(ex).__name__}: {str(ex)[:200]}"
    print(json.dumps(rec), flush=True)
