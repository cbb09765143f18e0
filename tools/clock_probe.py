"""Clock / power of the attention kernel under sustained load: back-to-back launches of the 128K
sparse (or dense) attention for ~SECS seconds while nvidia-smi samples clocks.sm and power.draw.instant
every 10 ms; prints median clock, power and the TFLOP/s achieved over the window (CUDA events).

  CFG=llama8b_128k SECS=3 DENSE=0 python tools/clock_probe.py
"""
import os, sys, json, subprocess, threading, time, statistics
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
cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), dev(to_pool(v, pt, npg, bs)).half(), torch.from_numpy(pt).cuda())
dq = dev(q); del k, v
p = cpa.make_params(cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, bs, C, P, alpha=0.06, flags=cpa.F_V_F16)
o = torch.empty(cfg.batch, C, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
t = cpa.alloc_tables(p); ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
cpa.build_tables(p, dq, cache, t, workspace=ws)
dense = os.environ.get("DENSE", "0") == "1"
tab = None if dense else t
ip = t.kv_indptr.cpu().numpy(); ix = t.kv_indices.cpu().numpy()[: ip[-1]]
E = cfg.num_q_heads // cfg.num_kv_heads
flops = 0.0  # exact causal pairs on tabled blocks (bench.py's algorithmic count)
for r in range(cfg.batch * (cfg.num_q_heads // E)):
    js = np.arange(-(-L // bs)) if dense else ix[ip[r]:ip[r + 1]]
    pos = P + np.arange(C)
    for j in js:
        lo = j * bs; hi = min(lo + bs, L)
        flops += np.clip(pos - lo + 1, 0, hi - lo).sum()
flops *= 4 * cfg.head_dim * E
for _ in range(5): cpa.paged_attention(p, dq, cache, tab, o, workspace=ws)
torch.cuda.synchronize()
q_ = "clocks.sm,power.draw.instant,clocks_event_reasons.sw_power_cap,temperature.gpu"
proc = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q_}", "--format=csv,noheader,nounits", "-lms", "10"],
                        stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
samples = []
threading.Thread(target=lambda: [samples.append(l.strip().split(", ")) for l in proc.stdout], daemon=True).start()
time.sleep(1.0); samples.clear()
secs = float(os.environ.get("SECS", "3")); n = 0
a = torch.cuda.Event(True); b = torch.cuda.Event(True); a.record()
t0 = time.time()
while time.time() - t0 < secs:
    for _ in range(20): cpa.paged_attention(p, dq, cache, tab, o, workspace=ws)
    n += 20
    torch.cuda.synchronize()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / n
snap = list(samples)
proc.terminate()
num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else None
clk = [num(s[0]) for s in snap if len(s) > 1 and num(s[0])]
pw = [num(s[1]) for s in snap if len(s) > 1 and num(s[1])]
print(json.dumps({"cfg": cfg.name, "mode": "dense" if dense else "sparse", "launches": n, "ms_per_launch": round(ms, 4),
                  "tflops": round(flops / ms / 1e9, 1), "sm_mhz_median": statistics.median(clk) if clk else None,
                  "sm_mhz_min": min(clk) if clk else None, "power_w_median": statistics.median(pw) if pw else None,
                  "power_w_max": max(pw) if pw else None, "samples": len(snap),
                  "power_cap_active_frac": round(sum(1 for s in snap if len(s) > 2 and s[2].startswith("Active")) / max(1, len(snap)), 2),
                  "temp_c": snap[-1][3] if snap and len(snap[-1]) > 3 else None}))
