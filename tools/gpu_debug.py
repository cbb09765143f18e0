"""Step-by-step GPU bring-up checks (each step in its own process under `timeout`)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2605_16839_b200 as cpa
from synth.workload import random_qkv, CONFIGS, make_kv, make_q
from tests.gpu_helpers import Case, tables_to_numpy, mask_to_bits, scores_to_bhij, rel_err

step = sys.argv[1]
if step == "maskin":
    M = np.zeros((1, 2, 1, 3), bool); M[0, 0, 0, :2] = True; M[0, 1, 0, 2] = True
    p = cpa.make_params(1, 2, 2, 64, 16, 16, 32, flags=cpa.F_MASK_IN)
    pages = torch.zeros(1, 2, 16, 64, dtype=torch.bfloat16, device="cuda")
    cache = cpa.PagedKVCache(pages, pages, torch.zeros(1, 3, dtype=torch.int32, device="cuda"))
    t = cpa.alloc_tables(p, status=True); t.mask_bits = torch.from_numpy(mask_to_bits(M)).cuda()
    cpa.build_tables(p, None, cache, t); torch.cuda.synchronize()
    print("maskin", tables_to_numpy(t), t.dev_status.item())
elif step in ("scores", "scores128"):
    d, bs, C, P = (64, 16, 64, 448) if step == "scores" else (128, 128, 256, 512)
    q, k, v = random_qkv(1, 8, 2, d, C, P + C, seed=1)
    case = Case(q, k, v, P, bs, seed=3)
    p = case.params; p.flags |= cpa.F_SCORES_OUT
    t = cpa.alloc_tables(p, scores=True)
    cpa.build_tables(p, case.dq, case.cache, t); torch.cuda.synchronize()
    m_ref = O.block_scores_pooled(q, k, P, bs); m_gpu = scores_to_bhij(t.scores, p)
    fin = np.isfinite(m_ref)
    print(step, "finite-pattern equal", np.array_equal(fin, np.isfinite(m_gpu)), "max err", np.abs(m_gpu[fin]-m_ref[fin]).max())
    print(m_ref[0,0,0,:8]); print(m_gpu[0,0,0,:8])
elif step in ("attn", "attn128", "attnb", "attn128b"):
    B, Hq, Hkv, d, bs, C, P = (1, 8, 2, 64, 16, 64, 448) if step.startswith("attn") and "128" not in step else (1, 8, 2, 128, 128, 256, 512)
    q, k, v = random_qkv(B, Hq, Hkv, d, C, P + C, seed=2)
    case = Case(q, k, v, P, bs, seed=5)
    p = case.params; p.flags |= cpa.F_OUT_F32 | (cpa.F_P_BF16 if step.endswith("b") else 0)
    o = case.out(True)
    cpa.paged_attention(p, case.dq, case.cache, None, o); torch.cuda.synchronize()
    got = o.cpu().numpy().astype(np.float64); ref = O.dense_causal_attention(q, k, v, P)
    print(step, "rel err", rel_err(got, ref)); print(ref[0, 5, 0, :6]); print(got[0, 5, 0, :6])
    bad = np.abs(got - ref).max(axis=-1)
    print("worst rows (p,h):", np.argwhere(bad[0] > 0.05)[:10])

if step == "dump128":
    B, Hq, Hkv, d, bs, C, P = (1, 8, 2, 128, 128, 256, 512)
    q, k, v = random_qkv(B, Hq, Hkv, d, C, P + C, seed=2)
    case = Case(q, k, v, P, bs, seed=5)
    p = case.params; p.flags |= cpa.F_OUT_F32
    o = case.out(True)
    cpa.paged_attention(p, case.dq, case.cache, None, o); torch.cuda.synchronize()
    np.save("gpurun_out/attn128.npy", o.cpu().numpy())
    print("saved")
