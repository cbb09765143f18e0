"""Every-row parity at full size, in bench.py's exact launch configuration.

For the 32K and 128K BASELINE configs: the bench's seeded inputs, its page layout, the fp16 V pool
(CPA_F_V_F16), the chunk's K/V re-appended, and the chunk step (append + estimator + tables +
attention) captured in a CUDA graph and replayed -- then
  * the tables are compared with the fp64 oracle's bit for bit;
  * EVERY output (B*C*Hq*d: 8.4M at 32K, 16.7M at 128K) is compared with the oracle's row
    (oracle/compact_attention.py unchanged, computed on all host cores by tests/oracle_pool.py):
    fp32 output: max|d| <= 1e-2 x RMS (north_star; R13);
    bf16 output (what bench.py times): equal to the fp32 output rounded to bf16, hence
    |d| <= 1e-2 x RMS + 2^-9 |O| (bf16's half-ulp; the output dtype fixes the extra term).
The statistics are printed and, with CPA_PARITY_OUT=<dir>, written there as JSON."""
import json
import os
import time

import numpy as np
import pytest
import torch

import oracle as O
import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool
from tests.gpu_helpers import tables_to_numpy
from tests.oracle_pool import oracle_all_rows

pytestmark = pytest.mark.gpu

ALPHA, RHO = 0.06, 0.30  # bench.py's workload parameters
ATOL_REL = 1e-2


def _bench_step(cfg_name):
    """bench.py's GPU arm at N=1, reduced to the launch it times: returns (tables, o32, o16)."""
    cfg = CONFIGS[cfg_name]
    seed = 16839 + list(CONFIGS).index(cfg_name)
    P, C, L = cfg.chunk_geometry()
    bs, d = cfg.block_size, cfg.head_dim
    k, v = make_kv(cfg, seed, RHO)
    q = make_q(cfg, seed)
    nkvb = -(-L // bs)
    pt, npages = page_layout(cfg.batch, nkvb, seed)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    cache = cpa.PagedKVCache(dev(to_pool(k, pt, npages, bs)), dev(to_pool(v, pt, npages, bs)).half(),
                             torch.from_numpy(pt).cuda())
    dq = dev(q)
    kc = dev(k[:, :, P:].transpose(0, 2, 1, 3))
    vc = dev(v[:, :, P:].transpose(0, 2, 1, 3))
    outs = {}
    for f32 in (True, False):
        p = cpa.make_params(cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, d, bs, C, P, alpha=ALPHA,
                            flags=cpa.F_V_F16 | (cpa.F_OUT_F32 if f32 else 0))
        tables = cpa.alloc_tables(p)
        ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
        o = torch.full((cfg.batch, C, cfg.num_q_heads, d), float("nan"),
                       dtype=torch.float32 if f32 else torch.bfloat16, device="cuda")
        for _ in range(2):
            cpa.chunk_step(p, dq, cache, tables, o, kc, vc, workspace=ws)
        torch.cuda.synchronize()
        o.fill_(float("nan"))
        tables.kv_indices.fill_(-1)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cpa.prepare_chunk(p, dq, cache, tables, kc, vc, workspace=ws)
            cpa.paged_attention(p, dq, cache, tables, o, workspace=ws)
        g.replay()
        g.replay()
        torch.cuda.synchronize()
        outs[f32] = (tables_to_numpy(tables), o.float().cpu().numpy().astype(np.float64))
    assert np.array_equal(outs[True][0][0], outs[False][0][0]) and np.array_equal(outs[True][0][1], outs[False][0][1])
    return (q, k, v, P, C, seed), outs[True][0], outs[True][1], outs[False][1]


@pytest.mark.parametrize("cfg_name", ["llama8b_32k", "llama8b_128k"])
def test_every_row_bench_config(cfg_name):
    cfg = CONFIGS[cfg_name]
    (q, k, v, P, C, seed), (ip, ix), o32, o16 = _bench_step(cfg_name)
    bs, E = cfg.block_size, cfg.group_size
    # oracle tables (estimator -> threshold -> unions -> CSR) on the same inputs: bit-exact
    m = O.block_scores_pooled(q, k, P, bs)
    M = O.threshold_mask(m, ALPHA, C, P, bs)
    rip, rix = O.tables_from_mask(M, E, P // bs)
    assert np.array_equal(ip, rip) and np.array_equal(ix, rix), "tables differ from the oracle's"
    del q, k, v, m, M
    t0 = time.time()
    ref = oracle_all_rows(cfg_name, seed, RHO, E, rip, rix, P, bs)
    t_oracle = time.time() - t0
    assert np.isfinite(ref).all()
    rms = float(np.sqrt(np.mean(ref ** 2)))
    d32 = np.abs(o32 - ref)
    err32 = float(d32.max()) / rms
    # bf16 output = fp32 output rounded to bf16 (same kernels; only the epilogue store differs)
    assert np.array_equal(torch.from_numpy(o32).float().to(torch.bfloat16).float().double().numpy(), o16)
    d16 = np.abs(o16 - ref)
    err16 = float(d16.max()) / rms
    ratio16 = float((d16 / (ATOL_REL * rms + 2.0 ** -9 * np.abs(ref))).max())
    stats = {"config": cfg_name, "outputs": int(ref.size), "rms": rms, "max_abs_err_over_rms_f32": err32,
             "mean_abs_err_over_rms_f32": float(d32.mean()) / rms, "max_abs_err_over_rms_bf16": err16,
             "bf16_bound_ratio": ratio16, "tabled_blocks": int(ip[-1]), "oracle_wall_s": round(t_oracle, 1),
             "launch": "CUDA graph replay of prepare_chunk (append + estimator + tables) + paged_attention, fp16 V pool"}
    print(json.dumps(stats))
    out_dir = os.environ.get("CPA_PARITY_OUT")
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, f"parity_full_{cfg_name}.json"), "w") as f:
            json.dump(stats, f, indent=1)
    assert err32 <= ATOL_REL, stats
    assert ratio16 <= 1.0, stats
