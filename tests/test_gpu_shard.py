"""KV-group sharding on one GPU: running the chunk step rank by rank on head slices (each rank with
its own page pool holding only its KV heads, q/o passed as strided head slices of the full tensors)
must reproduce the unsharded step bit for bit -- tables row by row and every output element -- since
every table row and every attention row is per (b, execution group)."""
import numpy as np
import pytest
import torch

import paper_2605_16839_b200 as cpa
from paper_2605_16839_b200.shard import head_shard
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool
from tests.gpu_helpers import tables_to_numpy, to_dev_bf16

pytestmark = pytest.mark.gpu


def _run(cfg, q, k, v, kv_heads, q_heads, o_full, seed):
    P, C, L = cfg.chunk_geometry()
    bs = cfg.block_size
    nkvb = -(-L // bs)
    pt, npages = page_layout(cfg.batch, nkvb, seed + kv_heads.start)
    kk, vv = k[:, kv_heads.start:kv_heads.stop], v[:, kv_heads.start:kv_heads.stop]
    cache = cpa.PagedKVCache(to_dev_bf16(to_pool(kk, pt, npages, bs)), to_dev_bf16(to_pool(vv, pt, npages, bs)),
                             torch.from_numpy(pt).cuda())
    Hq = cfg.num_q_heads
    p = cpa.make_params(cfg.batch, len(q_heads), len(kv_heads), cfg.head_dim, bs, C, P, alpha=0.06,
                        q_token_stride=Hq * cfg.head_dim)
    t = cpa.alloc_tables(p)
    qs = q[:, :, q_heads.start:q_heads.stop]       # strided head slice of the full q
    os_ = o_full[:, :, q_heads.start:q_heads.stop]  # written in place into the full output
    cpa.chunk_step(p, qs, cache, t, os_)
    torch.cuda.synchronize()
    return tables_to_numpy(t)


@pytest.mark.parametrize("cfg_name,world", [("tiny", 2), ("llama8b_32k", 2), ("llama8b_32k", 8)])
def test_sharded_equals_unsharded(cfg_name, world):
    cfg = CONFIGS[cfg_name]
    seed = 16839
    k, v = make_kv(cfg, seed)
    q = to_dev_bf16(make_q(cfg, seed))
    P, C, L = cfg.chunk_geometry()
    shape = (cfg.batch, C, cfg.num_q_heads, cfg.head_dim)
    o_ref = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    ip_ref, ix_ref = _run(cfg, q, k, v, range(cfg.num_kv_heads), range(cfg.num_q_heads), o_ref, seed)
    o_sh = torch.full(shape, float("nan"), dtype=torch.bfloat16, device="cuda")
    Gn = cfg.num_q_heads // cfg.group_size
    for r in range(world):
        kvh, qh = head_shard(cfg.num_q_heads, cfg.num_kv_heads, world, r)
        ip, ix = _run(cfg, q, k, v, kvh, qh, o_sh, seed)
        per = Gn // world
        for b in range(cfg.batch):
            for gl in range(per):
                G = b * Gn + r * per + gl
                rl = b * per + gl
                assert np.array_equal(ix[ip[rl]:ip[rl + 1]], ix_ref[ip_ref[G]:ip_ref[G + 1]])
    assert torch.equal(o_sh, o_ref)
