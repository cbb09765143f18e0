"""HostChunkStream (pipelined H2D / chunk step / D2H from pinned host buffers) must return exactly
what cpa_chunk_step returns for the same inputs, step by step, with the copies of neighbouring steps
overlapping (double-buffered staging, three streams)."""
import numpy as np
import pytest
import torch

import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool
from tests.gpu_helpers import to_dev_bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg_name,graphs", [("tiny", False), ("llama8b_32k", False), ("llama8b_32k", True)])
def test_host_stream_matches_chunk_step(cfg_name, graphs):
    cfg = CONFIGS[cfg_name]
    seed = 16839
    k, v = make_kv(cfg, seed)
    P, C, L = cfg.chunk_geometry()
    bs = cfg.block_size
    pt, npages = page_layout(cfg.batch, -(-L // bs), seed)
    cache = cpa.PagedKVCache(to_dev_bf16(to_pool(k, pt, npages, bs)), to_dev_bf16(to_pool(v, pt, npages, bs)),
                             torch.from_numpy(pt).cuda())
    p = cpa.make_params(cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, bs, C, P, alpha=0.06)
    kc = to_dev_bf16(k[:, :, P:].transpose(0, 2, 1, 3))
    vc = to_dev_bf16(v[:, :, P:].transpose(0, 2, 1, 3))
    qs = [to_dev_bf16(make_q(cfg, seed + i)) for i in range(4)]  # four different chunks of queries
    # reference: plain chunk_step, one at a time
    t_ref = cpa.alloc_tables(p)
    refs = []
    for q in qs:
        o = torch.empty(q.shape, dtype=torch.bfloat16, device="cuda")
        cpa.chunk_step(p, q, cache, t_ref, o, kc, vc)
        refs.append(o.cpu())
    torch.cuda.synchronize()
    runner = cpa.HostChunkStream(p, cache, cpa.alloc_tables(p), tuple(qs[0].shape), tuple(kc.shape), graphs=graphs)
    hq = [q.cpu().pin_memory() for q in qs]
    hk, hv = kc.cpu().pin_memory(), vc.cpu().pin_memory()
    ho = [torch.full(q.shape, float("nan"), dtype=torch.bfloat16).pin_memory() for q in qs]
    for i in range(len(qs)):
        runner.submit(hq[i], ho[i], hk, hv)
    runner.synchronize()
    for i in range(len(qs)):
        assert torch.equal(ho[i], refs[i]), i
