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


@pytest.mark.parametrize("cfg_name,world,f32", [("tiny", 2, True), ("llama8b_32k", 2, False),
                                                ("llama8b_32k", 4, False), ("llama8b_32k", 8, False),
                                                ("llama8b_128k", 8, True)])
def test_fused_peer_allgather(cfg_name, world, f32):
    """cpa_chunk_step_peer on W simulated ranks of one GPU (each rank on its own stream, its peers'
    gathered buffers and signal pads plain device tensors, so the P2P stores are local stores): every
    rank's gathered buffer [B, C, Hq, d] must equal the unsharded chunk step bit for bit, and the
    barrier must complete (dev_status 0) for several consecutive epochs."""
    cfg = CONFIGS[cfg_name]
    seed = 16839
    k, v = make_kv(cfg, seed)
    q = to_dev_bf16(make_q(cfg, seed))
    P, C, L = cfg.chunk_geometry()
    bs, d, Hq = cfg.block_size, cfg.head_dim, cfg.num_q_heads
    dt = torch.float32 if f32 else torch.bfloat16
    shape = (cfg.batch, C, Hq, d)
    nkvb = -(-L // bs)
    # unsharded reference
    pt, npages = page_layout(cfg.batch, nkvb, seed)
    cache = cpa.PagedKVCache(to_dev_bf16(to_pool(k, pt, npages, bs)), to_dev_bf16(to_pool(v, pt, npages, bs)),
                             torch.from_numpy(pt).cuda())
    pf = cpa.make_params(cfg.batch, Hq, cfg.num_kv_heads, d, bs, C, P, alpha=0.06,
                         flags=cpa.F_OUT_F32 if f32 else 0)
    o_ref = torch.empty(shape, dtype=dt, device="cuda")
    cpa.chunk_step(pf, q, cache, cpa.alloc_tables(pf), o_ref)
    torch.cuda.synchronize()
    # W ranks: own shard of the pool, own q slice (contiguous copy, as a rank would hold it)
    outs = [torch.full(shape, float("nan"), dtype=dt, device="cuda") for _ in range(world)]
    pads = [torch.zeros(world, dtype=torch.int32, device="cuda") for _ in range(world)]
    status = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(world)]
    ranks = []
    for r in range(world):
        kvh, qh = head_shard(Hq, cfg.num_kv_heads, world, r)
        ptr, npr = page_layout(cfg.batch, nkvb, seed + 7 * r)
        kk, vv = k[:, kvh.start:kvh.stop], v[:, kvh.start:kvh.stop]
        c = cpa.PagedKVCache(to_dev_bf16(to_pool(kk, ptr, npr, bs)), to_dev_bf16(to_pool(vv, ptr, npr, bs)),
                             torch.from_numpy(ptr).cuda())
        p = cpa.make_params(cfg.batch, len(qh), len(kvh), d, bs, C, P, alpha=0.06,
                            flags=cpa.F_OUT_F32 if f32 else 0)
        peers = cpa.PeerOut(world, r, [o.data_ptr() for o in outs], [x.data_ptr() for x in pads],
                            timeout_ms=5000, dev_status=status[r])
        ranks.append((p, q[:, :, qh.start:qh.stop].contiguous(), c, cpa.alloc_tables(p), peers,
                      torch.cuda.Stream(), torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")))
    for epoch in range(3):
        for o in outs:
            o.fill_(float("nan"))
        torch.cuda.synchronize()
        for p, qr, c, t, peers, st, ws in ranks:  # each rank owns its workspace, like a real rank
            cpa.chunk_step_peer(p, qr, c, t, peers, workspace=ws, stream=st)
        torch.cuda.synchronize()
        assert [int(s.item()) for s in status] == [0] * world
        assert all(int(x) == epoch + 1 for pad in pads for x in pad.cpu())
        for w in range(world):
            if cfg_name == "llama8b_128k":
                # a 1-group shard at 128K runs the persistent stream-K grid (the unsharded step does
                # not): equal up to the fp32 merge of cut units
                rms = float(o_ref.double().pow(2).mean().sqrt())
                assert float((outs[w] - o_ref).abs().max()) <= 5e-3 * rms, (epoch, w)
            else:
                assert torch.equal(outs[w], o_ref), (epoch, w)
    # CUDA-graph replays of every rank's step: the barrier keeps its epochs on the device
    graphs = []
    for p, qr, c, t, peers, st, ws in ranks:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            cpa.chunk_step_peer(p, qr, c, t, peers, workspace=ws)
        graphs.append((g, st))
    torch.cuda.synchronize()
    # capture does not execute: pads still hold epoch 3
    assert all(int(x) == 3 for pad in pads for x in pad.cpu())
    for rep in range(2):
        for o in outs:
            o.fill_(float("nan"))
        torch.cuda.synchronize()
        for g, st in graphs:
            with torch.cuda.stream(st):
                g.replay()
        torch.cuda.synchronize()
        assert [int(s.item()) for s in status] == [0] * world
        assert all(int(x) == 4 + rep for pad in pads for x in pad.cpu())
        for w in range(world):
            assert torch.isfinite(outs[w].float()).all(), (rep, w)
