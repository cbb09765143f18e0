"""world_size-2 gloo test of the multi-GPU path's host logic on CPU: each rank runs the chunk step
for its KV-group shard (here through the fp64 oracle, standing in for the rank's GPU), the head
outputs are all-gathered with the product's helper, and the result must equal the unsharded step:
tables bitwise (rows are per (b, g)) and outputs exactly (no cross-rank reduction)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2605_16839_b200.shard import allgather_heads, head_shard, heads_view
from synth.workload import CONFIGS, make_kv, make_q


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CONFIGS["tiny"]
    P, C, L = cfg.chunk_geometry()
    kvh, qh = head_shard(cfg.num_q_heads, cfg.num_kv_heads, world, rank)
    k, v = make_kv(cfg, 16839, kv_heads=kvh)   # each rank regenerates only its slice
    q = make_q(cfg, 16839, q_heads=qh)
    r = O.chunk_step(q, k, v, P, cfg.block_size, alpha=0.06)
    o_all = allgather_heads(torch.from_numpy(r["O"]))
    ip = torch.from_numpy(r["indptr"].astype(np.int64))
    ipl = [torch.empty_like(ip) for _ in range(world)]
    dist.all_gather(ipl, ip)
    n = torch.tensor([len(r["indices"])])
    ns = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    ix = torch.zeros(int(max(x.item() for x in ns)), dtype=torch.int64)
    ix[: len(r["indices"])] = torch.from_numpy(r["indices"].astype(np.int64))
    ixl = [torch.empty_like(ix) for _ in range(world)]
    dist.all_gather(ixl, ix)
    if rank == 0:
        np.savez(result_path, o=heads_view(o_all).numpy(),
                 **{f"ip{i}": ipl[i].numpy() for i in range(world)},
                 **{f"ix{i}": ixl[i].numpy()[: ns[i].item()] for i in range(world)})
    dist.barrier()
    dist.destroy_process_group()


def test_head_shard_ranges():
    assert head_shard(32, 8, 8, 3) == (range(3, 4), range(12, 16))
    assert head_shard(32, 8, 2, 1) == (range(4, 8), range(16, 32))
    with pytest.raises(ValueError):
        head_shard(32, 8, 3, 0)


def test_two_rank_gloo_equals_unsharded(tmp_path):
    world = 2
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    res = np.load(path)
    cfg = CONFIGS["tiny"]
    P, C, L = cfg.chunk_geometry()
    k, v = make_kv(cfg, 16839)
    q = make_q(cfg, 16839)
    full = O.chunk_step(q, k, v, P, cfg.block_size, alpha=0.06)
    assert np.array_equal(res["o"], full["O"])
    # rank r's CSR rows are the unsharded rows of its groups
    Gn = cfg.num_q_heads // cfg.group_size
    per = Gn // world
    for r in range(world):
        ip, ix = res[f"ip{r}"], res[f"ix{r}"]
        for g in range(per):
            G = r * per + g
            a = full["indices"][full["indptr"][G]:full["indptr"][G + 1]]
            b = ix[ip[g]:ip[g + 1]]
            assert np.array_equal(a, b)
