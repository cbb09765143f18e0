"""Multi-GPU plumbing: shard the chunk step by KV-head group, all-gather the head outputs.

Every block table is per (batch, execution group), so rank r of W owns KV heads
[r*Hkv/W, (r+1)*Hkv/W) and exactly their query heads; estimator, masks, tables and attention are
rank-local. The only exchange is one all-gather of the per-rank head outputs (the attention half of
the paper's TP=2 setting). Host-side bookkeeping only -- no math here.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_shard(num_q_heads: int, num_kv_heads: int, world: int, rank: int):
    """(kv_heads range, q_heads range) owned by `rank`; KV heads must divide evenly over ranks."""
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} KV heads do not shard over {world} ranks")
    if num_q_heads % num_kv_heads:
        raise ValueError("num_q_heads must be a multiple of num_kv_heads")
    hkv = num_kv_heads // world
    e = num_q_heads // num_kv_heads
    return range(rank * hkv, (rank + 1) * hkv), range(rank * hkv * e, (rank + 1) * hkv * e)


def allgather_heads(o_local: torch.Tensor, out: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """All-gather [B, C, Hq/W, d] per-rank outputs into [W, B, C, Hq/W, d] (NCCL: one
    all_gather_into_tensor over NVLink; gloo: list all_gather, used by the CPU tests)."""
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty((world,) + tuple(o_local.shape), dtype=o_local.dtype, device=o_local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, o_local.contiguous(), group=group)
    else:  # gloo (CPU tests, single-device bench smoke): gather through host memory
        host = [torch.empty(tuple(o_local.shape), dtype=o_local.dtype) for _ in range(world)]
        dist.all_gather(host, o_local.detach().cpu(), group=group)
        out.copy_(torch.stack(host))
    return out


def heads_view(o_all: torch.Tensor) -> torch.Tensor:
    """[W, B, C, Hq/W, d] -> [B, C, Hq, d] view (rank-major head order = global head order)."""
    W, B, C, H, d = o_all.shape
    return o_all.permute(1, 2, 0, 3, 4).reshape(B, C, W * H, d)
