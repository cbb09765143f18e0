#!/usr/bin/env python
"""Benchmark of the CompactAttention chunked-prefill hot path on B200 (BASELINE.json metric).

One step = one whole chunk step through the C ABI (cpa_chunk_step): append the chunk's K/V into
the pages, pooled-query estimator, threshold mask, Q-block + intra-group union, CSR tables and
paged attention over the tabled blocks, for the FINAL chunk of the workload (KV = full context).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama8b_128k] [--impl reference]

Prints ONE JSON line (rank 0). value = attention ms per chunk (lower is better), inputs resident
in HBM, L2 flushed before every timed step (a 512 MiB write), CUDA events on the launch stream,
max over ranks. N > 1: KV-head groups are sharded over ranks (one KV group per GPU at N=8) and
the per-rank head outputs are all-gathered each step (strong scaling: one chunk) -- by default
inside the attention kernel (P2P stores into every rank's symmetric-memory buffer over NVLink + a
signal barrier, cpa_chunk_step_peer); --collective nccl times NCCL all_gather_into_tensor instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth.workload import CONFIGS, make_kv, make_q, page_layout, to_pool  # noqa: E402

METRIC = "attention ms/chunk & speedup vs dense paged attn at 128K ctx (LLaMA-3.1-8B shape)"
UNIT = "ms/chunk"
ALPHA = 0.06          # PAPER.md:282 (CA-FP on LLaMA-3.1-8B)
RHO = 0.30            # needle density calibrated to the paper's 89.8% -> 70.2% sparsity


def seed_of(name):
    return 16839 + list(CONFIGS).index(name)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["bf16_tflops"], pk["hbm_gbs"], "measured (MEASURED_PEAKS.json, burst)"
    except Exception:
        return 1590.0, 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------ algorithmic work
def attention_flops(indptr, indices, C, P, bs, E, d):
    """4*d*E*sum over rows r of sum_p |A(p)| (exact causal pairs on the tabled blocks)."""
    L = P + C
    total = 0
    p_last = P + C  # exclusive bound of absolute query positions
    for r in range(len(indptr) - 1):
        js = np.asarray(indices[indptr[r]:indptr[r + 1]], np.int64)
        lo = js * bs
        hi = np.minimum(lo + bs, L)
        pre = hi <= P + 1  # every query sees the whole block
        total += int(((hi - lo)[pre]).sum()) * C
        for a, b in zip(lo[~pre], hi[~pre]):  # chunk blocks: sum_p max(0, min(b, P+p+1) - a)
            p = np.arange(C)
            total += int(np.clip(np.minimum(b, P + p + 1) - a, 0, None).sum())
    return 4 * d * E * total


def sparsity_report(bits, nkvb, pb, nqb, Hq, E_exec, E_kv):
    """Per-stage prefix sparsity (fraction of causal-valid PREFIX block slots not selected; the
    forced chunk blocks excluded, R14) from the GPU's mask bits [B, Hq, nqb, nwords]:
    pre-union, Q-block union, execution-group union, full-KV-group union."""
    b64 = bits.view(np.uint32).astype(np.uint64)
    B = b64.shape[0]
    M = ((b64[..., None] >> np.arange(32, dtype=np.uint64)) & 1).astype(bool).reshape(B, Hq, nqb, -1)[..., :pb]
    Mbar = M.any(axis=2)                                   # [B, Hq, pb]
    Gx = Mbar.reshape(B, Hq // E_exec, E_exec, pb).any(axis=2)
    Gk = Mbar.reshape(B, Hq // E_kv, E_kv, pb).any(axis=2)
    n = B * Hq * nqb * pb
    return {"pre_union": round(1 - M.sum() / n, 4),
            "q_block_union": round(1 - Mbar.sum() * nqb / n, 4),
            "exec_group_union": round(1 - np.repeat(Gx, E_exec, axis=1).sum() * nqb / n, 4),
            "kv_group_union": round(1 - np.repeat(Gk, E_kv, axis=1).sum() * nqb / n, 4)}


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, device_index=0):
        self.samples, self.proc, self.t = [], None, None
        self.idx = device_index

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 5.0:  # sampler live before timing starts
                time.sleep(0.01)
            self.samples.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------------------ CPU oracle leg
def cpu_oracle_sample(cfg, seed, q, k, v, P, C, budget_s=15.0):
    """Time the fp64 oracle (as it stands) on a bounded sample of the chunk step and extrapolate to
    ms/chunk: estimator for 2 query heads + attention for sampled query rows (rows/heads are
    independent, so the extrapolation is exact in work)."""
    import oracle as O
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count()
    bs, E = cfg.block_size, cfg.group_size
    B, Hq = cfg.batch, cfg.num_q_heads
    t0 = time.perf_counter()
    heads = [0, 1]
    m = O.block_scores_pooled(q[:, :, heads], k[:, :1], P, bs)
    t_est = (time.perf_counter() - t0) / (len(heads) * B) * B * Hq
    # tables of group 0 from the sampled heads' mask (the union is integer work; negligible)
    M = O.threshold_mask(m, ALPHA, C, P, bs)
    ip, ix = O.tables_from_mask(M, len(heads), P // bs)
    rng = np.random.default_rng(0)
    n_rows, t_attn = 0, 0.0
    t1 = time.perf_counter()
    while time.perf_counter() - t1 < budget_s and n_rows < 4096:
        rows = [(0, int(rng.integers(C)), int(rng.integers(2))) for _ in range(16)]
        O.paged_attention(q[:, :, :2], k[:, :1], v[:, :1], P, bs, ip, ix, E=2, rows=rows)
        n_rows += len(rows)
    t_attn = (time.perf_counter() - t1) / n_rows * B * C * Hq
    total_ms = (t_est + t_attn) * 1e3
    return {"value": total_ms, "unit": "ms/chunk", "cores": threads, "kind": "oracle",
            "sample": f"fp64 numpy oracle: pooled estimator for {len(heads)} of {B * Hq} (b,h) heads + "
                      f"attention for {n_rows} of {B * C * Hq} query rows, extrapolated linearly to the "
                      f"whole {cfg.name} final chunk"}


# ------------------------------------------------------------------------------ GPU arm
def peer_setup(torch, dist, cpa, full_shape, world, rank):
    """Symmetric-memory gathered output [B, C, Hq, d] + uint32 signal pads [W] on every rank, mapped
    into every peer (torch symmetric memory = CUDA IPC / fabric handles over NVLink)."""
    import torch.distributed._symmetric_memory as symm
    group = dist.group.WORLD
    try:
        symm.enable_symm_mem_for_group(group.group_name)
    except Exception:  # noqa: BLE001 -- newer torch enables it implicitly
        pass
    buf = symm.empty(full_shape, dtype=torch.bfloat16, device="cuda")
    hb = symm.rendezvous(buf, group)
    sig = symm.empty(world, dtype=torch.int32, device="cuda")
    sig.zero_()
    hs = symm.rendezvous(sig, group)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    dist.barrier()
    peers = cpa.PeerOut(world, rank, list(hb.buffer_ptrs), list(hs.buffer_ptrs), timeout_ms=20000,
                        dev_status=status)
    peers._keep = (buf, sig, hb, hs)
    return peers, buf


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2605_16839_b200 as cpa

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CPA_BENCH_ONE_DEVICE=1 (test only): every rank on cuda:0 with a gloo group, to exercise the
    # sharded code path on a single-GPU box; real runs use one GPU per rank and NCCL.
    one_dev = os.environ.get("CPA_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    backend = "gloo" if one_dev else "nccl"
    # CPA_BENCH_PEER_W1=1 (test only, under torchrun --nproc-per-node 1): a 1-rank NCCL group so the
    # fused peer path runs through real symmetric memory on a single-GPU box.
    force_peer = os.environ.get("CPA_BENCH_PEER_W1") == "1" and world == 1
    if world > 1 or force_peer:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def max_over_ranks(vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if one_dev else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.tolist()]
    cfg = CONFIGS[args.config]
    seed = seed_of(args.config)
    P, C, L = cfg.chunk_geometry()
    bs, d, E = cfg.block_size, cfg.head_dim, cfg.group_size
    from paper_2605_16839_b200.shard import allgather_heads, head_shard
    kvh, qh = head_shard(cfg.num_q_heads, cfg.num_kv_heads, world, rank)
    hkv_l, hq_l = len(kvh), len(qh)
    k, v = make_kv(cfg, seed, RHO, kv_heads=kvh)
    q = make_q(cfg, seed, q_heads=qh)
    nkvb = -(-L // bs)
    pt, npages = page_layout(cfg.batch, nkvb, seed)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    vpool = dev(to_pool(v, pt, npages, bs))
    if args.v_f16:  # CPA_F_V_F16: the V pool holds fp16 (exact for these bf16 values)
        vpool = vpool.half()
    cache = cpa.PagedKVCache(dev(to_pool(k, pt, npages, bs)), vpool, torch.from_numpy(pt).cuda())
    dq = dev(q)
    kc = dev(k[:, :, P:].transpose(0, 2, 1, 3))  # the chunk's own K/V [B, C, Hkv, d] (re-appended)
    vc = dev(v[:, :, P:].transpose(0, 2, 1, 3))
    E_exec = args.exec_group or E
    vflag = cpa.F_V_F16 if args.v_f16 else 0
    p = cpa.make_params(cfg.batch, hq_l, hkv_l, d, bs, C, P, alpha=ALPHA, exec_group_size=args.exec_group,
                        flags=(cpa.F_EXACT_SCORES if args.exact_scores else 0) | vflag)
    tables = cpa.alloc_tables(p)
    ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
    o = torch.empty(cfg.batch, C, hq_l, d, dtype=torch.bfloat16, device="cuda")
    o_all = torch.empty(world, cfg.batch, C, hq_l, d, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    # N > 1: the head-output all-gather is fused into the attention epilogue (P2P stores into every
    # rank's symmetric-memory buffer + a signal barrier, cpa_chunk_step_peer); NCCL all-gather after a
    # local step is the baseline (--collective nccl) and the fallback if symmetric memory is unavailable.
    collective = "none" if world == 1 and not force_peer else ("gloo all-gather" if one_dev else args.collective)
    peers = None
    if collective == "peer":
        try:
            peers, o_gathered = peer_setup(torch, dist, cpa, (cfg.batch, C, cfg.num_q_heads, d), world, rank)
            collective = "fused peer-store all-gather (NVLink P2P, cpa_chunk_step_peer)"
        except Exception as ex:  # noqa: BLE001 -- reported in the JSON line
            collective = f"nccl all-gather (symmetric memory unavailable: {type(ex).__name__}: {ex})"[:200]
    elif collective == "nccl":
        collective = "nccl all-gather"

    def step():
        if peers is not None:
            cpa.chunk_step_peer(p, dq, cache, tables, peers, kc, vc, workspace=ws)
            return
        cpa.chunk_step(p, dq, cache, tables, o, kc, vc, workspace=ws)
        if world > 1:
            allgather_heads(o, o_all)

    # The timed step is one replay of a CUDA graph of the whole chunk step (append, estimator, tables,
    # attention [, fused all-gather + barrier]): the C ABI is stream-ordered, never allocates or syncs,
    # so it captures as is; replays drop the per-kernel launch gaps (8% of the step at one KV group per
    # GPU). NCCL / gloo all-gather modes run directly.
    launch = "direct"
    step()  # one direct step: kernels per step for gpu_launches
    launches_per_step = cpa.last_launch_count()
    att_ev = None  # attention-kernel events inside the timed steps (roofline timing)
    if not args.no_graph and not one_dev and (world == 1 or peers is not None):
        step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        # thread_local: the NCCL watchdog thread may query events while this thread captures
        with torch.cuda.graph(graph, capture_error_mode="thread_local"):
            if peers is None:
                # cpa_chunk_step == append + build_tables + paged_attention (same workspace, same stream);
                # split here so that event nodes bracket the attention kernel inside every timed step
                att_ev = (torch.cuda.Event(enable_timing=True, external=True),
                          torch.cuda.Event(enable_timing=True, external=True))
                cpa.append_kv(p, kc, vc, cache)
                cpa.build_tables(p, dq, cache, tables, workspace=ws)
                att_ev[0].record()
                cpa.paged_attention(p, dq, cache, tables, o, workspace=ws)
                att_ev[1].record()
            else:
                step()
        torch.cuda.synchronize()
        step = graph.replay
        launch = "CUDA graph of the chunk step"

    att_in_step = []

    def timed(fn, iters, warm, inner=None):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            if inner is not None:
                inner.append(att_ev[0].elapsed_time(att_ev[1]))
        return ts

    # ---- headline: W warm-up steps, K timed steps, barrier + sync on both sides
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        ts = timed(step, args.steps, 0, att_in_step if att_ev is not None else None)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = max_over_ranks([float(np.mean(ts))])[0]
    if peers is not None and int(peers.dev_status.item()) != 0:
        raise RuntimeError(f"rank {rank}: peer barrier timed out waiting for rank {int(peers.dev_status.item()) - 1}")

    # ---- stage breakdown and the dense baseline (same kernels, tables = all blocks)
    reps = max(3, min(args.steps, 10))
    t_tables = float(np.mean(timed(lambda: cpa.build_tables(p, dq, cache, tables, workspace=ws), reps, 1)))
    t_attn = timed(lambda: cpa.paged_attention(p, dq, cache, tables, o, workspace=ws), reps, 1)
    t_attn = float(np.mean(t_attn))
    # roofline: the attention kernel's duration inside the timed steps (graph event nodes around it)
    # when available, else its separately timed launches
    t_attn_roof, roof_timing = t_attn, "separate launches (CUDA events, L2 flushed)"
    if att_in_step:
        t_attn_roof = float(np.mean(att_in_step))
        roof_timing = "inside the timed steps (CUDA-graph event nodes around the attention kernel)"
    t_dense = float(np.mean(timed(lambda: cpa.paged_attention(p, dq, cache, None, o, workspace=ws), reps, 1)))
    t_append = float(np.mean(timed(lambda: cpa.append_kv(p, kc, vc, cache), reps, 1)))
    ip = tables.kv_indptr.cpu().numpy()
    ix = tables.kv_indices.cpu().numpy()[: ip[-1]]
    Gx = hq_l // E_exec
    f_sel = attention_flops(ip, ix, C, P, bs, E_exec, d)
    all_ip = np.arange(cfg.batch * Gx + 1) * nkvb
    f_dense = attention_flops(all_ip, np.tile(np.arange(nkvb), cfg.batch * Gx), C, P, bs, E_exec, d)
    density = (ip[-1] - cfg.batch * Gx * (nkvb - P // bs)) / (cfg.batch * Gx * (P // bs))
    # per-stage sparsity from the GPU's own mask bits (one extra build, outside the timed region)
    pm = cpa.make_params(cfg.batch, hq_l, hkv_l, d, bs, C, P, alpha=ALPHA, exec_group_size=args.exec_group,
                         flags=cpa.F_MASK_OUT | (cpa.F_EXACT_SCORES if args.exact_scores else 0) | vflag)
    tm = cpa.alloc_tables(pm, mask=True)
    cpa.build_tables(pm, dq, cache, tm)
    nqb = -(-C // bs)
    sparsity = sparsity_report(tm.mask_bits.cpu().numpy(), nkvb, P // bs, nqb, hq_l, E_exec, E)

    # ---- e2e: the same step through the public API with HOST buffers (pinned), copies timed
    hq_pin = dq.cpu().pin_memory()
    hk_pin, hv_pin = kc.cpu().pin_memory(), vc.cpu().pin_memory()
    ho_pin = torch.empty(o.shape, dtype=o.dtype).pin_memory()
    dq2, kc2, vc2 = torch.empty_like(dq), torch.empty_like(kc), torch.empty_like(vc)

    def e2e_step():
        dq2.copy_(hq_pin, non_blocking=True)
        kc2.copy_(hk_pin, non_blocking=True)
        vc2.copy_(hv_pin, non_blocking=True)
        if peers is not None:
            cpa.chunk_step_peer(p, dq2, cache, tables, peers, kc2, vc2, workspace=ws)
            ho_pin.copy_(o_gathered[:, :, rank * hq_l:(rank + 1) * hq_l], non_blocking=True)
            return
        cpa.chunk_step(p, dq2, cache, tables, o, kc2, vc2, workspace=ws)
        if world > 1:
            allgather_heads(o, o_all)
        ho_pin.copy_(o, non_blocking=True)

    e2e_serial_ms = float(np.mean(timed(e2e_step, args.steps, 1)))
    e2e_ms, e2e_mode = e2e_serial_ms, "serial: H2D, chunk step, D2H in stream order, per step"
    if world == 1:
        # the same public API fed from pinned host buffers as a serving loop would: HostChunkStream
        # overlaps step i+1's H2D and step i-1's D2H with step i's kernels; the timed region spans all
        # K steps (first H2D to last D2H, CUDA events), every copy inside it.
        runner = cpa.HostChunkStream(p, cache, tables, tuple(dq.shape), tuple(kc.shape), workspace=ws,
                                     graphs=not args.no_graph)
        outs = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for _ in range(2)]
        for i in range(max(2, args.warmup)):
            runner.submit(hq_pin, outs[i & 1], hk_pin, hv_pin)
        runner.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(runner.s_in)
        for i in range(args.steps):
            runner.submit(hq_pin, outs[i & 1], hk_pin, hv_pin)
        b.record(runner.s_out)
        runner.synchronize()
        e2e_ms = a.elapsed_time(b) / args.steps
        e2e_mode = ("pipelined (HostChunkStream: H2D of step i+1 and D2H of step i-1 overlap step i), "
                    "K steps timed first H2D to last D2H; each step streams > L2 (268 MB of K pages)")
    h2d = (dq.numel() + kc.numel() + vc.numel()) * 2
    d2h = o.numel() * 2
    e2e_ms, e2e_serial_ms, t_attn, t_dense, t_tables = max_over_ranks([e2e_ms, e2e_serial_ms, t_attn, t_dense, t_tables])

    peak_tf, peak_bw, peak_src = peaks()
    achieved_tf = f_sel / (t_attn_roof * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_attention_summary.json")) as f:
            prof = json.load(f)
        traffic = prof.get(args.config, {}).get("dram_bytes_per_launch")
    except Exception:
        pass

    out = None
    if rank == 0:
        cpu = cpu_oracle_sample(cfg, seed, q, k, v, P, C, budget_s=args.cpu_budget) if world == 1 else None
        out = {
            "metric": METRIC, "value": round(ms, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg.name, "batch": cfg.batch, "context": cfg.context, "chunk": cfg.chunk,
                       "prefix": P, "q_heads": cfg.num_q_heads, "kv_heads": cfg.num_kv_heads, "head_dim": d,
                       "block_size": bs, "alpha": ALPHA, "needle_density": RHO, "exec_group_size": E_exec,
                       "scorer": "exact tile max (SPEC.md:223)" if args.exact_scores else "pooled query (SPEC.md:269)",
                       "parallelism": f"kv-group shard x{world}" + (f" + {collective}" if collective != "none" else ""),
                       "l2": "flushed (512 MiB write) before every timed step", "launch": launch,
                       "v_cache_dtype": "f16" if args.v_f16 else "bf16"},
            "dense_ms_per_chunk": round(t_dense, 4),
            "speedup_vs_dense": round(t_dense / ms, 3),
            "attention_only_speedup": round(t_dense / t_attn, 3),
            "stage_ms": {"append": round(t_append, 4), "estimator+tables": round(t_tables, 4),
                         "attention": round(t_attn, 4)},
            "tabled_prefix_density": round(float(density), 4),
            "sparsity": sparsity,
            "effective_tflops": round(f_dense / (ms * 1e-3) / 1e12, 1),
            "roofline": {"bound": "tensor", "achieved": round(achieved_tf, 1), "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": round(achieved_tf / peak_tf, 4), "traffic": traffic,
                         "kernel": "k_paged_attn", "peak_source": peak_src, "timing": roof_timing,
                         "algorithmic_flops_per_launch": f_sel},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_ms, 4), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "mode": e2e_mode, "serial_value": round(e2e_serial_ms, 4)},
            "clocks": clk.summary(),
            "gpu_launches": launches_per_step * args.steps,
            "paper_context": "2.72x attention speedup at 128K on 2xH200 (TP=2, B=8, chunk 1024; PAPER.md:612, 620)",
        }
        print(json.dumps(out), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------------------ reference arm
def run_reference(args):
    """The oracle as it stands on the host cores (the tier's reference arm)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    seed = seed_of(args.config)
    P, C, L = cfg.chunk_geometry()
    k, v = make_kv(cfg, seed, RHO, kv_heads=range(0, 1))
    q = make_q(cfg, seed, q_heads=range(0, cfg.group_size))
    qf = np.zeros((cfg.batch, C, cfg.num_q_heads, cfg.head_dim), np.float32)
    qf[:, :, :cfg.group_size] = q
    budget = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(cfg, seed, qf, k, v, P, C, budget_s=budget)
        if i >= args.warmup:
            vals.append(r["value"])
    val = float(np.mean(vals))
    out = {"impl": "reference", "metric": METRIC, "value": round(val, 2), "unit": UNIT, "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(val, 2), "higher_is_better": False,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": cfg.name, "batch": cfg.batch, "context": cfg.context, "chunk": cfg.chunk},
           "cpu_baseline": {**r, "value": round(val, 2)},
           "e2e": {"value": round(val, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="llama8b_128k", choices=[c for c in CONFIGS if c != "tiny"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--exact-scores", action="store_true", help="NEXT-1: SPEC's exact tile-max scorer")
    ap.add_argument("--exec-group", type=int, default=0,
                    help="execution-group size E (0 = full KV group; 4 = sub-KV-group union, PAPER.md:498)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-graph", action="store_true", help="launch the step directly instead of a CUDA graph")
    ap.add_argument("--v-bf16", dest="v_f16", action="store_false",
                    help="keep the V pool in bf16 (converted per page inside the attention kernel) instead of the "
                         "default fp16 pool (CPA_F_V_F16: converted once at append; bitwise-identical outputs)")
    ap.add_argument("--collective", default="peer", choices=["peer", "nccl"],
                    help="N>1 head-output all-gather: fused P2P stores in the attention epilogue, or NCCL")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
