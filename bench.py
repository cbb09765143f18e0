#!/usr/bin/env python
"""Benchmark of the CompactAttention chunked-prefill hot path on B200 (BASELINE.json metric).

One step = one whole chunk step through the C ABI (cpa_chunk_step): append the chunk's K/V into
the pages, pooled-query estimator, threshold mask, Q-block + intra-group union, CSR tables and
paged attention over the tabled blocks, for the FINAL chunk of the workload (KV = full context).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama8b_128k] [--impl reference]

Prints ONE JSON line (rank 0). value = attention ms per chunk (lower is better), inputs resident
in HBM, L2 flushed before every timed step (a 512 MiB write), CUDA events on the launch stream,
max over ranks. --gpus N > 1 without a torchrun environment re-launches itself under
`torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL); under torchrun, WORLD_SIZE must
equal --gpus. KV-head groups are sharded over the ranks (one KV group per GPU at N=8) and the per-rank
head outputs are all-gathered each step (strong scaling: one chunk) -- by default inside the attention
kernel (P2P stores into every rank's symmetric-memory buffer over NVLink + a signal barrier,
cpa_chunk_step_peer); --collective nccl times NCCL all_gather_into_tensor instead.

--impl reference runs the tier's reference arm: the fp64 CPU oracle (oracle/, as it stands) on the
host cores, on the same workload and metric; the GPU arm's cpu_baseline is that arm on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
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


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def bench_config(args, world):
    """The `config` object of the JSON line: a function of the command line only, so the GPU arm and
    the reference arm (same flags) print the same dict."""
    cfg = CONFIGS[args.config]
    P, C, L = cfg.chunk_geometry()
    one_dev = os.environ.get("CPA_BENCH_ONE_DEVICE") == "1"
    if world == 1:
        par = "kv-group shard x1"
    elif one_dev:
        par = f"kv-group shard x{world} + gloo all-gather (single-device test mode)"
    elif args.collective == "peer":
        par = f"kv-group shard x{world} + fused peer-store all-gather (NVLink P2P, cpa_chunk_step_peer)"
    else:
        par = f"kv-group shard x{world} + nccl all-gather"
    graph = not args.no_graph and not one_dev and (world == 1 or args.collective == "peer")
    return {"workload": cfg.name, "batch": cfg.batch, "context": cfg.context, "chunk": cfg.chunk,
            "prefix": P, "q_heads": cfg.num_q_heads, "kv_heads": cfg.num_kv_heads, "head_dim": cfg.head_dim,
            "block_size": cfg.block_size, "alpha": ALPHA, "needle_density": args.rho,
            "exec_group_size": args.exec_group or cfg.group_size,
            "scorer": "exact tile max (SPEC.md:223)" if args.exact_scores else "pooled query (SPEC.md:269)",
            "parallelism": par, "l2": "flushed (512 MiB write) before every timed step",
            "launch": "CUDA graph of the chunk step" if graph else "direct",
            "v_cache_dtype": "f16" if args.v_f16 else "bf16",
            **({"workload_variant": args.variant} if args.variant != "base" else {})}


# ------------------------------------------------------------------------------ algorithmic work
def attention_flops(indptr, indices, C, P, bs, E, d):
    """4*d*E*sum over rows r of sum_p |A(p)| (exact causal pairs on the tabled blocks)."""
    L = P + C
    total = 0
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
             "clocks_event_reasons.sw_power_cap,power.draw,power.limit")
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
        num = lambda v: v.replace(".", "", 1).isdigit()
        pw = [float(s[7]) for s in self.samples if len(s) > 7 and num(s[7])]
        pl = [float(s[8]) for s in self.samples if len(s) > 8 and num(s[8])]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_median": statistics.median(pw) if pw else None, "power_w_max": max(pw) if pw else None,
                "power_limit_w": max(pl) if pl else None}


# ------------------------------------------------------------------------------ CPU oracle (reference arm)
# The oracle as it stands, on every host core: one worker process per core (fork: the parent's inputs are
# shared copy-on-write; BLAS limited to one thread per worker). Work unit = one execution group (b, g):
# its estimator + threshold + unions + CSR row, then its attention rows in batches.
_OR = {}


def _or_init():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _or_group_slices(gi):
    d = _OR
    b, g = divmod(gi, d["Gn"])
    kvh = (g * d["E"]) // d["E_kv"]
    q = d["q"][b:b + 1, :, g * d["E"]:(g + 1) * d["E"]]
    return q, d["k"][b:b + 1, kvh:kvh + 1], d["v"][b:b + 1, kvh:kvh + 1]


def _or_tables(gi):
    import oracle as O
    d = _OR
    q, k, _ = _or_group_slices(gi)
    if d["exact"]:
        m = O.block_scores_exact(q, k, d["P"], d["bs"])
    else:
        m = O.block_scores_pooled(q, k, d["P"], d["bs"])
    M = O.threshold_mask(m, ALPHA, d["C"], d["P"], d["bs"])
    return O.tables_from_mask(M, d["E"], d["P"] // d["bs"])


def _or_rows(task):
    import oracle as O
    gi, ip, ix, rows = task
    q, k, v = _or_group_slices(gi)
    O.paged_attention(q, k, v, _OR["P"], _OR["bs"], ip, ix, E=_OR["E"], rows=rows)
    return len(rows)


def _pairs(ix, C, P, bs, L):
    """Causal (query position, key) pairs of one execution group's table (per query head)."""
    pos = P + np.arange(C)
    tot = 0
    for j in ix:
        lo, hi = int(j) * bs, min(int(j) * bs + bs, L)
        tot += int(np.clip(pos - lo + 1, 0, hi - lo).sum())
    return tot


def oracle_chunk(args, rows_per_group=None, log=None, one_group=None):
    """Time the oracle on the final chunk of args.config: every group's estimator + tables, then the
    attention rows (all of them, or `rows_per_group` evenly spaced query positions x all heads of each
    group, or -- one_group = gi -- every row of execution group gi only, scaled to the chunk by the exact
    causal-pair counts of all groups' tables). Returns (ms/chunk, timed wall ms, description)."""
    import multiprocessing as mp
    cfg = CONFIGS[args.config]
    seed = seed_of(args.config)
    P, C, L = cfg.chunk_geometry()
    E_kv = cfg.group_size
    E = args.exec_group or E_kv
    Gn = cfg.num_q_heads // E
    t_gen = time.perf_counter()
    k, v = make_kv(cfg, seed, args.rho, variant=args.variant)
    q = make_q(cfg, seed, variant=args.variant)
    _OR.update(q=q, k=k, v=v, P=P, C=C, bs=cfg.block_size, E=E, E_kv=E_kv, Gn=Gn, exact=args.exact_scores)
    cores = host_cores()
    groups = cfg.batch * Gn
    if rows_per_group is None or rows_per_group >= C * E:
        ps = list(range(C))
    else:
        ps = sorted(set(np.linspace(0, C - 1, max(1, rows_per_group // E)).round().astype(int).tolist()))
    rows_g = [(0, int(p), hl) for p in ps for hl in range(E)]
    n_total = groups * C * E
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_or_init) as pool:
        pool.map(int, range(cores))  # workers up before the clock starts
        if log:
            log(f"[oracle] inputs generated in {time.perf_counter() - t_gen:.1f} s; {cores} worker processes")
        t0 = time.perf_counter()
        tabs = pool.map(_or_tables, range(groups), chunksize=1)
        t1 = time.perf_counter()
        att_groups = range(groups) if one_group is None else [one_group % groups]
        per = max(1, min(64, len(rows_g) // max(1, (2 * cores) // len(att_groups) + 1)))
        tasks = [(gi, tabs[gi][0], tabs[gi][1], rows_g[s:s + per]) for gi in att_groups
                 for s in range(0, len(rows_g), per)]
        done = sum(pool.imap_unordered(_or_rows, tasks, chunksize=1))
        t2 = time.perf_counter()
    n_timed = done
    t_est, t_att = (t1 - t0) * 1e3, (t2 - t1) * 1e3
    if one_group is not None:
        gi = one_group % groups
        pairs = [_pairs(tabs[g][1], C, P, cfg.block_size, L) for g in range(groups)]
        ratio = sum(pairs) / pairs[gi]
        ms = t_est + t_att * ratio
        desc = (f"estimator + tables of all {groups} execution groups (complete, {t_est:.0f} ms) + attention for "
                f"every row of execution group {gi} ({n_timed} (b, p, h) rows, {t_att:.0f} ms), scaled to the chunk "
                f"by the exact causal-pair count of all groups' tables (x{ratio:.3f}; groups differ only in "
                f"needle placement); fp64 numpy oracle, {cores} worker processes")
    else:
        ms = t_est + t_att * (n_total / n_timed)
    if one_group is not None:
        pass
    elif n_timed == n_total:
        desc = (f"whole {cfg.name} final chunk: estimator + tables of all {groups} execution groups and "
                f"attention for all {n_total} (b, p, h) query rows, fp64 numpy oracle, {cores} worker processes")
    else:
        desc = (f"estimator + tables of all {groups} execution groups (complete, {t_est:.0f} ms) + attention "
                f"for {n_timed} of {n_total} (b, p, h) query rows ({len(ps)} evenly spaced query positions x "
                f"all heads of every group, {t_att:.0f} ms), extrapolated linearly in rows; fp64 numpy oracle, "
                f"{cores} worker processes")
    return ms, (t2 - t0) * 1e3, desc, cores


def run_reference(args):
    """The tier's reference arm: the fp64 oracle as it stands on the host cores, same workload, metric
    and config as the GPU arm. Rank 0 only (other torchrun ranks exit without work). One step = the
    whole final chunk (no extrapolation) unless --oracle-rows-per-group samples it (cpu_baseline leg)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    log = lambda m: print(m, file=sys.stderr, flush=True)
    vals, walls = [], []
    whole = args.oracle_rows_per_group is None and args.ref_whole_chunk
    per_group = args.oracle_rows_per_group is None and not args.ref_whole_chunk
    n_steps = 1 if args.oracle_rows_per_group is None else max(1, args.steps)
    for st in range(n_steps):
        ms, wall, desc, cores = oracle_chunk(args, args.oracle_rows_per_group, log,
                                             one_group=st if per_group else None)
        vals.append(ms)
        walls.append(wall)
    val = float(np.mean(vals))
    out = {"impl": "reference", "metric": METRIC, "value": round(val, 2), "unit": UNIT, "n_gpus": args.gpus,
           "steps": n_steps, "warmup": 0, "ms_per_step": round(val, 2), "higher_is_better": False,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": bench_config(args, args.gpus),
           "cpu_baseline": {"value": round(val, 2), "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": desc, "timed_wall_ms": round(float(np.mean(walls)), 1)},
           "e2e": {"value": round(val, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "note": ("steps = whole chunks actually timed (one chunk of the oracle takes minutes on the host "
                    "cores, so --steps/--warmup are not repeated); warm-up = input generation + worker start-up"
                    if whole else
                    ("one step = the whole estimator + every attention row of one execution group, scaled to the "
                     "chunk by exact pair counts (--ref-whole-chunk times the whole chunk: r02a measured 360 s "
                     "for 128K on 16 cores); --steps/--warmup are not repeated"
                     if per_group else "bounded sample per step, extrapolated to ms/chunk (see cpu_baseline.sample)"))}
    print(json.dumps(out), flush=True)


def cpu_baseline_leg(args):
    """The oracle on a bounded sample of the same chunk (the reference arm with
    --oracle-rows-per-group), run in a child process: it forks one worker per core, which must not
    happen in a process that holds a CUDA context."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", args.config,
           "--oracle-rows-per-group", str(args.cpu_rows_per_group), "--steps", "1", "--gpus", str(args.gpus),
           "--collective", args.collective]
    if args.exact_scores:
        cmd.append("--exact-scores")
    if args.exec_group:
        cmd += ["--exec-group", str(args.exec_group)]
    if not args.v_f16:
        cmd.append("--v-bf16")
    if args.no_graph:
        cmd.append("--no-graph")
    cmd += ["--rho", str(args.rho), "--variant", args.variant]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
        return json.loads(line)["cpu_baseline"]
    except Exception as ex:  # noqa: BLE001 -- reported, never fatal for the GPU arm
        return {"value": None, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
                "sample": f"failed: {type(ex).__name__}: {ex}"[:300]}


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
    # CPA_BENCH_PEER_W1=1 (test only, under torchrun --nproc-per-node 1): a 1-rank NCCL group so the
    # fused peer path runs through real symmetric memory on a single-GPU box.
    force_peer = os.environ.get("CPA_BENCH_PEER_W1") == "1" and world == 1
    if world > 1 or force_peer:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()  # eager communicator init (NCCL_DEBUG=INFO logs it on stderr)
        print(f"[bench] rank {rank}/{world}: process group up ({dist.get_backend()}), cuda:{local}",
              file=sys.stderr, flush=True)

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
    from paper_2605_16839_b200.shard import allgather_heads, head_shard, heads_view
    kvh, qh = head_shard(cfg.num_q_heads, cfg.num_kv_heads, world, rank)
    hkv_l, hq_l = len(kvh), len(qh)
    k, v = make_kv(cfg, seed, args.rho, kv_heads=kvh, variant=args.variant)
    q = make_q(cfg, seed, q_heads=qh, variant=args.variant)
    nkvb = -(-L // bs)
    pt, npages = page_layout(cfg.batch, nkvb, seed)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    kpool = dev(to_pool(k, pt, npages, bs))
    vpool_bf16 = dev(to_pool(v, pt, npages, bs))
    vpool = vpool_bf16.half() if args.v_f16 else vpool_bf16  # CPA_F_V_F16: fp16 pool (exact for these values)
    ptab = torch.from_numpy(pt).cuda()
    cache = cpa.PagedKVCache(kpool, vpool, ptab)
    dq = dev(q)
    kc = dev(k[:, :, P:].transpose(0, 2, 1, 3))  # the chunk's own K/V [B, C, Hkv, d] (re-appended)
    vc = dev(v[:, :, P:].transpose(0, 2, 1, 3))
    del k, v
    E_exec = args.exec_group or E
    vflag = cpa.F_V_F16 if args.v_f16 else 0
    if os.environ.get("CPA_BENCH_NO_PDL") == "1":  # A/B only: launch the chain without PDL
        vflag |= cpa.F_NO_PDL
    vflag |= int(os.environ.get("CPA_BENCH_EXTRA_FLAGS", "0"))  # A/B only (e.g. CPA_F_ATTN_V1)
    sflag = cpa.F_EXACT_SCORES if args.exact_scores else 0
    p = cpa.make_params(cfg.batch, hq_l, hkv_l, d, bs, C, P, alpha=ALPHA, exec_group_size=args.exec_group,
                        flags=sflag | vflag)
    tables = cpa.alloc_tables(p)
    ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
    o = torch.empty(cfg.batch, C, hq_l, d, dtype=torch.bfloat16, device="cuda")
    o_all = torch.empty(world, cfg.batch, C, hq_l, d, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    config = bench_config(args, world)
    # N > 1: the head-output all-gather is fused into the attention epilogue (P2P stores into every
    # rank's symmetric-memory buffer + a signal barrier, cpa_chunk_step_peer); NCCL all-gather after a
    # local step is the baseline (--collective nccl) and the fallback if symmetric memory is unavailable.
    peers = None
    peer_check = None
    full_shape = (cfg.batch, C, cfg.num_q_heads, d)
    if (world > 1 or force_peer) and not one_dev and args.collective == "peer":
        try:
            peers, o_gathered = peer_setup(torch, dist, cpa, full_shape, world, rank)
        except Exception as ex:  # noqa: BLE001 -- reported in the JSON line
            config["parallelism"] = (f"kv-group shard x{world} + nccl all-gather (fallback: symmetric memory "
                                     f"unavailable: {type(ex).__name__}: {ex})")[:240]
            config["launch"] = "direct"
    if peers is not None:
        # validate the fused path once against the local step + NCCL all-gather before timing it: a rank
        # whose gathered buffer differs, or a barrier timeout, switches every rank to the NCCL baseline
        # (recorded in `parallelism`) instead of losing the run
        why = ""
        try:
            cpa.chunk_step_peer(p, dq, cache, tables, peers, kc, vc, workspace=ws)
            torch.cuda.synchronize()
            st_ = int(peers.dev_status.item())
            if st_ != 0:
                why = f"peer barrier timed out waiting for rank {st_ - 1}"
        except Exception as ex:  # noqa: BLE001 -- reported in the JSON line
            why = f"{type(ex).__name__}: {ex}"
        try:
            cpa.chunk_step(p, dq, cache, tables, o, kc, vc, workspace=ws)
        except Exception as ex:  # noqa: BLE001
            why = why or f"{type(ex).__name__}: {ex}"
        allgather_heads(o, o_all)  # every rank, whatever happened above (same collective sequence)
        torch.cuda.synchronize()
        if not why and not torch.equal(heads_view(o_all), o_gathered):
            why = "fused all-gather output differs from the NCCL all-gather"
        ok = torch.tensor([0 if why else 1], dtype=torch.int32, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            print(f"[bench] rank {rank}: fused peer path failed validation ({why or 'another rank'}); "
                  f"using NCCL all-gather", file=sys.stderr, flush=True)
            peers = None
            config["parallelism"] = (f"kv-group shard x{world} + nccl all-gather (fallback: fused peer path "
                                     f"failed validation: {why or 'on another rank'})")[:240]
            config["launch"] = "direct"
        peer_check = "fused all-gather bit-equal to local step + NCCL all-gather" if peers is not None else why
    use_graph = config["launch"].startswith("CUDA graph")

    def step():
        if peers is not None:
            cpa.chunk_step_peer(p, dq, cache, tables, peers, kc, vc, workspace=ws)
            return
        cpa.chunk_step(p, dq, cache, tables, o, kc, vc, workspace=ws)
        if world > 1:
            allgather_heads(o, o_all)

    # The timed step is one replay of a CUDA graph of the whole chunk step (append, estimator, tables,
    # attention [, fused all-gather + barrier]): the C ABI is stream-ordered, never allocates or syncs,
    # so it captures as is; replays drop the per-kernel launch gaps. Event nodes captured around the
    # attention kernel time it inside every timed step (roofline). NCCL / gloo all-gather modes run directly.
    step()  # one direct step: kernels per step for gpu_launches
    launches_per_step = cpa.last_launch_count()
    att_ev = None

    def capture(p_, cache_):
        ev = (torch.cuda.Event(enable_timing=True, external=True),
              torch.cuda.Event(enable_timing=True, external=True))
        g = torch.cuda.CUDAGraph()
        # thread_local: the NCCL watchdog thread may query events while this thread captures
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            # == cpa_chunk_step(_peer): prepare (append + estimator + tables) + attention (same workspace,
            # same stream), split so that event nodes bracket the attention kernel
            cpa.prepare_chunk(p_, dq, cache_, tables, kc, vc, workspace=ws)
            ev[0].record()
            if peers is not None:
                cpa.paged_attention_peer(p_, dq, cache_, tables, peers, workspace=ws)
            else:
                cpa.paged_attention(p_, dq, cache_, tables, o, workspace=ws)
            ev[1].record()
        return g, ev

    if use_graph:
        step()
        torch.cuda.synchronize()
        graph, att_ev = capture(p, cache)
        torch.cuda.synchronize()
        step = graph.replay

    def timed(fn, iters, warm, inner=None, ev=None, flush_l2=True):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            if flush_l2:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            if inner is not None:
                inner.append(ev[0].elapsed_time(ev[1]))
        return ts

    # ---- headline: W warm-up steps, K timed steps, barrier + sync on both sides
    att_in_step = []
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        ts = timed(step, args.steps, 0, att_in_step if att_ev is not None else None, att_ev)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = max_over_ranks([float(np.mean(ts))])[0]
    if peers is not None and int(peers.dev_status.item()) != 0:
        raise RuntimeError(f"rank {rank}: peer barrier timed out waiting for rank {int(peers.dev_status.item()) - 1}")

    # ---- stage breakdown and the dense baseline (same kernels, tables = all blocks), rank-local
    reps = max(3, min(args.steps, 10))
    t_tables = float(np.mean(timed(lambda: cpa.build_tables(p, dq, cache, tables, workspace=ws), reps, 1)))
    t_attn = float(np.mean(timed(lambda: cpa.paged_attention(p, dq, cache, tables, o, workspace=ws), reps, 1)))
    t_attn_roof, roof_timing = t_attn, "separate launches (CUDA events, L2 flushed)"
    if att_in_step:
        t_attn_roof = float(np.mean(att_in_step))
        roof_timing = "inside the timed steps (CUDA-graph event nodes around the attention kernel)"
    # dense baseline timed exactly like the headline step (W warm-ups, then K reps, L2 flushed before
    # each); and, for context, interleaved (step, dense) pairs: the chip is power-capped, so a step
    # right after a 6.8 ms dense kernel runs hotter / slower than in a run of steps
    dense_fn = lambda: cpa.paged_attention(p, dq, cache, None, o, workspace=ws)
    t_dense = float(np.mean(timed(dense_fn, args.steps, args.warmup)))
    t_dense_l, t_step_l = [], []
    for _ in range(reps):
        t_step_l += timed(step, 1, 0)
        t_dense_l += timed(dense_fn, 1, 0)
    t_dense_i = float(np.median(t_dense_l))
    t_step_pair = float(np.median(t_step_l))
    t_append = float(np.mean(timed(lambda: cpa.append_kv(p, kc, vc, cache), reps, 1)))
    # SURVEY §8(d) protocol extras: the timed steps' spread, and the step with a warm L2 (no flush)
    t_warm = float(np.median(timed(step, args.steps, 1, flush_l2=False)))
    step_stats = {"min": round(float(np.min(ts)), 4), "median": round(float(np.median(ts)), 4),
                  "p90": round(float(np.percentile(ts, 90)), 4), "warm_l2_median": round(t_warm, 4),
                  "note": "rank 0's K timed steps (L2 flushed before each); warm_l2: K steps without the flush"}
    ip = tables.kv_indptr.cpu().numpy()
    ix = tables.kv_indices.cpu().numpy()[: ip[-1]]
    Gx = hq_l // E_exec
    f_sel = attention_flops(ip, ix, C, P, bs, E_exec, d)
    all_ip = np.arange(cfg.batch * Gx + 1) * nkvb
    f_dense = attention_flops(all_ip, np.tile(np.arange(nkvb), cfg.batch * Gx), C, P, bs, E_exec, d)
    density = (ip[-1] - cfg.batch * Gx * (nkvb - P // bs)) / (cfg.batch * Gx * (P // bs))
    # per-stage sparsity from the GPU's own mask bits (one extra build, outside the timed region)
    pm = cpa.make_params(cfg.batch, hq_l, hkv_l, d, bs, C, P, alpha=ALPHA, exec_group_size=args.exec_group,
                         flags=cpa.F_MASK_OUT | sflag | vflag)
    tm = cpa.alloc_tables(pm, mask=True)
    cpa.build_tables(pm, dq, cache, tm)
    nqb = -(-C // bs)
    sparsity = sparsity_report(tm.mask_bits.cpu().numpy(), nkvb, P // bs, nqb, hq_l, E_exec, E)

    # ---- the same step with the other V pool dtype (bf16 pool: V converted per page in the kernel)
    other_pool = None
    if use_graph and peers is None:
        p_o = cpa.make_params(cfg.batch, hq_l, hkv_l, d, bs, C, P, alpha=ALPHA, exec_group_size=args.exec_group,
                              flags=sflag | (0 if args.v_f16 else cpa.F_V_F16))
        cache_o = cpa.PagedKVCache(kpool, vpool_bf16 if args.v_f16 else vpool_bf16.half(), ptab)
        cpa.chunk_step(p_o, dq, cache_o, tables, o, kc, vc, workspace=ws)
        torch.cuda.synchronize()
        g_o, _ = capture(p_o, cache_o)
        t_o = float(np.mean(timed(g_o.replay, args.steps, 2)))
        other_pool = {"v_cache_dtype": "bf16" if args.v_f16 else "f16", "ms_per_chunk": round(t_o, 4)}
        del g_o, cache_o
        cpa.chunk_step(p, dq, cache, tables, o, kc, vc, workspace=ws)  # restore this arm's pool contents

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
    if world == 1 or peers is not None:
        # the same public API fed from pinned host buffers as a serving loop would: HostChunkStream
        # overlaps step i+1's H2D and step i-1's D2H with step i's kernels; the timed region spans all
        # K steps (first H2D to last D2H, CUDA events), every copy inside it. N > 1: one symmetric-memory
        # gathered buffer per staging slot (three slots, see HostChunkStream).
        hp, hg = None, None
        if peers is not None:
            hp, hg = [peers], [o_gathered]
            for _ in range(2):
                pr, gb = peer_setup(torch, dist, cpa, full_shape, world, rank)
                hp.append(pr)
                hg.append(gb)
        runner = cpa.HostChunkStream(p, cache, tables, tuple(dq.shape), tuple(kc.shape), workspace=ws,
                                     graphs=use_graph, peers=hp, gathered=hg, rank=rank)
        outs = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for _ in range(runner.n)]
        for i in range(max(runner.n, args.warmup)):
            runner.submit(hq_pin, outs[i % runner.n], hk_pin, hv_pin)
        runner.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(runner.s_in)
        for i in range(args.steps):
            runner.submit(hq_pin, outs[i % runner.n], hk_pin, hv_pin)
        b.record(runner.s_out)
        runner.synchronize()
        e2e_ms = a.elapsed_time(b) / args.steps
        e2e_mode = ("pipelined (HostChunkStream: H2D of step i+1 and D2H of step i-1 overlap step i), "
                    "K steps timed first H2D to last D2H; each step streams > L2 (the K pages)")
    h2d = (dq.numel() + kc.numel() + vc.numel()) * 2
    d2h = o.numel() * 2
    e2e_ms, e2e_serial_ms, t_attn, t_attn_roof, t_dense, t_tables, t_append, t_step_pair, t_dense_i = max_over_ranks(
        [e2e_ms, e2e_serial_ms, t_attn, t_attn_roof, t_dense, t_tables, t_append, t_step_pair, t_dense_i])
    # algorithmic FLOPs of the whole job's attention launches (sum over ranks) / the slowest rank's time
    if world > 1:
        tf = torch.tensor([float(f_sel), float(f_dense)], dtype=torch.float64, device="cpu" if one_dev else "cuda")
        dist.all_reduce(tf)
        f_sel, f_dense = int(tf[0].item()), int(tf[1].item())

    peak_tf, peak_bw, peak_src = peaks()
    achieved_tf = f_sel / (t_attn_roof * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_attention_summary.json")) as f:
            prof = json.load(f)
        traffic = prof.get(args.config, {}).get("dram_bytes_per_launch")
    except Exception:
        pass

    cpu = cpu_baseline_leg(args) if rank == 0 and not args.no_cpu else None
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(ms, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": config,
            "dense_ms_per_chunk": round(t_dense, 4),
            "speedup_vs_dense": round(t_dense / ms, 3),
            "speedup_timing": (f"dense timed like the step ({args.warmup} warm-ups + {args.steps} reps, L2 flushed); "
                               f"interleaved (step, dense) pairs, median of {reps}: {t_step_pair:.4f} vs "
                               f"{t_dense_i:.4f} ms = {t_dense_i / t_step_pair:.3f}x"),
            "attention_only_speedup": round(t_dense / t_attn, 3),
            "step_ms_stats": step_stats,
            "stage_ms": {"append": round(t_append, 4), "estimator+tables": round(t_tables, 4),
                         "attention": round(t_attn, 4)},
            "other_v_pool": other_pool,
            "tabled_prefix_density": round(float(density), 4),
            "sparsity": sparsity,
            "effective_tflops": round(f_dense / (ms * 1e-3) / 1e12, 1),
            "roofline": {"bound": "tensor", "achieved": round(achieved_tf, 1), "peak": peak_tf * world,
                         "unit": "TFLOP/s", "frac": round(achieved_tf / (peak_tf * world), 4), "traffic": traffic,
                         "kernel": "k_paged_attn_2cta", "peak_source": peak_src + (f" x {world} GPUs" if world > 1 else ""),
                         "timing": roof_timing, "algorithmic_flops_per_launch": f_sel},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_ms, 4), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "mode": e2e_mode, "serial_value": round(e2e_serial_ms, 4),
                    "bytes_note": "per rank" if world > 1 else "whole job"},
            "clocks": clk.summary(),
            "gpu_launches": launches_per_step * args.steps,
            **({"peer_check": peer_check} if peer_check is not None else {}),
            "paper_context": "2.72x attention speedup at 128K on 2xH200 (TP=2, B=8, chunk 1024; PAPER.md:612, 620)",
        }
        print(json.dumps(out), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------------------ launcher
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run, one rank per GPU
    (the driver's own invocation is torchrun; both end up here with WORLD_SIZE == N)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")           # communicator init lines (nRanks) for the record
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # keep stdout = the JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


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
    ap.add_argument("--cpu-rows-per-group", type=int, default=256,
                    help="cpu_baseline leg: oracle attention rows timed per execution group (extrapolated)")
    ap.add_argument("--oracle-rows-per-group", type=int, default=None,
                    help="reference arm: sample this many rows per group instead of the whole chunk")
    ap.add_argument("--no-graph", action="store_true", help="launch the step directly instead of a CUDA graph")
    ap.add_argument("--v-bf16", dest="v_f16", action="store_false",
                    help="keep the V pool in bf16 (converted per page inside the attention kernel) instead of the "
                         "default fp16 pool (CPA_F_V_F16: converted once at append; bitwise-identical outputs)")
    ap.add_argument("--collective", default="peer", choices=["peer", "nccl"],
                    help="N>1 head-output all-gather: fused P2P stores in the attention epilogue, or NCCL")
    ap.add_argument("--rho", type=float, default=RHO, help="needle density of the planted workload (NEXT-4 sweep)")
    ap.add_argument("--variant", default="base", choices=["base", "qdiverse"],
                    help="workload variant (synth/workload.py; qdiverse: union density grows with chunk size)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (sweeps)")
    ap.add_argument("--ref-whole-chunk", action="store_true",
                    help="reference arm: time the oracle on the whole chunk (minutes) instead of one execution group")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return 0
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        return launch_ranks(args)
    if ws is not None and int(ws) != args.gpus:
        print(f"[bench] refusing to run: WORLD_SIZE={ws} but --gpus {args.gpus}", file=sys.stderr, flush=True)
        return 2
    if os.environ.get("CPA_BENCH_LAUNCH_PROBE") == "1":  # test only (CPU): the launcher's rank wiring
        import torch
        import torch.distributed as dist
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if world > 1:
            dist.init_process_group("gloo")
        t = torch.ones(1)
        if world > 1:
            dist.all_reduce(t)
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"n_gpus": world, "ranks_seen": int(t.item())}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return 0
    run_gpu(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
