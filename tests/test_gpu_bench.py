"""bench.py end to end on the GPU (the driver's invocation, small config): one JSON line with every
key of the contract, positive timings, the CUDA-graph launch path, and the attention roofline timed
inside the timed steps; and the N>1 path (two ranks on one GPU, gloo) through the launcher."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, **env):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_json_line():
    d = _bench(["--config", "llama8b_32k", "--steps", "3", "--warmup", "3", "--cpu-rows-per-group", "32"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert key in d, key
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["higher_is_better"] is False
    assert d["config"]["workload"] == "llama8b_32k" and d["config"]["launch"].startswith("CUDA graph")
    roof = d["roofline"]
    assert roof["bound"] == "tensor" and 0 < roof["frac"] < 1.2 and roof["timing"].startswith("inside the timed")
    cpu = d["cpu_baseline"]
    assert cpu["kind"] == "oracle" and cpu["value"] > 0 and cpu["cores"] == len(os.sched_getaffinity(0))
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["e2e"]["mode"].startswith("pipelined")
    assert d["gpu_launches"] >= 3 * 3  # >= 3 libcpa kernels per step
    assert d["speedup_vs_dense"] > 1.0
    assert d["other_v_pool"]["v_cache_dtype"] == "bf16" and d["other_v_pool"]["ms_per_chunk"] > 0


def test_bench_two_ranks_one_device():
    """--gpus 2 without torchrun: the launcher starts two ranks (here both on cuda:0 over gloo, the
    single-GPU stand-in for NCCL); KV groups are sharded, outputs all-gathered, times max-reduced."""
    d = _bench(["--gpus", "2", "--config", "llama8b_32k", "--steps", "2", "--warmup", "3", "--cpu-rows-per-group", "16"],
               CPA_BENCH_ONE_DEVICE="1")
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"].startswith("kv-group shard x2")
    assert d["roofline"]["frac"] > 0 and d["cpu_baseline"]["value"] > 0


def test_bench_fused_peer_path_validated():
    """The fused peer all-gather path of an N>1 run, exercised on one GPU with a 1-rank NCCL group
    (CPA_BENCH_PEER_W1 under torchrun): torch symmetric memory, cpa_chunk_step_peer, the pre-timing
    check against the local step + NCCL all-gather, and the CUDA-graph-replayed timed step."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e["CPA_BENCH_PEER_W1"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "1", "--config",
           "llama8b_32k", "--steps", "2", "--warmup", "3", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert d["peer_check"].startswith("fused all-gather bit-equal"), d.get("peer_check")
    assert d["config"]["launch"].startswith("CUDA graph") and d["value"] > 0
