"""bench.py's launcher (CPU): `--gpus N` outside torchrun re-launches itself with N ranks under
torch.distributed.run, and a WORLD_SIZE that disagrees with --gpus is refused (the driver's SCALE run
relies on both). CPA_BENCH_LAUNCH_PROBE=1 stops each rank right after a gloo rendezvous + all-reduce."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, **env):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, env=e, cwd=ROOT)


def test_gpus_2_launches_two_ranks():
    r = _run(["--gpus", "2"], CPA_BENCH_LAUNCH_PROBE="1")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d == {"n_gpus": 2, "ranks_seen": 2}


def test_world_size_mismatch_refused():
    r = _run(["--gpus", "2"], WORLD_SIZE="4", RANK="0", CPA_BENCH_LAUNCH_PROBE="1")
    assert r.returncode == 2 and "refusing" in r.stderr


def test_reference_arm_config_matches_gpu_arm_flags():
    """The reference arm echoes the GPU arm's config dict for the same flags (same_config)."""
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    a = argparse.Namespace(config="llama8b_128k", exec_group=0, exact_scores=False, collective="peer",
                           no_graph=False, v_f16=True, rho=0.3, variant="base")
    c1 = bench.bench_config(a, 1)
    assert c1["workload"] == "llama8b_128k" and c1["launch"].startswith("CUDA graph") and c1["v_cache_dtype"] == "f16"
    assert bench.bench_config(a, 8)["parallelism"].startswith("kv-group shard x8 + fused peer-store")
