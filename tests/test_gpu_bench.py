"""bench.py end to end on the GPU (the driver's invocation, small config): one JSON line with every
key of the contract, positive timings, the CUDA-graph launch path, and the attention roofline timed
inside the timed steps."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "llama8b_32k", "--steps", "3",
                        "--warmup", "3", "--cpu-budget", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert key in d, key
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["higher_is_better"] is False
    assert d["config"]["workload"] == "llama8b_32k" and d["config"]["launch"].startswith("CUDA graph")
    roof = d["roofline"]
    assert roof["bound"] == "tensor" and 0 < roof["frac"] < 1.2 and roof["timing"].startswith("inside the timed")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 3 * 3  # >= 3 libcpa kernels per step
    assert d["speedup_vs_dense"] > 1.0
