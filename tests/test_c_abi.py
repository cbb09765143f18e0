"""The C ABI from plain C (tests/c_abi/cpa_c_smoke.c): no Python, torch or ctypes on the call path.
CPU: the program compiles as C99 with -Wall -Werror against include/cpa.h and links against libcpa.so.
GPU: it runs one cpa_chunk_step on seeded synthetic inputs (tiny config and a d=128 / bs=128 case that
takes the cta_group::2 kernel) and checks the tables bit for bit and the outputs within 1e-2 x RMS
against the fp64 oracle (north_star tolerance)."""
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c_abi", "cpa_c_smoke.c")
LIBDIR = os.path.join(ROOT, "paper_2605_16839_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    from paper_2605_16839_b200.build import build
    build()
    cc = shutil.which("gcc") or shutil.which("cc")
    assert cc, "no C compiler"
    exe = str(tmp_path / "cpa_c_smoke")
    cmd = [cc, "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), SRC, "-o", exe, "-L", LIBDIR, "-lcpa",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{LIBDIR}",
           f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


def _bf16_bits(x):
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["tiny", "d128"])
def test_c_program_chunk_step_matches_oracle(tmp_path, case):
    import oracle as O
    from synth.workload import CONFIGS, make_kv, make_q, page_layout, random_qkv, to_pool
    if case == "tiny":
        cfg = CONFIGS["tiny"]
        k, v = make_kv(cfg, 16839)
        q = make_q(cfg, 16839)
        P, C, L = cfg.chunk_geometry()
        bs = cfg.block_size
    else:
        bs, C, P = 128, 200, 384
        q, k, v = random_qkv(1, 8, 2, 128, C, P + C, seed=21)
        L = P + C
    B, _, Hq, d = q.shape
    Hkv = k.shape[1]
    nkvb = -(-L // bs)
    pt, npages = page_layout(B, nkvb, 16839)
    ref = O.chunk_step(q, k, v, P, bs, alpha=0.06)
    out = tmp_path / "data"
    out.mkdir()
    (out / "meta.txt").write_text(f"{B} {Hq} {Hkv} {d} {bs} {C} {P} {npages} {pt.shape[1]} 0.06\n")
    _bf16_bits(q).tofile(out / "q.bin")
    _bf16_bits(to_pool(k, pt, npages, bs)).tofile(out / "k.bin")
    _bf16_bits(to_pool(v, pt, npages, bs)).tofile(out / "v.bin")
    np.ascontiguousarray(pt, dtype=np.int32).tofile(out / "pt.bin")
    np.asarray(ref["indptr"], dtype=np.int32).tofile(out / "ip.bin")
    np.asarray(ref["indices"], dtype=np.int32).tofile(out / "ix.bin")
    np.ascontiguousarray(ref["O"], dtype=np.float64).tofile(out / "o.bin")
    exe = _build(tmp_path)
    r = subprocess.run([exe, str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "c abi ok=1" in r.stdout
