"""compute-sanitizer memcheck over small chunk steps of every kernel family (tools/sanitize_case.py:
1-CTA and 2-CTA attention, fp16 V pool, persistent stream-K grid, exact scorer, MASK_IN tables):
no out-of-bounds or misaligned access, no leaked error. (racecheck / synccheck findings are analysed
in DESIGN.md §11: tcgen05.alloc's shared-memory write and mbarrier phases that are waited lazily.)"""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_memcheck_clean():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    assert os.path.exists(exe), "compute-sanitizer not found"
    r = subprocess.run([exe, "--tool", "memcheck", "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_case.py")], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out and "sanitize cases ok" in out, out[-3000:]
