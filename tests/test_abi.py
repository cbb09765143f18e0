"""CPU-side checks of the C ABI: libcpa.so loads, exports every symbol include/cpa.h declares,
and its host-side validation / workspace logic behaves as the header documents (no kernel runs)."""
import ctypes
import os
import re

import pytest

import paper_2605_16839_b200 as cpa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "cpa.h")).read()
    return sorted(set(re.findall(r"CPA_API\s+[\w\s\*]+?\b(cpa_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2605_16839_b200.build import build
    build()
    return cpa.lib()


def test_exports_every_declared_symbol(L):
    declared = _declared_symbols()
    assert len(declared) >= 9
    assert sorted(cpa.EXPORTED_SYMBOLS) == declared
    for name in declared:
        assert hasattr(L, name), name


def test_version_and_status_strings(L):
    assert L.cpa_version() == 1
    for i, name in enumerate(cpa.STATUS):
        assert L.cpa_status_string(i).decode() == name


def _p(**kw):
    base = dict(batch=1, num_q_heads=32, num_kv_heads=8, head_dim=128, block_size=128, chunk_len=4096,
                prefix_len=126976, alpha=0.06)
    base.update(kw)
    return cpa.make_params(**base)


def test_workspace_bytes_host_only(L):
    ws = cpa.workspace_bytes(_p())
    # qbar hi/lo 2*8*128*128*2 + scores 8*1024*128*4 + row max + G words
    assert ws >= 2 * 8 * 128 * 128 * 2 + 8 * 1024 * 128 * 4
    assert cpa.workspace_bytes(_p(alpha=0.0)) == 0  # invalid params -> 0


@pytest.mark.parametrize("kw,status", [
    (dict(alpha=0.0), 5), (dict(alpha=1.5), 5), (dict(num_q_heads=30), 2), (dict(exec_group_size=3), 2),
    (dict(head_dim=96), 3), (dict(block_size=48), 3), (dict(prefix_len=100), 4), (dict(chunk_len=0), 2),
])
def test_validation_errors(L, kw, status):
    p = _p(**kw)
    c = cpa._Cache(16, 16, 0, 0, 16, 2048, 10)
    t = cpa._Tables(16, 16, 1 << 20, None, None, None, None)
    r = L.cpa_build_tables(ctypes.byref(p), 16, ctypes.byref(c), ctypes.byref(t), 16, 1 << 30, None)
    assert r == status, L.cpa_last_error()
    assert L.cpa_last_error().decode()


def test_null_cache_rejected(L):
    p = _p()
    r = L.cpa_paged_attention(ctypes.byref(p), 16, None, None, 16, None, 0, None)
    assert r == 1


def test_capacity_and_geometry(L):
    p = _p()
    nqb, nkvb, pb, Gn, nwords, Rpad = cpa.geometry(p)
    assert (nqb, nkvb, pb, Gn, nwords, Rpad) == (32, 1024, 992, 8, 32, 128)
