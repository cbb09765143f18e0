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


def _peer(world, rank, outs=16, sigs=16, epoch=1, stride=0):
    o = (ctypes.c_void_p * max(world, 1))(*([outs] * max(world, 1)))
    s = (ctypes.c_void_p * max(world, 1))(*([sigs] * max(world, 1)))
    return cpa._PeerOut(world, rank, o if outs is not None else None, stride, s if sigs is not None else None,
                        epoch, 0, None), (o, s)


@pytest.mark.parametrize("world,rank,kw,status", [
    (0, 0, {}, 2), (9, 0, {}, 2), (2, 2, {}, 2), (2, -1, {}, 2),
    (2, 0, dict(sigs=None), 1), (2, 0, dict(outs=None), 1), (2, 0, dict(sigs=0), 1), (2, 0, dict(sigs=18), 4),
    (2, 0, dict(outs=24), 4), (2, 0, dict(stride=100), 2),
])
def test_peer_validation(L, world, rank, kw, status):
    """cpa_chunk_step_peer validates the peer description before touching the device (cpa.h)."""
    p = _p(num_q_heads=16, num_kv_heads=4)  # one rank's shard of the LLaMA shape at W=2
    pr, keep = _peer(world, rank, **kw)
    c = cpa._Cache(16, 16, 0, 0, 16, 2048, 10)
    t = cpa._Tables(16, 16, 1 << 20, None, None, None, None)
    r = L.cpa_chunk_step_peer(ctypes.byref(p), 16, None, None, ctypes.byref(c), ctypes.byref(t), ctypes.byref(pr),
                              16, 1 << 30, None)
    assert r == status, L.cpa_last_error()


@pytest.mark.parametrize("world,rank,kw,status", [
    (0, 0, {}, 2), (2, 2, {}, 2), (2, 0, dict(sigs=None), 1), (2, 0, dict(outs=24), 4), (2, 0, dict(stride=100), 2),
])
def test_attention_peer_validation(L, world, rank, kw, status):
    """cpa_paged_attention_peer validates the peer description before touching the device (cpa.h)."""
    p = _p(num_q_heads=16, num_kv_heads=4)
    pr, keep = _peer(world, rank, **kw)
    c = cpa._Cache(16, 16, 0, 0, 16, 2048, 10)
    r = L.cpa_paged_attention_peer(ctypes.byref(p), 16, ctypes.byref(c), None, ctypes.byref(pr), 16, 1 << 30, None)
    assert r == status, L.cpa_last_error()


def test_paged_kv_cache_num_pages():
    """PagedKVCache: num_pages is shape[0] only for the default [pages, Hkv, bs, d] pool; explicit strides
    (e.g. the per-sequence [B, Hkv, L, d] layout) need it given; the V dtype must match CPA_F_V_F16."""
    import torch
    kp = torch.zeros(4, 2, 16, 64, dtype=torch.bfloat16)
    pt = torch.zeros(1, 4, dtype=torch.int32)
    assert cpa.PagedKVCache(kp, kp, pt)._c().num_pages == 4
    with pytest.raises(ValueError):
        cpa.PagedKVCache(kp, kp, pt, page_stride=16 * 64, head_stride=64 * 64)._c()
    assert cpa.PagedKVCache(kp, kp, pt, page_stride=16 * 64, head_stride=64 * 64, num_pages=4)._c().num_pages == 4
    p = cpa.make_params(1, 4, 2, 64, 16, 16, 48, flags=cpa.F_V_F16)
    with pytest.raises(ValueError):
        cpa.PagedKVCache(kp, kp, pt)._check_v(p)
    cpa.PagedKVCache(kp, kp.half(), pt)._check_v(p)
