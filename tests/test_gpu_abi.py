"""C ABI behaviour that needs the device: a synchronous validation error leaves every output untouched
(cpa.h conventions), even in cpa_chunk_step, whose first kernel writes the KV pages."""
import numpy as np
import pytest
import torch

import paper_2605_16839_b200 as cpa
from synth.workload import random_qkv
from tests.gpu_helpers import Case, to_dev_bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fault", ["workspace", "capacity", "mask_out", "null_o"])
def test_failed_chunk_step_leaves_outputs_untouched(fault):
    Hq, Hkv, d, bs, C, P = 8, 2, 128, 128, 256, 512
    q, k, v = random_qkv(1, Hq, Hkv, d, C, P + C, seed=3)
    case = Case(q, k, v, P, bs, seed=1)
    p = case.params
    if fault == "mask_out":
        p.flags |= cpa.F_MASK_OUT  # without tables.mask_bits -> CPA_ERR_NULL
    t = cpa.alloc_tables(p)
    t.kv_indptr.fill_(-7)
    t.kv_indices.fill_(-7)
    if fault == "capacity":
        t.kv_indices = t.kv_indices[:-1]
    ws_n = cpa.workspace_bytes(p) - (4096 if fault == "workspace" else 0)
    ws = torch.empty(ws_n, dtype=torch.uint8, device="cuda")
    o = case.out(False).fill_(3.0)
    kc = to_dev_bf16(np.full((1, C, Hkv, d), 0.5, np.float32))  # differs from the pages' chunk contents
    vc = to_dev_bf16(np.full((1, C, Hkv, d), 0.5, np.float32))
    k0, v0 = case.cache.k_pages.clone(), case.cache.v_pages.clone()
    with pytest.raises(cpa.CpaError) as ei:
        cpa.chunk_step(p, case.dq, case.cache, t, None if fault == "null_o" else o, kc, vc, workspace=ws)
    torch.cuda.synchronize()
    expect = {"workspace": "CPA_ERR_WORKSPACE", "capacity": "CPA_ERR_CAPACITY", "mask_out": "CPA_ERR_NULL",
              "null_o": "CPA_ERR_NULL"}[fault]
    assert str(ei.value).startswith(expect), str(ei.value)
    assert torch.equal(case.cache.k_pages, k0) and torch.equal(case.cache.v_pages, v0)
    assert bool((t.kv_indptr == -7).all()) and bool((t.kv_indices == -7).all())
    assert bool((o == 3.0).all())
    assert cpa.last_launch_count() == 0
