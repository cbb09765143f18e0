"""GPU parity of the block-sparse executor (NEXT-3 execution ablation)
and of the q-uniform table expansion, through the C ABI, against the fp64 oracle.

Bars: expansion bit-exact (integer work); outputs max|delta| <= 1e-2 x RMS (fp32 output mode).
"""
import dataclasses

import numpy as np
import pytest
import torch

import oracle as O
import paper_2605_16839_b200 as cpa
from synth.workload import CONFIGS, make_kv, make_q, random_block_mask, random_qkv
from tests.gpu_helpers import Case, bits_to_mask, mask_to_bits, rel_err, tables_to_numpy

pytestmark = pytest.mark.gpu
ATOL_REL = 1e-2


def _bs_attn(case: Case, M: np.ndarray) -> np.ndarray:
    p = case.params
    p.flags |= cpa.F_OUT_F32
    o = case.out(f32=True)
    bits = torch.from_numpy(mask_to_bits(M)).cuda()
    cpa.block_sparse_attention(p, case.dq, case.cache, bits, o)
    torch.cuda.synchronize()
    return o.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("B,Hq,Hkv,d,C,P,density", [
    (2, 8, 2, 128, 256, 1024, 0.2),
    (1, 4, 1, 128, 300, 768, 0.5),    # ragged last q-block
    (1, 8, 2, 64, 130, 512, 0.1),     # d = 64, one-token tail block
    (1, 2, 2, 128, 128, 0, 1.0),      # first chunk, MHA
])
def test_block_sparse_per_qblock_masks(B, Hq, Hkv, d, C, P, density):
    # per-(h, i) distinct masks, incl. bits beyond the causal limit (must be ignored)
    bs = 128
    q, k, v = random_qkv(B, Hq, Hkv, d, C, P + C, seed=C + P + d)
    case = Case(q, k, v, P, bs, seed=3)
    nqb, nkvb, pb, _ = O.geometry(C, P, bs)
    M = random_block_mask(B, Hq, nqb, nkvb, density, seed=C + 1)
    for i in range(nqb):
        M[:, :, i, pb + i] = True  # diagonal tile: every query row has a visible key
    got = _bs_attn(case, M)
    ref = O.block_sparse_attention(q, k, v, P, bs, M)
    assert rel_err(got, ref) <= ATOL_REL


def test_block_sparse_empty_rows_give_zero():
    # SPEC.md:445 makes an empty (b,h,i) row an error; the kernel defines it as O = 0 (cpa.h)
    B, Hq, Hkv, d, bs, C, P = 1, 4, 1, 128, 128, 256, 512
    q, k, v = random_qkv(B, Hq, Hkv, d, C, P + C, seed=77)
    case = Case(q, k, v, P, bs, seed=4)
    nqb, nkvb, pb, _ = O.geometry(C, P, bs)
    M = np.ones((B, Hq, nqb, nkvb), bool)
    M[0, 1, 0, :] = False
    got = _bs_attn(case, M)
    assert np.all(got[0, :128, 1] == 0.0)
    keep = M.copy()
    keep[0, 1, 0, :] = True  # oracle on the non-empty rows only
    ref = O.block_sparse_attention(q, k, v, P, bs, keep)
    ref[0, :128, 1] = 0.0
    assert rel_err(got, ref) <= ATOL_REL


@pytest.mark.parametrize("bs,E", [(16, 0), (128, 0), (64, 2)])
def test_expand_tables_bit_exact(bs, E):
    B, Hq, Hkv, d, C, P = 2, 8, 2, 64, 200, 40 * bs
    q, k, v = random_qkv(B, Hq, Hkv, d, C, P + C, seed=bs)
    case = Case(q, k, v, P, bs, seed=5, E=E)
    nqb, nkvb, pb, _ = O.geometry(C, P, bs)
    M = random_block_mask(B, Hq, nqb, nkvb, 0.1, seed=bs + 2)
    M[..., pb:] = True
    ip, ix = O.tables_from_mask(M, case.E, pb)
    t = cpa.BlockTables(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda())
    nwords = -(-nkvb // 32)
    bits = torch.full((B, Hq, nqb, nwords), -1, dtype=torch.int32, device="cuda")  # overwritten
    cpa.expand_tables(case.params, t, bits)
    torch.cuda.synchronize()
    ref = O.expand_tables_to_mask(ip, ix, B, Hq, case.E, C, P, bs)
    assert np.array_equal(bits.cpu().numpy(), mask_to_bits(ref))


def test_q_uniform_block_sparse_equals_zero_copy():
    # SPEC.md:447 / 454: block-sparse over the q-uniform expansion == the table executor. The 1-CTA
    # zero-copy kernel (F_NO_2CTA) runs the same per-head arithmetic, so the bits must agree; the
    # 2-CTA kernel orders the key sums differently (128-key pages) -> tolerance.
    B, Hq, Hkv, d, bs, C, P = 2, 8, 2, 128, 128, 384, 16 * 128
    q, k, v = random_qkv(B, Hq, Hkv, d, C, P + C, seed=123)
    case = Case(q, k, v, P, bs, seed=6)
    nqb, nkvb, pb, _ = O.geometry(C, P, bs)
    M = random_block_mask(B, Hq, nqb, nkvb, 0.1, seed=124)
    M[..., pb:] = True
    ip, ix = O.tables_from_mask(M, case.E, pb)
    t = cpa.BlockTables(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda())
    p = case.params
    p.flags |= cpa.F_OUT_F32
    bits = torch.empty(B, Hq, nqb, -(-nkvb // 32), dtype=torch.int32, device="cuda")
    cpa.expand_tables(p, t, bits)
    o_bs, o_zc, o_zc2 = case.out(True), case.out(True), case.out(True)
    cpa.block_sparse_attention(p, case.dq, case.cache, bits, o_bs)
    cpa.paged_attention(p, case.dq, case.cache, t, o_zc2)
    p.flags |= cpa.F_NO_2CTA
    cpa.paged_attention(p, case.dq, case.cache, t, o_zc)
    torch.cuda.synchronize()
    assert torch.equal(o_bs, o_zc)
    ref = O.paged_attention(q, k, v, P, bs, ip, ix)
    assert rel_err(o_bs.cpu().numpy().astype(np.float64), ref) <= ATOL_REL
    assert rel_err(o_zc2.cpu().numpy().astype(np.float64), ref) <= ATOL_REL


def test_block_sparse_of_estimator_mask_planted():
    # FlashPrefill-style execution of the estimator's own 2D mask (no unions), on the planted workload
    cfg = dataclasses.replace(CONFIGS["llama8b_32k"], name="mid", num_q_heads=8, num_kv_heads=2,
                              context=4096, chunk=512)
    seed = 4242
    k, v = make_kv(cfg, seed)
    q = make_q(cfg, seed)
    P, C, L = cfg.chunk_geometry()
    case = Case(q, k, v, P, cfg.block_size, seed=seed)
    p = case.params
    t = cpa.alloc_tables(p, mask=True)
    p.flags |= cpa.F_MASK_OUT
    ws = torch.empty(cpa.workspace_bytes(p), dtype=torch.uint8, device="cuda")
    cpa.build_tables(p, case.dq, case.cache, t, workspace=ws)
    p.flags = (p.flags & ~cpa.F_MASK_OUT) | cpa.F_OUT_F32
    o = case.out(True)
    cpa.block_sparse_attention(p, case.dq, case.cache, t.mask_bits, o)
    torch.cuda.synchronize()
    nqb, nkvb, pb, _ = O.geometry(C, P, cfg.block_size)
    M_gpu = bits_to_mask(t.mask_bits.cpu().numpy(), nkvb)
    M = O.threshold_mask(O.block_scores_pooled(q, k, P, cfg.block_size), 0.06, C, P, cfg.block_size)
    assert np.array_equal(M_gpu, M)
    ref = O.block_sparse_attention(q, k, v, P, cfg.block_size, M)
    assert rel_err(o.cpu().numpy().astype(np.float64), ref) <= ATOL_REL
    # executed per-(h,i) density is below the unioned tables' (the union's sparsity loss)
    ip, ix = tables_to_numpy(t)
    assert M[..., :pb].mean() < (ip[-1] - case.params.batch * 2 * (nkvb - pb)) / (2 * pb)


def test_block_sparse_rejects_unsupported_block_size():
    q, k, v = random_qkv(1, 4, 1, 64, 64, 128, seed=1)
    case = Case(q, k, v, 64, 32, seed=1)
    bits = torch.zeros(1, 4, 2, 1, dtype=torch.int32, device="cuda")
    with pytest.raises(cpa.CpaError) as e:
        cpa.block_sparse_attention(case.params, case.dq, case.cache, bits, case.out(False))
    assert e.value.status == 3  # CPA_ERR_UNSUPPORTED
