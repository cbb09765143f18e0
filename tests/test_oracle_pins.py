"""Pins of the fp64 oracle against values the paper/spec print, closed forms,
library routines, invariants and brute force (CPU only).

Every test names the passage it checks. None of them re-types the oracle's
formula: each one compares against an independent computation.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
from synth.workload import random_qkv, random_block_mask


def _sdpa_fp64(q, k, v, P, allowed=None):
    """torch SDPA (library routine) in fp64 with an explicit boolean mask.
    q [B,C,Hq,d]; k,v [B,Hkv,L,d]. allowed: [B,Hq,C,L] bool or None (causal)."""
    B, C, Hq, d = q.shape
    Hkv, L = k.shape[1], k.shape[2]
    E = Hq // Hkv
    qt = torch.from_numpy(q.astype(np.float64)).permute(0, 2, 1, 3)
    kt = torch.from_numpy(k.astype(np.float64)).repeat_interleave(E, dim=1)
    vt = torch.from_numpy(v.astype(np.float64)).repeat_interleave(E, dim=1)
    if allowed is None:
        t = torch.arange(L)[None, :]
        p = torch.arange(C)[:, None]
        allowed = (t <= P + p)[None, None].expand(B, Hq, C, L)
    else:
        allowed = torch.from_numpy(allowed)
    o = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=allowed)
    return o.permute(0, 2, 1, 3).numpy()


# --------------------------------------------------------------------------- attention

def test_dense_uniform_worked_example(golden):
    ex = golden["dense_uniform"]
    q = np.array(ex["q"], np.float32)[None, :, None, :]
    k = np.array(ex["k"], np.float32)[None, None]
    v = np.array(ex["v"], np.float32)[None, None]
    out = O.dense_causal_attention(q, k, v, P=ex["prefix_len"])
    assert out[0, 0, 0, 0] == ex["out"][0][0]
    out2 = O.paged_attention(q, k, v, P=ex["prefix_len"], bs=1)
    assert out2[0, 0, 0, 0] == ex["out"][0][0]


def test_single_allowed_kv_returns_v0():
    # prefix_len=0, chunk_len=1 -> out == v[0] exactly regardless of q, k
    q, k, v = random_qkv(1, 2, 1, 8, 1, 1, seed=3)
    out = O.dense_causal_attention(q, k, v, P=0)
    assert np.array_equal(out[0, 0, 0], v[0, 0, 0].astype(np.float64))
    assert np.array_equal(out[0, 0, 1], v[0, 0, 0].astype(np.float64))


@pytest.mark.parametrize("Hq,Hkv", [(4, 4), (8, 2), (8, 1)])
def test_dense_matches_torch_sdpa(Hq, Hkv):
    # SPEC.md:56 (independent brute force) -- here torch's SDPA in fp64
    q, k, v = random_qkv(2, Hq, Hkv, 16, 12, 40, seed=11)
    ref = _sdpa_fp64(q, k, v, P=28)
    out = O.dense_causal_attention(q, k, v, P=28)
    assert np.abs(out - ref).max() < 1e-12


def test_full_table_equals_dense():
    # full table == dense causal attention
    q, k, v = random_qkv(2, 8, 2, 16, 24, 72, seed=5)
    P, bs = 48, 8
    o1 = O.paged_attention(q, k, v, P, bs)
    o2 = O.dense_causal_attention(q, k, v, P)
    assert np.abs(o1 - o2).max() < 1e-12


def test_singleton_and_two_term_softmax():
    # singleton allowed set -> v[t]; two allowed keys -> hand 2-term softmax
    rng = np.random.default_rng(0)
    qp = rng.standard_normal(4)
    k = rng.standard_normal((8, 4))
    v = rng.standard_normal((8, 4))
    a = np.zeros(8, bool)
    a[5] = True
    assert np.array_equal(O.masked_attention_row(qp, k, v, a, 0.5), v[5])
    a[2] = True
    s2, s5 = 0.5 * qp @ k[2], 0.5 * qp @ k[5]
    w2 = 1.0 / (1.0 + math.exp(s5 - s2))
    hand = w2 * v[2] + (1.0 - w2) * v[5]
    assert np.abs(O.masked_attention_row(qp, k, v, a, 0.5) - hand).max() < 1e-14
    with pytest.raises(ValueError):
        O.masked_attention_row(qp, k, v, np.zeros(8, bool), 0.5)


def test_random_table_equals_masked_sdpa():
    # random table == masked dense attention with block-expanded allowed sets
    B, Hq, Hkv, d, bs = 2, 8, 2, 16, 8
    P, C = 64, 24
    L = P + C
    q, k, v = random_qkv(B, Hq, Hkv, d, C, L, seed=9)
    nqb, nkvb, pb, _ = O.geometry(C, P, bs)
    M = random_block_mask(B, Hq, nqb, nkvb, 0.2, seed=9)
    M[..., pb:] = True
    indptr, indices = O.tables_from_mask(M, Hq // Hkv, pb)
    out = O.paged_attention(q, k, v, P, bs, indptr, indices)
    allowed = np.zeros((B, Hq, C, L), bool)
    E = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            g = h // E
            for j in range(nkvb):
                if M[b, g * E:(g + 1) * E, :, j].any():
                    allowed[b, h, :, j * bs:(j + 1) * bs] = True
    for p in range(C):
        allowed[:, :, p, P + p + 1:] = False
    ref = _sdpa_fp64(q, k, v, P, allowed)
    assert np.abs(out - ref).max() < 1e-12


def test_chunk_only_table_is_fresh_dense_over_chunk():
    # table = current-chunk blocks only -> dense over the chunk alone, fresh causal mask
    B, Hq, Hkv, d, bs, P, C = 1, 4, 2, 16, 8, 32, 20
    q, k, v = random_qkv(B, Hq, Hkv, d, C, P + C, seed=21)
    nqb, nkvb, pb, _ = O.geometry(C, P, bs)
    G = np.zeros((B, Hq // (Hq // Hkv), nkvb), bool)
    G[..., pb:] = True
    indptr, indices = O.build_block_table(G, pb, nkvb)
    out = O.paged_attention(q, k, v, P, bs, indptr, indices)
    ref = _sdpa_fp64(q, k[:, :, P:], v[:, :, P:], 0)
    assert np.abs(out - ref).max() < 1e-12


@pytest.mark.parametrize("chunk", [512, 1024, 2048])
def test_chunking_transparency(chunk):
    # L=4096, D=32, B=2, Hq=8; chunked (full selection) == one-shot dense
    B, Hq, Hkv, d, L = 2, 8, 8, 32, 4096
    q, k, v = random_qkv(B, Hq, Hkv, d, L, L, seed=618)
    one_shot = _sdpa_fp64(q, k, v, P=0)  # library one-shot causal prefill
    outs = [O.dense_causal_attention(q[:, P:P + chunk], k[:, :, :P + chunk], v[:, :, :P + chunk], P)
            for P in range(0, L, chunk)]
    assert np.abs(np.concatenate(outs, axis=1) - one_shot).max() < 1e-10


def test_chunking_transparency_through_tables():
    # the table path with full selection, chunk by chunk, equals one-shot dense
    B, Hq, Hkv, d, L, bs, chunk = 1, 4, 2, 8, 96, 8, 32
    q, k, v = random_qkv(B, Hq, Hkv, d, L, L, seed=7)
    one_shot = _sdpa_fp64(q, k, v, P=0)
    outs = []
    for P in range(0, L, chunk):
        qs, ks, vs = q[:, P:P + chunk], k[:, :, :P + chunk], v[:, :, :P + chunk]
        nqb, nkvb, pb, _ = O.geometry(chunk, P, bs)
        M = np.ones((B, Hq, nqb, nkvb), bool)
        ip, ix = O.tables_from_mask(M, Hq // Hkv, pb)
        outs.append(O.paged_attention(qs, ks, vs, P, bs, ip, ix))
    assert np.abs(np.concatenate(outs, axis=1) - one_shot).max() < 1e-12


def test_causal_perturbation_invariance():
    # perturbing causally forbidden KV tokens changes no output (delta == 0)
    B, Hq, Hkv, d, bs, P, C = 1, 4, 2, 8, 8, 16, 16
    q, k, v = random_qkv(B, Hq, Hkv, d, C, P + C, seed=4)
    p0 = 5
    o1 = O.paged_attention(q, k, v, P, bs)
    k2, v2 = k.copy(), v.copy()
    k2[:, :, P + p0 + 1:] += 7.0
    v2[:, :, P + p0 + 1:] -= 3.0
    o2 = O.paged_attention(q, k2, v2, P, bs)
    assert np.array_equal(o1[:, :p0 + 1], o2[:, :p0 + 1])
    assert not np.array_equal(o1[:, p0 + 1:], o2[:, p0 + 1:])


# --------------------------------------------------------------------------- estimator

def test_threshold_worked_example(golden):
    ex = golden["threshold_row"]
    bs = 4
    m = np.log(np.array(ex["scores"]))[None, None, None, :]  # score = exp(m - m*) with m* = 0
    P, C = ex["chunk_block"] * bs, bs
    for case in ex["cases"]:
        for sink in (True, False):
            M = O.threshold_mask(m, case["alpha"], C, P, bs, sink=sink)
            assert M[0, 0, 0].astype(int).tolist() == case["bits"]


def test_threshold_boundaries():
    # alpha -> 0+ gives the full causal mask; alpha = 1 keeps argmax + forced
    q, k, _ = random_qkv(1, 4, 2, 16, 24, 88, seed=17)
    P, bs = 64, 8
    m = O.block_scores_pooled(q, k, P, bs)
    nqb, nkvb, pb, _ = O.geometry(24, P, bs)
    full = O.threshold_mask(m, 1e-300, 24, P, bs)
    for i in range(nqb):
        assert full[..., i, :pb + i + 1].all() and not full[..., i, pb + i + 1:].any()
    one = O.threshold_mask(m, 1.0, 24, P, bs, sink=False)
    for h in range(4):
        for i in range(nqb):
            arg = int(np.argmax(m[0, h, i]))
            expect = {arg} | set(range(pb, pb + i + 1))
            assert set(np.nonzero(one[0, h, i])[0].tolist()) == expect
    with pytest.raises(ValueError):
        O.threshold_mask(m, 0.0, 24, P, bs)
    with pytest.raises(ValueError):
        O.threshold_mask(m, 1.5, 24, P, bs)


def test_alpha_monotone():
    # alpha1 <= alpha2 => mask(alpha1) superset of mask(alpha2)
    q, k, _ = random_qkv(1, 4, 1, 16, 16, 80, seed=23)
    m = O.block_scores_pooled(q, k, 64, 8)
    alphas = [0.001, 0.01, 0.06, 0.2, 0.5, 1.0]
    masks = [O.threshold_mask(m, a, 16, 64, 8) for a in alphas]
    for a, b in zip(masks, masks[1:]):
        assert (a | b == a).all()


def test_pooled_scores_brute_force():
    # per-tile max agrees with brute force (pure-Python dot products and means)
    B, Hq, Hkv, d, bs, P, C = 1, 2, 1, 4, 4, 8, 7  # partial last q-block and last kv-block
    q, k, _ = random_qkv(B, Hq, Hkv, d, C, P + C, seed=31)
    m = O.block_scores_pooled(q, k, P, bs)
    L = P + C
    scale = 1.0 / math.sqrt(d)
    for h in range(Hq):
        for i in range(2):
            ps = [p for p in range(i * bs, min(i * bs + bs, C))]
            qbar = [sum(float(q[0, p, h, e]) for p in ps) / len(ps) for e in range(d)]
            for j in range(4):
                ts = [t for t in range(j * bs, min(j * bs + bs, L)) if t <= P + ps[-1]]
                if j > P // bs + i:
                    assert m[0, h, i, j] == -np.inf
                    continue
                best = max(scale * sum(qbar[e] * float(k[0, 0, t, e]) for e in range(d)) for t in ts)
                assert abs(m[0, h, i, j] - best) < 1e-12


@pytest.mark.parametrize("C,seed", [(7, 41), (12, 42), (16, 43)])
def test_exact_scores_brute_force(C, seed):
    # SPEC.md:223 (tile max over every causal (query, key) pair of the tile, t <= P + p for EACH
    # query p) and SPEC.md:228 ("random instance -> per-tile max-logit agrees with brute-force max
    # over the tile"). Distinct queries, partial last q-block / kv-block, diagonal tiles included:
    # pure-Python dot products over the explicit pair set, no matmul, no block arithmetic reuse.
    B, Hq, Hkv, d, bs, P = 1, 4, 2, 4, 4, 8
    L = P + C
    q, k, _ = random_qkv(B, Hq, Hkv, d, C, L, seed=seed)
    m = O.block_scores_exact(q, k, P, bs)
    scale = 1.0 / math.sqrt(d)
    nqb, nkvb = -(-C // bs), -(-L // bs)
    assert m.shape == (B, Hq, nqb, nkvb)
    for h in range(Hq):
        kvh = h // (Hq // Hkv)
        for i in range(nqb):
            for j in range(nkvb):
                pairs = [(p, t) for p in range(C) if p // bs == i
                         for t in range(L) if t // bs == j and t <= P + p]
                if not pairs:
                    assert m[0, h, i, j] == -np.inf, (h, i, j)
                    continue
                best = max(scale * sum(float(q[0, p, h, e]) * float(k[0, kvh, t, e]) for e in range(d))
                           for p, t in pairs)
                assert abs(m[0, h, i, j] - best) < 1e-12, (h, i, j)


def test_exact_scores_per_query_causal_limit():
    # on a diagonal tile a key is visible only to the queries at or after it. Plant a
    # key at chunk position 3 that aligns with query 0 only (query 0 cannot see it: 3 > 0), and make
    # query 3 orthogonal to it: the exact tile max must NOT contain that pair, while the pooled
    # scorer (union limit t <= P + last_p, R6) does see the key.
    d, bs, P, C = 4, 4, 4, 4
    q = np.zeros((1, C, 1, d), np.float32)
    k = np.zeros((1, 1, P + C, d), np.float32)
    q[0, 0, 0] = [1, 0, 0, 0]
    q[0, 1, 0] = [0, 1, 0, 0]
    q[0, 2, 0] = [0, 0, 1, 0]
    q[0, 3, 0] = [0, 0, 0, 1]
    k[0, 0, P + 3] = [50, 0, 0, 0]   # huge only against query 0, which is causally blind to it
    k[0, 0, P + 0] = [0, 0, 0, 2]    # seen by every query; logit 2*0.5 = 1.0 with query 3
    me = O.block_scores_exact(q, k, P, bs)
    assert me[0, 0, 0, 1] == pytest.approx(1.0, abs=1e-12)   # max over causal pairs = q3.k(P+0)
    mp = O.block_scores_pooled(q, k, P, bs)
    assert mp[0, 0, 0, 1] == pytest.approx(50 * 0.25 * 0.5, abs=1e-12)  # qbar = 1/4 of each axis


def test_constant_keys_keep_everything():
    # identical keys everywhere -> all in-causal scores equal -> all kept
    q, k, _ = random_qkv(1, 4, 1, 8, 16, 48, seed=2)
    k[:] = k[:, :, :1]
    m = O.block_scores_pooled(q, k, 32, 8)
    M = O.threshold_mask(m, 0.999, 16, 32, 8, sink=False)
    for i in range(2):
        assert M[..., i, :4 + i + 1].all()


def test_dominant_key():
    # one key with dominant logit -> its block scores the row max, others strictly less
    q, k, _ = random_qkv(1, 1, 1, 8, 8, 40, seed=8)
    qbar = q[0, :, 0].astype(np.float64).mean(axis=0)
    k[0, 0, 13] = (40.0 * qbar / np.linalg.norm(qbar)).astype(np.float32)
    m = O.block_scores_pooled(q, k, 32, 8)
    row = m[0, 0, 0]
    assert np.argmax(row) == 1 and (np.delete(row, 1) < row[1]).all()


def test_pooled_equals_exact_for_constant_qblocks():
    # Derived pin: when all queries of a q-block are identical, pooled == exact
    # except that exact uses per-query causal sets; on prefix tiles both are the plain tile max.
    q, k, _ = random_qkv(1, 4, 2, 16, 16, 48, seed=12)
    q[:, 0:8] = q[:, 0:1]
    q[:, 8:16] = q[:, 8:9]
    P, bs = 32, 8
    mp = O.block_scores_pooled(q, k, P, bs)
    me = O.block_scores_exact(q, k, P, bs)
    pb = P // bs
    assert np.abs(mp[..., :pb] - me[..., :pb]).max() < 1e-12
    # exact can only be <= pooled on chunk tiles (subset of pairs for the same query value)
    assert (me[..., pb:][np.isfinite(me[..., pb:])] <= mp[..., pb:][np.isfinite(me[..., pb:])] + 1e-12).all()


# --------------------------------------------------------------------------- unions / tables

def test_union_worked_examples(golden):
    M = np.array(golden["q_block_union"]["M"], bool)[None, None]
    assert O.q_block_union(M)[0, 0].astype(int).tolist() == golden["q_block_union"]["out"]
    heads = np.array(golden["intra_group_union"]["heads"], bool)[None]
    assert O.intra_group_union(heads, 2)[0, 0].astype(int).tolist() == golden["intra_group_union"]["out"]
    assert (O.intra_group_union(heads, 1) == heads).all()  # SPEC.md:336 identity


def test_csr_worked_examples(golden):
    G = np.array(golden["table_row"]["G"], bool)[None, None]
    ip, ix = O.build_block_table(G)
    assert ix.tolist() == golden["table_row"]["table"] and ip.tolist() == [0, 3]
    G = np.array(golden["csr_two_groups"]["G"], bool)[None]
    ip, ix = O.build_block_table(G)
    assert ip.tolist() == golden["csr_two_groups"]["kv_indptr"]
    assert ix.tolist() == golden["csr_two_groups"]["kv_indices"]
    with pytest.raises(ValueError):  # SPEC.md:344 open-chunk violation
        O.build_block_table(G, pb=2, nkvb=3)


def test_head_to_group(golden):
    for c in golden["head_to_group"]["cases"]:
        assert O.head_to_group(c["h"], c["Hq"], c["Hkv"], c["E"]) == c["g"]
    s = golden["head_to_group"]["subgroups"]
    gs = sorted({O.head_to_group(h, s["Hq"], s["Hkv"], s["E"]) for h in range(s["Hq"])
                 if O.kv_head_of(h, s["Hq"], s["Hkv"]) == 0})
    assert gs == s["groups_sharing_kv0"]
    with pytest.raises(IndexError):
        O.head_to_group(32, 32, 8, 4)


def _brute_table(M, E, pb):
    B, Hq, nqb, nkvb = M.shape
    rows = []
    for b in range(B):
        for g in range(Hq // E):
            rows.append([j for j in range(nkvb)
                         if j >= pb or any(M[b, h, i, j] for h in range(g * E, (g + 1) * E) for i in range(nqb))])
    return rows


def test_union_coverage_minimality_random():
    # SPEC.md:616 acceptance #1 (>=1000 random masks; B<=4, Hq<=32, 8 q-blocks, 32 kv-blocks, GQA 1/4/8)
    rng = np.random.default_rng(616)
    for trial in range(1000):
        B = int(rng.integers(1, 5))
        Hkv = int(rng.choice([1, 2, 4]))
        E = int(rng.choice([1, 4, 8]))
        Hq = min(Hkv * E, 32)
        nqb, nkvb = 8, 32
        pb = nkvb - nqb
        M = rng.random((B, Hq, nqb, nkvb)) < rng.random()
        for i in range(nqb):
            M[:, :, i, pb + i + 1:] = False
            M[:, :, i, pb:pb + i + 1] = True
        ip, ix = O.tables_from_mask(M, E, pb)
        rows = _brute_table(M, E, pb)
        assert ip.tolist() == np.cumsum([0] + [len(r) for r in rows]).tolist()
        assert ix.tolist() == [j for r in rows for j in r]
        assert O.check_minimality(ip, ix, M, E, pb)


def test_minimality_counterexample():
    # one extra prefix block injected -> minimality check fails
    M = np.zeros((1, 4, 2, 8), bool)
    M[0, 1, 0, 2] = True
    M[..., 6:] = True
    M[:, :, 0, 7] = False
    ip, ix = O.tables_from_mask(M, 4, 6)
    assert O.check_minimality(ip, ix, M, 4, 6)
    ix2 = np.sort(np.append(ix, 4)).astype(np.int32)
    ip2 = ip.copy()
    ip2[1:] += 1
    assert not O.check_minimality(ip2, ix2, M, 4, 6)


def test_unions_commute_and_idempotent():
    # SPEC.md:373-374
    M = random_block_mask(2, 8, 4, 16, 0.2, seed=77)
    a = O.intra_group_union(O.q_block_union(M), 4)
    heador = np.zeros((2, 2, 4, 16), bool)
    for h in range(8):
        heador[:, h // 4] |= M[:, h]
    b = O.q_block_union(heador)
    assert (a == b).all()
    Mbar = O.q_block_union(M)
    assert (O.q_block_union(Mbar[:, :, None, :]) == Mbar).all()


def test_sparsity_full_and_hand_count(golden):
    # SPEC.md:366 full causal -> 0 everywhere
    P, C, bs = 32, 8, 8
    s = O.sparsity_stats(np.ones((1, 4, 1, 5), bool), 4, C, P, bs)
    assert all(abs(v) < 1e-15 for v in s.values())
    # 4 heads of one group each select a disjoint singleton among 4 prefix
    # blocks (+ forced chunk block 4, excluded from the stats)
    M = np.zeros((1, 4, 1, 5), bool)
    for h in range(4):
        M[0, h, 0, h] = True
    M[..., 4] = True
    s = O.sparsity_stats(M, 4, 8, 32, 8, prefix_only=True)
    ex = golden["sparsity_hand_count"]
    assert abs(s["q_union"] - ex["q_union"]) < 1e-15
    assert abs(s["group_union"] - ex["group_union"]) < 1e-15
    assert abs(s["pre"] - 0.75) < 1e-15


def test_sparsity_monotone_random():
    # SPEC.md:368, 375, 620; ordering of PAPER.md:515-519
    rng = np.random.default_rng(620)
    for _ in range(200):
        M = rng.random((2, 8, 4, 20)) < rng.random() * 0.5
        s = O.sparsity_stats(M, 8, 32, 128, 8, sub=4)
        assert s["pre"] >= s["q_union"] >= s["subgroup_union"] >= s["group_union"]


def test_ideal_speedup_ten(golden):
    # q-uniform 90%-sparse selection -> dense/sparse flops = 10 +/- 2%
    C, bs, d, E = 128, 128, 128, 4
    P = 1280 * bs
    nkvb = P // bs + 1
    dense_ip = np.array([0, nkvb])
    dense_ix = np.arange(nkvb)
    keep = np.arange(0, nkvb - 1, 10)  # 10% of prefix blocks
    sp_ix = np.concatenate([keep, [nkvb - 1]])
    sp_ip = np.array([0, len(sp_ix)])
    ratio = O.attention_flops(dense_ip, dense_ix, C, P, bs, E, d) / O.attention_flops(sp_ip, sp_ix, C, P, bs, E, d)
    ex = golden["ideal_speedup"]
    assert abs(ratio - ex["value"]) / ex["value"] < ex["rel_tol"]


def test_chunk_step_end_to_end_tiny():
    # PAPER.md:165-175 pipeline on the tiny config; tables minimal & chunk-open; O finite
    from synth.workload import CONFIGS, make_kv, make_q
    cfg = CONFIGS["tiny"]
    k, v = make_kv(cfg, 16839)
    q = make_q(cfg, 16839)
    P, C, L = cfg.chunk_geometry()
    r = O.chunk_step(q, k, v, P, cfg.block_size, alpha=0.06)
    nqb, nkvb, pb, _ = O.geometry(C, P, cfg.block_size)
    assert O.check_minimality(r["indptr"], r["indices"], r["M"], cfg.group_size, pb)
    assert np.isfinite(r["O"]).all()


# ---- block-sparse executor (Fig. 7(c) baseline)

def test_block_sparse_per_qblock_mask_equals_masked_sdpa():
    # per-i distinct masks == masked dense attention with per-query allowed sets
    B, Hq, Hkv, d, bs, P, C = 2, 4, 2, 16, 8, 48, 21
    L = P + C
    q, k, v = random_qkv(B, Hq, Hkv, d, C, L, seed=31)
    nqb, nkvb, pb, _ = O.geometry(C, P, bs)
    M = random_block_mask(B, Hq, nqb, nkvb, 0.3, seed=31)
    for i in range(nqb):
        M[:, :, i, pb + i] = True  # the diagonal tile keeps every row non-empty
    out = O.block_sparse_attention(q, k, v, P, bs, M)
    allowed = torch.zeros(B, Hq, C, L, dtype=torch.bool)
    Mt = torch.from_numpy(M)
    for p in range(C):
        allowed[:, :, p, :] = Mt[:, :, p // bs, :].repeat_interleave(bs, dim=-1)[..., :L]
        allowed[:, :, p, P + p + 1:] = False
    ref = _sdpa_fp64(q, k, v, P, allowed.numpy())
    assert np.abs(out - ref).max() < 1e-12


def test_block_sparse_full_mask_equals_dense():
    # SPEC.md:448 "full mask -> equals dense oracle"
    B, Hq, Hkv, d, bs, P, C = 1, 4, 1, 16, 8, 32, 17
    q, k, v = random_qkv(B, Hq, Hkv, d, C, P + C, seed=32)
    nqb, nkvb, _, _ = O.geometry(C, P, bs)
    out = O.block_sparse_attention(q, k, v, P, bs, np.ones((B, Hq, nqb, nkvb), bool))
    assert np.abs(out - O.dense_causal_attention(q, k, v, P)).max() < 1e-12


def test_block_sparse_of_q_uniform_expansion_equals_tables():
    # SPEC.md:447 + invariant SPEC.md:454: q-uniform expansion of the table == zero-copy executor
    B, Hq, Hkv, d, bs, P, C = 2, 8, 2, 16, 8, 64, 24
    q, k, v = random_qkv(B, Hq, Hkv, d, C, P + C, seed=33)
    nqb, nkvb, pb, _ = O.geometry(C, P, bs)
    M = random_block_mask(B, Hq, nqb, nkvb, 0.15, seed=33)
    M[..., pb:] = True
    E = Hq // Hkv
    indptr, indices = O.tables_from_mask(M, E, pb)
    Mq = O.expand_tables_to_mask(indptr, indices, B, Hq, E, C, P, bs)
    # the expansion is causal-consistent and lowers back to the same tables
    for i in range(nqb):
        assert not Mq[:, :, i, pb + i + 1:].any()
    ip2, ix2 = O.tables_from_mask(Mq, E, pb)
    assert np.array_equal(ip2, indptr) and np.array_equal(ix2, indices)
    a = O.block_sparse_attention(q, k, v, P, bs, Mq)
    b_ = O.paged_attention(q, k, v, P, bs, indptr, indices)
    assert np.abs(a - b_).max() < 1e-12


def test_block_sparse_empty_row_raises():
    # empty row per (b,h,i) -> error
    q, k, v = random_qkv(1, 2, 1, 8, 8, 16, seed=34)
    M = np.zeros((1, 2, 1, 2), bool)
    with pytest.raises(ValueError):
        O.block_sparse_attention(q, k, v, 8, 8, M)
