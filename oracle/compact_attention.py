"""fp64 CPU oracle for CompactAttention's chunked-prefill hot path.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module. The product path
(paper_2605_16839_b200) never imports it and has no CPU fallback.

Plain, slow, obviously-correct numpy in float64, written step by step in the
paper's order and notation (arXiv 2605.16839, /root/reference/PAPER.md) with the
estimator SPEC.md fixes. Citations are PAPER.md / SPEC.md line numbers. It shares
no code with the CUDA path; its only inputs are the seeded bf16-valued tensors
from synth/.

Notation (§3.2):
  B batch, Hq query heads, Hkv KV heads, E = execution-group size (query heads per
  group, default Hq/Hkv: "a KV group by default"), G = Hq/E groups,
  d head dim, bs block size (= page size = Q-block size), C chunk
  length, P prefix length (tokens cached before the chunk, P % bs == 0),
  L = P + C, nqb = ceil(C/bs), nkvb = ceil(L/bs), pb = P/bs.
  Query position p in [0, C) has absolute position P + p.
Layouts: q [B, C, Hq, d]; k, v logical flat [B, Hkv, L, d] (PAPER.md:246
"KV-head-major layout [B, H_kv, L, D]").

Parity status:
  dense / masked attention ....... pinned (closed forms, torch SDPA fp64, chunking transparency)
  unions, table, CSR ............. pinned (SPEC worked examples, brute-force triple loop)
  threshold_mask ................. pinned (SPEC.md:236-238 worked examples, boundaries)
  block_scores_pooled ............ pinned (brute-force tile max; pooled == exact when a
                                   q-block's queries are identical)
  block_scores_exact ............. pinned (pure-Python brute force over the explicit causal
                                   (p, t) pair set incl. partial diagonal tiles, SPEC.md:223, 228;
                                   planted per-query causal-limit case)
  pooled estimator on real model activations: parity unpinned (the paper prints no
  scores, masks or FlashPrefill formula).
"""
from __future__ import annotations

import math
from typing import Optional

import numpy as np

NEG_INF = -np.inf


# ----------------------------------------------------------------------------
# Geometry and GQA map
# ----------------------------------------------------------------------------

def geometry(C: int, P: int, bs: int):
    """(nqb, nkvb, pb, L) of a chunk. SPEC.md:40-45 CausalLayout; P % bs == 0 (R8)."""
    if P % bs != 0:
        raise ValueError("prefix_len must be a multiple of block_size")
    L = P + C
    return -(-C // bs), -(-L // bs), P // bs, L


def head_to_group(h: int, Hq: int, Hkv: int, E: int) -> int:
    """g = floor(h / E) (PAPER.md:203 H(g)); E must divide Hq/Hkv."""
    if not (0 <= h < Hq):
        raise IndexError("query head out of range")
    if Hq % Hkv != 0 or (Hq // Hkv) % E != 0:
        raise ValueError("exec_group_size must divide Hq/Hkv")
    return h // E


def kv_head_of(h: int, Hq: int, Hkv: int) -> int:
    """Query head h reads KV head floor(h / (Hq/Hkv))."""
    return h // (Hq // Hkv)


def causal_valid(i: int, j: int, pb: int) -> bool:
    """Tile (q-block i, kv-block j) has at least one causal pair iff j <= pb + i."""
    return j <= pb + i


# ----------------------------------------------------------------------------
# (a1, a2) Pattern search: FlashPrefill-style max-threshold scorer, pooled-query variant
# ----------------------------------------------------------------------------

def pool_queries(q: np.ndarray, bs: int) -> np.ndarray:
    """qbar[b,h,i,:] = mean over the valid queries p of q-block i of q[b,p,h,:], fp64.

    SPEC.md:269 "a query-pooled variant (score with block-mean queries)". The last
    q-block may be partial; the mean is over its valid queries (R8).
    Returns [B, Hq, nqb, d] float64.
    """
    B, C, Hq, d = q.shape
    nqb = -(-C // bs)
    out = np.empty((B, Hq, nqb, d), np.float64)
    for i in range(nqb):
        blk = q[:, i * bs:min((i + 1) * bs, C)].astype(np.float64)  # [B, n_i, Hq, d]
        out[:, :, i, :] = blk.mean(axis=1)
    return out


def block_scores_pooled(q: np.ndarray, k: np.ndarray, P: int, bs: int,
                        sm_scale: Optional[float] = None) -> np.ndarray:
    """Tile max of pooled logits, m[b,h,i,j] (fp64), -inf outside the causal region.

    SPEC.md:220-228 (score = max over the tile of the raw logit q.k/sqrt(D)) with the
    pooled query of SPEC.md:269 standing for the tile's queries:
      m[b,h,i,j] = max_{t in block j, t <= P + last_p(i), t < L} scale * qbar[b,h,i] . k[b, kvh(h), t]
    last_p(i) = min((i+1)*bs, C) - 1 (the pooled query's causal set is the union of its
    queries' sets, R6). Returns [B, Hq, nqb, nkvb].
    """
    B, C, Hq, d = q.shape
    _, Hkv, L, _ = k.shape
    nqb, nkvb, pb, L2 = geometry(C, P, bs)
    assert L == L2, "k length must equal P + C"
    scale = 1.0 / math.sqrt(d) if sm_scale is None else float(sm_scale)
    qbar = pool_queries(q, bs)
    m = np.full((B, Hq, nqb, nkvb), NEG_INF)
    for b in range(B):
        for h in range(Hq):
            kh = k[b, kv_head_of(h, Hq, Hkv)].astype(np.float64)  # [L, d]
            logits = scale * (qbar[b, h] @ kh.T)  # [nqb, L]  (library matmul as one step)
            for i in range(nqb):
                last_abs = P + min((i + 1) * bs, C) - 1
                for j in range(nkvb):
                    if not causal_valid(i, j, pb):
                        continue
                    lo, hi = j * bs, min((j + 1) * bs, L, last_abs + 1)
                    m[b, h, i, j] = logits[i, lo:hi].max()
    return m


def block_scores_exact(q: np.ndarray, k: np.ndarray, P: int, bs: int,
                       sm_scale: Optional[float] = None) -> np.ndarray:
    """SPEC's default scorer: tile max over all causal (p, t) pairs of q_p.k_t*scale.

    Test-only here (NEXT-1 on GPU). Returns [B, Hq, nqb, nkvb] fp64, -inf outside causal region.
    """
    B, C, Hq, d = q.shape
    _, Hkv, L, _ = k.shape
    nqb, nkvb, pb, _ = geometry(C, P, bs)
    scale = 1.0 / math.sqrt(d) if sm_scale is None else float(sm_scale)
    m = np.full((B, Hq, nqb, nkvb), NEG_INF)
    for b in range(B):
        for h in range(Hq):
            kh = k[b, kv_head_of(h, Hq, Hkv)].astype(np.float64)
            for i in range(nqb):
                qs = q[b, i * bs:min((i + 1) * bs, C), h].astype(np.float64)
                logits = scale * (qs @ kh.T)  # [n_i, L]
                for j in range(nkvb):
                    if not causal_valid(i, j, pb):
                        continue
                    best = NEG_INF
                    for pp in range(qs.shape[0]):
                        p = i * bs + pp
                        lo, hi = j * bs, min((j + 1) * bs, L, P + p + 1)
                        if hi > lo:
                            best = max(best, logits[pp, lo:hi].max())
                    m[b, h, i, j] = best
    return m


def row_max(m: np.ndarray) -> np.ndarray:
    """m*[b,h,i] = max_j' m[b,h,i,j'] over all causal-valid j' incl. chunk tiles (R3)."""
    return m.max(axis=-1)


def threshold_mask(m: np.ndarray, alpha: float, C: int, P: int, bs: int, sink: bool = True) -> np.ndarray:
    """2D block mask M[b,h,i,j] from max-threshold scores.

    SPEC.md:233 keep rule: score >= alpha * max_j' score, with score = exp(m - m*)
    (SPEC.md:223), i.e. in the log domain m - m* >= ln(alpha) (exp is monotone and the
    row-max score is exp(0) = 1).  OR the block overlaps the current chunk (fully-open
    rule), OR j == 0 when the sink flag is on
    (SPEC.md:268).  The "local anchor" of SPEC.md:233 is the row's last causal block,
    which lies inside the chunk and is already forced (R4, pinned by
    SPEC.md:238).  Causal-invalid tiles are 0.
    """
    if not (0.0 < alpha <= 1.0):
        raise ValueError("alpha must be in (0, 1]")
    B, Hq, nqb, nkvb = m.shape
    _, nkvb2, pb, _ = geometry(C, P, bs)
    assert nkvb == nkvb2
    mstar = row_max(m)
    ln_alpha = math.log(alpha)
    M = np.zeros(m.shape, dtype=bool)
    for i in range(nqb):
        for j in range(nkvb):
            if not causal_valid(i, j, pb):
                continue
            keep = (m[:, :, i, j] - mstar[:, :, i]) >= ln_alpha
            forced = (j >= pb) or (sink and j == 0)
            M[:, :, i, j] = keep | forced
    return M


# ----------------------------------------------------------------------------
# (a4, a5) Block-union KV table construction
# ----------------------------------------------------------------------------

def q_block_union(M: np.ndarray) -> np.ndarray:
    """Mbar[b,h,j] = OR_i M[b,h,i,j]."""
    B, Hq, nqb, nkvb = M.shape
    out = np.zeros((B, Hq, nkvb), dtype=bool)
    for i in range(nqb):
        out |= M[:, :, i, :]
    return out


def intra_group_union(Mbar: np.ndarray, E: int) -> np.ndarray:
    """G[b,g,j] = OR_{h in H(g)} Mbar[b,h,j], H(g) = [g*E, (g+1)*E)."""
    B, Hq, nkvb = Mbar.shape
    if Hq % E != 0:
        raise ValueError("grouping mismatch")
    G = np.zeros((B, Hq // E, nkvb), dtype=bool)
    for h in range(Hq):
        G[:, h // E, :] |= Mbar[:, h, :]
    return G


def build_block_table(G: np.ndarray, pb: Optional[int] = None, nkvb: Optional[int] = None):
    """T[b,g] = {j | G[b,g,j] = 1} as CSR over pseudo-rows r = b*G + g.

    kv_indptr[0] = 0, kv_indptr[r+1] - kv_indptr[r] = |T[b,g]|, kv_indices ascending within
    a row. If pb is given, every row must contain
    the chunk blocks [pb, nkvb) (open-chunk rule); otherwise ValueError.
    """
    B, Gn, nk = G.shape
    indptr = [0]
    indices = []
    for b in range(B):
        for g in range(Gn):
            row = [j for j in range(nk) if G[b, g, j]]
            if pb is not None:
                top = nk if nkvb is None else nkvb
                for j in range(pb, top):
                    if not G[b, g, j]:
                        raise ValueError(f"open-chunk violation in row {b * Gn + g}")
            indices.extend(row)
            indptr.append(len(indices))
    return np.asarray(indptr, np.int32), np.asarray(indices, np.int32)


def tables_from_mask(M: np.ndarray, E: int, pb: Optional[int] = None):
    """Full lowering: Q-block union -> intra-group union -> CSR table."""
    G = intra_group_union(q_block_union(M), E)
    return build_block_table(G, pb, M.shape[-1])


def check_minimality(indptr, indices, M: np.ndarray, E: int, pb: int) -> bool:
    """every tabled j has a witness (h in H(g), i) with M=1, or is a chunk block."""
    B, Hq, nqb, nkvb = M.shape
    Gn = Hq // E
    for b in range(B):
        for g in range(Gn):
            r = b * Gn + g
            for j in indices[indptr[r]:indptr[r + 1]]:
                if j >= pb:
                    continue
                if not any(M[b, h, i, j] for h in range(g * E, (g + 1) * E) for i in range(nqb)):
                    return False
    return True


def sparsity_stats(M: np.ndarray, E: int, C: int, P: int, bs: int, sub: Optional[int] = None,
                   prefix_only: bool = False):
    """SPEC.md:360-368 SparsityReport over causal-valid slots (R14).

    pre: per (b,h,i,j) slot; q_union: slot (b,h,i,j) counted selected if Mbar[b,h,j];
    subgroup (exec group of size `sub`, default E) and group (full KV group of size
    Hq/Hkv = E_kv passed as E) likewise. prefix_only restricts the slots to prefix blocks
    j < pb (forced chunk blocks excluded). Returns fractions NOT selected.
    """
    B, Hq, nqb, nkvb = M.shape
    _, _, pb, _ = geometry(C, P, bs)
    valid = np.zeros((nqb, nkvb), dtype=bool)
    for i in range(nqb):
        for j in range(nkvb):
            valid[i, j] = causal_valid(i, j, pb) and (not prefix_only or j < pb)
    n_valid = valid.sum() * B * Hq
    Mbar = q_block_union(M)
    sub = E if sub is None else sub
    Gs = intra_group_union(Mbar, sub)
    Gk = intra_group_union(Mbar, E)
    sel = {"pre": 0, "q_union": 0, "subgroup_union": 0, "group_union": 0}
    for h in range(Hq):
        sel["pre"] += (M[:, h] & valid).sum()
        sel["q_union"] += (Mbar[:, h][:, None, :] & valid).sum()
        sel["subgroup_union"] += (Gs[:, h // sub][:, None, :] & valid).sum()
        sel["group_union"] += (Gk[:, h // E][:, None, :] & valid).sum()
    return {k: 1.0 - v / n_valid for k, v in sel.items()}


# ----------------------------------------------------------------------------
# (a6) Attention over tabled blocks, in absolute coordinates
# ----------------------------------------------------------------------------

def allowed_from_tables(indptr, indices, b: int, g: int, Gn: int, P: int, p: int, bs: int, L: int) -> np.ndarray:
    """A(p) = {t : floor(t/bs) in T[b,g], t <= P + p, t < L}."""
    r = b * Gn + g
    allowed = np.zeros(L, dtype=bool)
    for j in indices[indptr[r]:indptr[r + 1]]:
        allowed[j * bs:min((j + 1) * bs, L)] = True
    allowed[P + p + 1:] = False
    return allowed


def masked_attention_row(qp: np.ndarray, k: np.ndarray, v: np.ndarray, allowed: np.ndarray,
                         scale: float) -> np.ndarray:
    """out = sum_t softmax_t(scale q.k_t) v_t over allowed t, max-subtracted, fp64."""
    idx = np.nonzero(allowed)[0]
    if idx.size == 0:
        raise ValueError("degenerate row: empty allowed set (SPEC.md:62)")
    s = scale * (k[idx].astype(np.float64) @ qp.astype(np.float64))
    w = np.exp(s - s.max())
    w /= w.sum()
    return w @ v[idx].astype(np.float64)


def paged_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, P: int, bs: int,
                    indptr=None, indices=None, E: Optional[int] = None,
                    sm_scale: Optional[float] = None, rows=None) -> np.ndarray:
    """O[b,p,h] over the tabled blocks T[b, g(h)] in ORIGINAL absolute positions.

    PAPER.md:226-253 (zero-copy paged execution; the value is masked_dense_attention with
    block-expanded allowed sets). indptr=None means the dense baseline:
    every block [0, nkvb). `rows` = optional list of (b, p, h) to compute
    (others left NaN) for sampled parity at full size.
    Returns [B, C, Hq, d] float64.
    """
    B, C, Hq, d = q.shape
    _, Hkv, L, _ = k.shape
    nqb, nkvb, pb, L2 = geometry(C, P, bs)
    assert L == L2
    E = Hq // Hkv if E is None else E
    Gn = Hq // E
    scale = 1.0 / math.sqrt(d) if sm_scale is None else float(sm_scale)
    if indptr is None:
        indptr = np.arange(B * Gn + 1, dtype=np.int64) * nkvb
        indices = np.tile(np.arange(nkvb), B * Gn)
    out = np.full((B, C, Hq, d), np.nan)
    if rows is None:
        rows = [(b, p, h) for b in range(B) for h in range(Hq) for p in range(C)]
    for (b, p, h) in rows:
        g = h // E
        allowed = allowed_from_tables(indptr, indices, b, g, Gn, P, p, bs, L)
        kv = kv_head_of(h, Hq, Hkv)
        out[b, p, h] = masked_attention_row(q[b, p, h], k[b, kv], v[b, kv], allowed, scale)
    return out


def expand_tables_to_mask(indptr, indices, B: int, Hq: int, E: int, C: int, P: int, bs: int) -> np.ndarray:
    """q-uniform expansion of the block tables into a 2D per-(b,h,i) mask ("q-uniform
    expansion of table"; "the same unioned block mask"): Mq[b,h,i,j] = [j in T[b, h//E]]
    for every q-block i, restricted to the causal-valid tiles j <= pb + i (SPEC.md:441 pre:
    "mask causal-consistent")."""
    nqb, nkvb, pb, _ = geometry(C, P, bs)
    Gn = Hq // E
    Mq = np.zeros((B, Hq, nqb, nkvb), dtype=bool)
    for b in range(B):
        for h in range(Hq):
            r = b * Gn + h // E
            for j in indices[indptr[r]:indptr[r + 1]]:
                for i in range(nqb):
                    if causal_valid(i, int(j), pb):
                        Mq[b, h, i, j] = True
    return Mq


def block_sparse_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, P: int, bs: int,
                           mask: np.ndarray, sm_scale: Optional[float] = None, rows=None) -> np.ndarray:
    """Block-sparse execution of a 2D mask (the Fig. 7(c) baseline executor: "executes
    this mask directly with a block-sparse kernel"; SPEC.md:440-449 exec_block_sparse): query p of
    q-block i = p // bs under head h attends the tokens of the blocks {j : mask[b,h,i,j]} that are
    causally visible, t <= P + p. Per-query-block rows, so the value differs from
    the table executors unless the mask is q-uniform. An empty row raises.
    Returns [B, C, Hq, d] float64 (`rows` as in paged_attention)."""
    B, C, Hq, d = q.shape
    _, Hkv, L, _ = k.shape
    nqb, nkvb, pb, L2 = geometry(C, P, bs)
    assert L == L2 and mask.shape == (B, Hq, nqb, nkvb)
    scale = 1.0 / math.sqrt(d) if sm_scale is None else float(sm_scale)
    out = np.full((B, C, Hq, d), np.nan)
    if rows is None:
        rows = [(b, p, h) for b in range(B) for h in range(Hq) for p in range(C)]
    for (b, p, h) in rows:
        i = p // bs
        allowed = np.repeat(mask[b, h, i], bs)[:L].copy()
        allowed[P + p + 1:] = False
        kv = kv_head_of(h, Hq, Hkv)
        out[b, p, h] = masked_attention_row(q[b, p, h], k[b, kv], v[b, kv], allowed, scale)
    return out


def dense_causal_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, P: int,
                           sm_scale: Optional[float] = None) -> np.ndarray:
    """Dense causal chunked attention: query p sees t <= P + p. fp64.

    Written as plain matrix algebra per (b, h) (independent from the table path above).
    """
    B, C, Hq, d = q.shape
    _, Hkv, L, _ = k.shape
    scale = 1.0 / math.sqrt(d) if sm_scale is None else float(sm_scale)
    out = np.empty((B, C, Hq, d), np.float64)
    t = np.arange(L)[None, :]
    p = np.arange(C)[:, None]
    forbid = t > P + p
    for b in range(B):
        for h in range(Hq):
            kv = kv_head_of(h, Hq, Hkv)
            s = scale * (q[b, :, h].astype(np.float64) @ k[b, kv].astype(np.float64).T)
            s[forbid] = -np.inf
            s -= s.max(axis=1, keepdims=True)
            w = np.exp(s)
            w /= w.sum(axis=1, keepdims=True)
            out[b, :, h] = w @ v[b, kv].astype(np.float64)
    return out


# ----------------------------------------------------------------------------
# Whole chunk step (north_star (1)-(3))
# ----------------------------------------------------------------------------

def chunk_step(q, k, v, P: int, bs: int, alpha: float = 0.06, E: Optional[int] = None,
               sink: bool = True, sm_scale: Optional[float] = None, rows=None,
               scorer: str = "pooled", mask_in: Optional[np.ndarray] = None):
    """Estimator -> mask -> Q-block union -> intra-group union -> CSR -> attention.

    Returns dict(m, M, indptr, indices, O). PAPER.md:165-175 (§3.1 pipeline).
    """
    B, C, Hq, d = q.shape
    Hkv = k.shape[1]
    E = Hq // Hkv if E is None else E
    nqb, nkvb, pb, L = geometry(C, P, bs)
    m = None
    if mask_in is None:
        if scorer == "pooled":
            m = block_scores_pooled(q, k, P, bs, sm_scale)
        else:
            m = block_scores_exact(q, k, P, bs, sm_scale)
        M = threshold_mask(m, alpha, C, P, bs, sink)
    else:
        M = mask_in
    indptr, indices = tables_from_mask(M, E, pb)
    O = paged_attention(q, k, v, P, bs, indptr, indices, E, sm_scale, rows)
    return {"m": m, "M": M, "indptr": indptr, "indices": indices, "O": O}


def attention_flops(indptr, indices, C: int, P: int, bs: int, E: int, d: int) -> int:
    """Algorithmic FLOPs = 4*d*sum_{b,h} sum_p |A(p)| (exact causal pairs on tabled blocks;
    DESIGN.md "Algorithmic work"). Multiply-add = 2 FLOP."""
    L = P + C
    p = np.arange(C)
    total = 0
    for r in range(len(indptr) - 1):
        for j in indices[indptr[r]:indptr[r + 1]]:
            lo, hi = int(j) * bs, min((int(j) + 1) * bs, L)
            total += int(np.clip(np.minimum(hi, P + p + 1) - lo, 0, None).sum())
    return 4 * d * E * total
