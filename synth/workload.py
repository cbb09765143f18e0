"""Seeded synthetic inputs for the CompactAttention chunked-prefill hot path.

This module is shared by the oracle side (tests, bench cpu_baseline) and the
CUDA side (tests, bench, smoke). It holds NONE of the method's arithmetic: it
only draws Q/K/V tensors, random masks and page tables. Everything it returns
is bf16-representable float32 (so the fp64 oracle and the bf16 GPU path see
bit-identical input values).

Workload recipe: LLaMA-3.1-8B-shaped
Q/K/V (PAPER.md:262-263 names the model; 32 q heads / 8 KV heads / d=128 are its
public shape) with N(0,1) background and planted "needle" KV blocks, so the
estimator's masks are non-trivial (BASELINE.json north_star: "random data, with
planted high-score 'needle' blocks").
  * per (b, KV group) an orthonormal topic basis U (d x 3E, E = Hq/Hkv: 12 topics for GQA 4);
  * background q, k projected onto U-perp (no topic cross-talk), v ~ N(0,1);
  * n_N = round(rho * (pb_max - 1)) needle blocks drawn without replacement
    from prefix blocks [1, pb_max); each gets a topic c and all its keys get
    +beta_k * u_c;
  * query head h (local index hl within its group) has topic pool
    {(3*hl + t) mod 3E : t < 6}; each (h, q-block) draws s=4 pool topics and all
    its queries get +beta_q * sum u_c (for GQA 8 the two 4-head sub-groups cover
    overlapping but different topic sets, so sub-KV-group union keeps fewer blocks);
  * beta_q * beta_k / sqrt(d) = 6 (needle pooled logit ~ 6 vs background ~0.3).
Variant "qdiverse" (NEXT-4 chunk-size sweep): 64 topics per group, head
pools of 32 topics offset by 16 per head, 2 topics per q-block. A q-block then sees few topics, so
the Q-block union (and the group union) keeps more needles the more q-blocks a chunk has: the
post-union density grows with the chunk size, the effect PAPER.md:644-645 names ("larger chunks
increase Q-block union within each chunk, reducing effective sparsity"). Expected coverage of the
group's topics after the union of nqb q-blocks: 1 - (15/16)^(2 nqb).
Random numbers come from numpy Philox keyed by (seed, tensor, b, head, chunk), so
any slice (one KV head for one rank, one chunk's Q) regenerates identically.
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import Optional

import numpy as np

N_TOPICS = 12
TOPICS_PER_POOL = 6
TOPICS_PER_QBLOCK = 4
LOGIT_GAP = 6.0  # beta_q * beta_k / sqrt(d)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    batch: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    block_size: int
    context: int  # total tokens after the final chunk (L of the final chunk)
    chunk: int  # chunk length C

    @property
    def group_size(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def num_chunks(self) -> int:
        return -(-self.context // self.chunk)

    def chunk_geometry(self, chunk_index: Optional[int] = None):
        """(P, C, L) of chunk `chunk_index` (default: the final chunk)."""
        t = self.num_chunks - 1 if chunk_index is None else chunk_index
        P = t * self.chunk
        C = min(self.chunk, self.context - P)
        return P, C, P + C


# BASELINE.json "configs" (index 0..4). configs[0] is the oracle-sized case.
CONFIGS = {
    "tiny": Config("tiny", 1, 8, 2, 64, 16, 512, 64),
    "llama8b_32k": Config("llama8b_32k", 1, 32, 8, 128, 128, 32768, 2048),
    "llama8b_128k": Config("llama8b_128k", 1, 32, 8, 128, 128, 131072, 4096),
    "llama8b_64k_b4": Config("llama8b_64k_b4", 4, 32, 8, 128, 128, 65536, 2048),
    # NEXT-2: GQA 8:1 (Qwen3-30B-A3B attention shape: 32 q / 4 KV heads, d=128;
    # PAPER.md:673-699), run with sub-KV-group union (exec_group_size=4)
    "qwen3_30b_128k": Config("qwen3_30b_128k", 1, 32, 4, 128, 128, 131072, 4096),
}


def _key(seed: int, *parts) -> np.random.Generator:
    h = hashlib.blake2b(repr((int(seed),) + tuple(parts)).encode(), digest_size=16).digest()
    k0 = int.from_bytes(h[:8], "little")
    k1 = int.from_bytes(h[8:], "little")
    return np.random.Generator(np.random.Philox(key=[k0, k1]))


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return (u.astype(np.uint32)).view(np.float32)


# per variant: topics per group, topics per head pool, pool offset between heads, topics per q-block
VARIANTS = {"base": None, "qdiverse": (64, 32, 16, 2)}


def n_topics(cfg: "Config", variant: str = "base") -> int:
    if variant != "base":
        return VARIANTS[variant][0]
    return 3 * cfg.group_size if cfg.group_size > 4 else N_TOPICS


def _pool(cfg: "Config", hl: int, variant: str):
    """Topic pool of query head hl (local index in its group) and the number drawn per q-block."""
    if variant != "base":
        nt, size, stride, per = VARIANTS[variant]
        return [(stride * hl + s) % nt for s in range(size)], per
    nt = n_topics(cfg)
    return [(3 * hl + s) % nt for s in range(TOPICS_PER_POOL)], TOPICS_PER_QBLOCK


def _topics(seed: int, b: int, g: int, d: int, nt: int = N_TOPICS) -> np.ndarray:
    rng = _key(seed, "topics", b, g) if nt == N_TOPICS else _key(seed, "topics", b, g, nt)
    a = rng.standard_normal((d, nt))
    qmat, _ = np.linalg.qr(a)
    return qmat.astype(np.float32)  # d x nt, orthonormal columns


def needle_plan(cfg: Config, seed: int, rho: float, b: int, g: int, variant: str = "base"):
    """Needle blocks (ascending) and their topics for group (b, g)."""
    bs = cfg.block_size
    pb_max = (cfg.context - cfg.chunk) // bs if cfg.context > cfg.chunk else 0
    n_cand = max(pb_max - 1, 0)
    n_n = int(round(rho * n_cand))
    rng = _key(seed, "plan", b, g)
    blocks = np.sort(rng.choice(np.arange(1, pb_max), size=n_n, replace=False)) if n_n > 0 else np.zeros(0, np.int64)
    if variant == "base":
        topics = rng.integers(0, n_topics(cfg, variant), size=n_n)
    else:  # balanced: every topic owns floor or ceil(n_n / T) needles (no q-block without a needle)
        nt = n_topics(cfg, variant)
        topics = rng.permutation(np.arange(n_n) % nt) if n_n > 0 else np.zeros(0, np.int64)
    return blocks, topics


def _betas(d: int):
    beta = math.sqrt(LOGIT_GAP * math.sqrt(d))
    return beta, beta


def make_kv(cfg: Config, seed: int, rho: float = 0.30, length: Optional[int] = None,
            kv_heads: Optional[range] = None, needles: bool = True, graded: bool = False,
            variant: str = "base"):
    """Logical flat K, V [B, Hkv_sel, L, d] float32 (bf16-valued).

    graded=True (alpha-sweep workload): needle j's key boost is scaled by
    its own gain ~ U(0.1, 1), so the needles' pooled-logit gaps spread over ~0.6..6 nats and the
    threshold alpha decides how many of them are kept."""
    L = cfg.context if length is None else length
    d = cfg.head_dim
    heads = range(cfg.num_kv_heads) if kv_heads is None else kv_heads
    k = np.empty((cfg.batch, len(heads), L, d), np.float32)
    v = np.empty_like(k)
    _, beta_k = _betas(d)
    for b in range(cfg.batch):
        for hi, g in enumerate(heads):
            rng = _key(seed, "kv", b, g)
            kk = rng.standard_normal((L, d), dtype=np.float32)
            vv = rng.standard_normal((L, d), dtype=np.float32)
            if needles:
                U = _topics(seed, b, g, d, n_topics(cfg, variant))
                kk -= (kk @ U) @ U.T
                blocks, topics = needle_plan(cfg, seed, rho, b, g, variant)
                gains = (_key(seed, "grade", b, g).uniform(0.1, 1.0, size=len(blocks)) if graded
                         else np.ones(len(blocks)))
                bs = cfg.block_size
                for j, c, gn in zip(blocks, topics, gains):
                    lo, hi_ = j * bs, min((j + 1) * bs, L)
                    if lo < L:
                        kk[lo:hi_] += (gn * beta_k) * U[:, c]
            k[b, hi] = round_bf16(kk)
            v[b, hi] = round_bf16(vv)
    return k, v


def make_q(cfg: Config, seed: int, chunk_index: Optional[int] = None,
           q_heads: Optional[range] = None, needles: bool = True, variant: str = "base"):
    """Q of one chunk, [B, C, Hq_sel, d] float32 (bf16-valued)."""
    P, C, _ = cfg.chunk_geometry(chunk_index)
    t = P // cfg.chunk
    d, bs, E = cfg.head_dim, cfg.block_size, cfg.group_size
    heads = range(cfg.num_q_heads) if q_heads is None else q_heads
    q = np.empty((cfg.batch, C, len(heads), d), np.float32)
    beta_q, _ = _betas(d)
    for b in range(cfg.batch):
        for hi, h in enumerate(heads):
            rng = _key(seed, "q", b, h, t)
            qq = rng.standard_normal((C, d), dtype=np.float32)
            if needles:
                g, hl = h // E, h % E
                U = _topics(seed, b, g, d, n_topics(cfg, variant))
                qq -= (qq @ U) @ U.T
                pool, per = _pool(cfg, hl, variant)
                nqb = -(-C // bs)
                for i in range(nqb):
                    sel = rng.choice(pool, size=per, replace=False)
                    boost = beta_q * U[:, sel].sum(axis=1)
                    qq[i * bs:min((i + 1) * bs, C)] += boost
            q[b, :, hi] = round_bf16(qq)
    return q


def random_qkv(B: int, Hq: int, Hkv: int, d: int, C: int, L: int, seed: int, scale: float = 1.0):
    """Plain N(0, scale^2) Q [B,C,Hq,d] and K/V [B,Hkv,L,d], bf16-valued float32."""
    rng = _key(seed, "random_qkv", B, Hq, Hkv, d, C, L)
    q = round_bf16(scale * rng.standard_normal((B, C, Hq, d), dtype=np.float32))
    k = round_bf16(scale * rng.standard_normal((B, Hkv, L, d), dtype=np.float32))
    v = round_bf16(rng.standard_normal((B, Hkv, L, d), dtype=np.float32))
    return q, k, v


def random_block_mask(B: int, Hq: int, nqb: int, nkvb: int, density: float, seed: int) -> np.ndarray:
    """Random boolean block mask [B, Hq, nqb, nkvb] (no structure imposed)."""
    rng = _key(seed, "mask", B, Hq, nqb, nkvb)
    return rng.random((B, Hq, nqb, nkvb)) < density


def page_layout(B: int, nblocks: int, seed: int, extra_pages: int = 3, shuffle: bool = True):
    """Physical page assignment: page_table [B, nblocks] int32 into a pool of
    B*nblocks+extra_pages pages (random permutation unless shuffle=False)."""
    n = B * nblocks + extra_pages
    if shuffle:
        perm = _key(seed, "pages", B, nblocks).permutation(n)[: B * nblocks]
    else:
        perm = np.arange(B * nblocks)
    return perm.reshape(B, nblocks).astype(np.int32), n


def to_pool(x_flat: np.ndarray, page_table: np.ndarray, num_pages: int, bs: int) -> np.ndarray:
    """Scatter logical [B,Hkv,L,d] into a zero-initialised pool [num_pages,Hkv,bs,d]."""
    B, H, L, d = x_flat.shape
    pool = np.zeros((num_pages, H, bs, d), x_flat.dtype)
    nb = -(-L // bs)
    for b in range(B):
        for j in range(nb):
            lo, hi = j * bs, min((j + 1) * bs, L)
            pool[page_table[b, j], :, : hi - lo] = x_flat[b, :, lo:hi]
    return pool
