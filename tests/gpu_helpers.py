"""Helpers for the GPU parity tests: seeded synth inputs -> device tensors for libcpa."""
from __future__ import annotations

import numpy as np
import torch

import paper_2605_16839_b200 as cpa
from synth.workload import page_layout, to_pool


def to_dev_bf16(x: np.ndarray) -> torch.Tensor:
    # x is bf16-valued float32: the conversion is exact
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(torch.bfloat16)


class Case:
    """One chunk: q [B,C,Hq,d], logical k/v [B,Hkv,L,d] (numpy, bf16-valued) + paged device copy."""

    def __init__(self, q, k, v, P, bs, alpha=0.06, E=0, sink=True, seed=0, shuffle=True, flags=0,
                 extra_blocks=0):
        self.q, self.k, self.v = q, k, v
        B, C, Hq, d = q.shape
        Hkv, L = k.shape[1], k.shape[2]
        assert L == P + C
        self.P, self.C, self.L, self.bs = P, C, L, bs
        nkvb = -(-L // bs)
        self.page_table, self.num_pages = page_layout(B, nkvb + extra_blocks, seed, shuffle=shuffle)
        self.k_pool = to_pool(k, self.page_table, self.num_pages, bs)
        self.v_pool = to_pool(v, self.page_table, self.num_pages, bs)
        self.dq = to_dev_bf16(q)
        self.cache = cpa.PagedKVCache(to_dev_bf16(self.k_pool), to_dev_bf16(self.v_pool),
                                      torch.from_numpy(self.page_table).to("cuda"))
        self.params = cpa.make_params(B, Hq, Hkv, d, bs, C, P, alpha=alpha, exec_group_size=E, sink=sink,
                                      flags=flags)
        self.E = E or Hq // Hkv

    def out(self, f32=True):
        B, C, Hq, d = self.q.shape
        return torch.empty(B, C, Hq, d, dtype=torch.float32 if f32 else torch.bfloat16, device="cuda")


def tables_to_numpy(t: cpa.BlockTables):
    ip = t.kv_indptr.cpu().numpy()
    ix = t.kv_indices.cpu().numpy()[: ip[-1]]
    return ip, ix


def scores_to_bhij(scores: torch.Tensor, p: cpa.Params) -> np.ndarray:
    """[B,Gn,nkvb,Rpad] -> [B,Hq,nqb,nkvb] (row r = hl*nqb + i)."""
    nqb, nkvb, pb, Gn, nwords, Rpad = cpa.geometry(p)
    E = p.num_q_heads // Gn
    s = scores.cpu().numpy()[..., : E * nqb]  # [B,Gn,nkvb,E*nqb]
    s = s.reshape(p.batch, Gn, nkvb, E, nqb).transpose(0, 1, 3, 4, 2)
    return s.reshape(p.batch, Gn * E, nqb, nkvb)


def rowmax_to_bhi(row_max: torch.Tensor, p: cpa.Params) -> np.ndarray:
    nqb, nkvb, pb, Gn, nwords, Rpad = cpa.geometry(p)
    E = p.num_q_heads // Gn
    r = row_max.cpu().numpy()[..., : E * nqb]
    return r.reshape(p.batch, Gn, E, nqb).reshape(p.batch, Gn * E, nqb)


def mask_to_bits(M: np.ndarray) -> np.ndarray:
    """bool [B,Hq,nqb,nkvb] -> int32 words [B,Hq,nqb,nwords] (bit j%32 of word j/32)."""
    B, Hq, nqb, nkvb = M.shape
    nwords = -(-nkvb // 32)
    pad = np.zeros((B, Hq, nqb, nwords * 32), bool)
    pad[..., :nkvb] = M
    w = (pad.reshape(B, Hq, nqb, nwords, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)).sum(-1)
    return w.astype(np.uint32).view(np.int32)


def bits_to_mask(bits: np.ndarray, nkvb: int) -> np.ndarray:
    b = bits.view(np.uint32).astype(np.uint64)
    B, Hq, nqb, nwords = b.shape
    M = ((b[..., None] >> np.arange(32, dtype=np.uint64)) & 1).astype(bool).reshape(B, Hq, nqb, nwords * 32)
    return M[..., :nkvb]


def rel_err(gpu: np.ndarray, ref: np.ndarray):
    """max |delta| / RMS(ref) over finite reference entries (north_star tolerance form)."""
    m = np.isfinite(ref)
    rms = float(np.sqrt(np.mean(ref[m] ** 2)))
    return float(np.abs(gpu[m] - ref[m]).max()) / rms
