"""paper_2605_16839_b200 -- B200-native CompactAttention chunked-prefill hot path.

Thin Python binding over libcpa.so (include/cpa.h). Argument marshalling only: every step of
the path (estimator, masks, unions, CSR tables, paged attention, append) runs in the sm_100a
kernels of csrc/. PyTorch supplies device memory and streams. There is no CPU fallback: if the
native library is missing or the device is not sm_100 every call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import torch

__all__ = [
    "CpaError", "Params", "PagedKVCache", "BlockTables", "lib", "make_params", "workspace_bytes",
    "alloc_tables", "build_tables", "paged_attention", "chunk_step", "append_kv", "prepare_chunk", "last_launch_count",
    "paged_attention_copy", "block_sparse_attention", "expand_tables", "PeerOut", "chunk_step_peer",
    "paged_attention_peer", "peer_barrier", "HostChunkStream",
    "F_SINK", "F_MASK_IN", "F_MASK_OUT", "F_SCORES_OUT", "F_OUT_F32", "F_EXACT_SCORES", "F_P_BF16", "F_NO_2CTA", "F_NO_PERSIST", "F_PERSIST", "F_V_F16", "F_NO_PDL", "F_ATTN_RS", "F_ATTN_KS4", "EXPORTED_SYMBOLS",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CPA_LIB_PATH") or os.path.join(_HERE, "libcpa.so")  # override: dev A/B builds

F_SINK, F_MASK_IN, F_MASK_OUT, F_SCORES_OUT, F_OUT_F32, F_EXACT_SCORES, F_P_BF16, F_NO_2CTA = 1, 2, 4, 8, 16, 32, 256, 512
F_NO_PERSIST, F_PERSIST, F_V_F16, F_NO_PDL, F_ATTN_RS = 1024, 2048, 4096, 8192, 16384
F_ATTN_KS4 = 65536
STATUS = ["CPA_OK", "CPA_ERR_NULL", "CPA_ERR_SHAPE", "CPA_ERR_UNSUPPORTED", "CPA_ERR_MISALIGNED",
          "CPA_ERR_ALPHA", "CPA_ERR_WORKSPACE", "CPA_ERR_CAPACITY", "CPA_ERR_CUDA"]
EXPORTED_SYMBOLS = ["cpa_workspace_bytes", "cpa_build_tables", "cpa_paged_attention", "cpa_chunk_step",
                    "cpa_append_kv", "cpa_prepare_chunk", "cpa_copy_workspace_bytes", "cpa_paged_attention_copy",
                    "cpa_block_sparse_attention", "cpa_expand_tables", "cpa_chunk_step_peer",
                    "cpa_paged_attention_peer", "cpa_peer_barrier", "cpa_status_string", "cpa_last_error", "cpa_version", "cpa_last_launch_count"]


class CpaError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{name}: {detail}")


class Params(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("block_size", ctypes.c_int32), ("exec_group_size", ctypes.c_int32),
                ("chunk_len", ctypes.c_int32), ("prefix_len", ctypes.c_int32), ("alpha", ctypes.c_float),
                ("sm_scale", ctypes.c_float), ("flags", ctypes.c_uint32), ("q_token_stride", ctypes.c_int64)]


class _Cache(ctypes.Structure):
    _fields_ = [("k_pages", ctypes.c_void_p), ("v_pages", ctypes.c_void_p), ("page_stride", ctypes.c_int64),
                ("head_stride", ctypes.c_int64), ("page_table", ctypes.c_void_p),
                ("max_blocks_per_seq", ctypes.c_int32), ("num_pages", ctypes.c_int32)]


class _Tables(ctypes.Structure):
    _fields_ = [("kv_indptr", ctypes.c_void_p), ("kv_indices", ctypes.c_void_p), ("capacity", ctypes.c_int64),
                ("mask_bits", ctypes.c_void_p), ("scores", ctypes.c_void_p), ("row_max", ctypes.c_void_p),
                ("dev_status", ctypes.c_void_p)]


class _PeerOut(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("peer_out", ctypes.POINTER(ctypes.c_void_p)),
                ("out_token_stride", ctypes.c_int64), ("peer_signal", ctypes.POINTER(ctypes.c_void_p)),
                ("epoch", ctypes.c_uint32), ("timeout_ms", ctypes.c_uint32), ("dev_status", ctypes.c_void_p)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libcpa.so (in-tree). Raises if it is missing -- there is no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"native library {LIB_PATH} is missing; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32 = ctypes.c_void_p, ctypes.c_int
        L.cpa_workspace_bytes.argtypes = [ctypes.POINTER(Params)]
        L.cpa_workspace_bytes.restype = ctypes.c_size_t
        L.cpa_build_tables.argtypes = [ctypes.POINTER(Params), vp, ctypes.POINTER(_Cache), ctypes.POINTER(_Tables),
                                       vp, ctypes.c_size_t, vp]
        L.cpa_paged_attention.argtypes = [ctypes.POINTER(Params), vp, ctypes.POINTER(_Cache),
                                          ctypes.POINTER(_Tables), vp, vp, ctypes.c_size_t, vp]
        L.cpa_chunk_step.argtypes = [ctypes.POINTER(Params), vp, vp, vp, ctypes.POINTER(_Cache),
                                     ctypes.POINTER(_Tables), vp, vp, ctypes.c_size_t, vp]
        L.cpa_append_kv.argtypes = [ctypes.POINTER(Params), vp, vp, ctypes.POINTER(_Cache), vp]
        L.cpa_prepare_chunk.argtypes = [ctypes.POINTER(Params), vp, vp, vp, ctypes.POINTER(_Cache),
                                        ctypes.POINTER(_Tables), vp, ctypes.c_size_t, vp]
        L.cpa_copy_workspace_bytes.argtypes = [ctypes.POINTER(Params)]
        L.cpa_copy_workspace_bytes.restype = ctypes.c_size_t
        L.cpa_paged_attention_copy.argtypes = [ctypes.POINTER(Params), vp, ctypes.POINTER(_Cache),
                                               ctypes.POINTER(_Tables), vp, vp, ctypes.c_size_t, vp]
        L.cpa_paged_attention_copy.restype = i32
        L.cpa_block_sparse_attention.argtypes = [ctypes.POINTER(Params), vp, ctypes.POINTER(_Cache), vp, vp, vp,
                                                 ctypes.c_size_t, vp]
        L.cpa_block_sparse_attention.restype = i32
        L.cpa_expand_tables.argtypes = [ctypes.POINTER(Params), ctypes.POINTER(_Tables), vp, vp]
        L.cpa_expand_tables.restype = i32
        L.cpa_chunk_step_peer.argtypes = [ctypes.POINTER(Params), vp, vp, vp, ctypes.POINTER(_Cache),
                                          ctypes.POINTER(_Tables), ctypes.POINTER(_PeerOut), vp, ctypes.c_size_t, vp]
        L.cpa_peer_barrier.argtypes = [ctypes.POINTER(_PeerOut), vp]
        L.cpa_paged_attention_peer.argtypes = [ctypes.POINTER(Params), vp, ctypes.POINTER(_Cache),
                                               ctypes.POINTER(_Tables), ctypes.POINTER(_PeerOut), vp,
                                               ctypes.c_size_t, vp]
        for f in (L.cpa_build_tables, L.cpa_paged_attention, L.cpa_chunk_step, L.cpa_append_kv, L.cpa_prepare_chunk,
                  L.cpa_chunk_step_peer, L.cpa_peer_barrier, L.cpa_paged_attention_peer):
            f.restype = i32
        L.cpa_status_string.argtypes = [i32]
        L.cpa_status_string.restype = ctypes.c_char_p
        L.cpa_last_error.restype = ctypes.c_char_p
        L.cpa_version.restype = i32
        L.cpa_last_launch_count.restype = i32
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise CpaError(status, lib().cpa_last_error().decode())


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def make_params(batch: int, num_q_heads: int, num_kv_heads: int, head_dim: int, block_size: int,
                chunk_len: int, prefix_len: int, alpha: float = 0.06, exec_group_size: int = 0,
                sink: bool = True, flags: int = 0, sm_scale: float = 0.0, q_token_stride: int = 0) -> Params:
    return Params(batch, num_q_heads, num_kv_heads, head_dim, block_size, exec_group_size, chunk_len,
                  prefix_len, alpha, sm_scale, flags | (F_SINK if sink else 0), q_token_stride)


def geometry(p: Params):
    """(nqb, nkvb, pb, Gn, nwords, Rpad) -- plain integer bookkeeping from the header's notation."""
    bs = p.block_size
    E = p.exec_group_size or p.num_q_heads // p.num_kv_heads
    nqb = -(-p.chunk_len // bs)
    nkvb = -(-(p.prefix_len + p.chunk_len) // bs)
    Gn = p.num_q_heads // E
    return nqb, nkvb, p.prefix_len // bs, Gn, -(-nkvb // 32), 128 * (-(-(E * nqb) // 128))


def workspace_bytes(p: Params) -> int:
    return int(lib().cpa_workspace_bytes(ctypes.byref(p)))


@dataclass
class PagedKVCache:
    """K/V page pools (bf16, each (page, kv head) a contiguous [bs, d] region) + int32 page table
    [B, max_blocks_per_seq]. Strides are in elements (0 => pool laid out [pages, Hkv, bs, d])."""
    k_pages: torch.Tensor
    v_pages: torch.Tensor
    page_table: torch.Tensor
    page_stride: int = 0
    head_stride: int = 0
    num_pages: int = 0  # 0 => k_pages.shape[0] (only valid for the default [pages, Hkv, bs, d] pool)

    def _c(self) -> _Cache:
        assert self.k_pages.dtype == torch.bfloat16 and self.v_pages.dtype in (torch.bfloat16, torch.float16)
        assert self.page_table.dtype == torch.int32 and self.page_table.is_contiguous()
        if self.num_pages:
            num_pages = self.num_pages
        elif self.page_stride == 0 and self.head_stride == 0:
            num_pages = self.k_pages.shape[0]
        else:
            raise ValueError("PagedKVCache with explicit strides needs num_pages (the page index range of the pool)")
        return _Cache(_ptr(self.k_pages), _ptr(self.v_pages), self.page_stride, self.head_stride,
                      _ptr(self.page_table), self.page_table.shape[-1], num_pages)

    def _check_v(self, p: "Params"):
        """The V pool dtype must match CPA_F_V_F16 (fp16 pool <=> flag), else results are garbage."""
        if (self.v_pages.dtype == torch.float16) != bool(p.flags & F_V_F16):
            raise ValueError(f"v_pages dtype {self.v_pages.dtype} does not match CPA_F_V_F16 "
                             f"({'set' if p.flags & F_V_F16 else 'unset'})")


@dataclass
class BlockTables:
    """CSR block tables T[b,g] + optional debug outputs."""
    kv_indptr: torch.Tensor
    kv_indices: torch.Tensor
    mask_bits: Optional[torch.Tensor] = None
    scores: Optional[torch.Tensor] = None
    row_max: Optional[torch.Tensor] = None
    dev_status: Optional[torch.Tensor] = None

    def _c(self) -> _Tables:
        return _Tables(_ptr(self.kv_indptr), _ptr(self.kv_indices), self.kv_indices.numel(),
                       _ptr(self.mask_bits), _ptr(self.scores), _ptr(self.row_max), _ptr(self.dev_status))


def alloc_tables(p: Params, device="cuda", mask: bool = False, scores: bool = False,
                 status: bool = False) -> BlockTables:
    nqb, nkvb, pb, Gn, nwords, Rpad = geometry(p)
    B = p.batch
    t = BlockTables(torch.empty(B * Gn + 1, dtype=torch.int32, device=device),
                    torch.empty(B * Gn * nkvb, dtype=torch.int32, device=device))
    if mask:
        t.mask_bits = torch.zeros(B, p.num_q_heads, nqb, nwords, dtype=torch.int32, device=device)
    if scores:
        t.scores = torch.empty(B, Gn, nkvb, Rpad, dtype=torch.float32, device=device)
        t.row_max = torch.empty(B, Gn, Rpad, dtype=torch.float32, device=device)
    if status:
        t.dev_status = torch.zeros(1, dtype=torch.int32, device=device)
    return t


def _ws(p: Params, workspace: Optional[torch.Tensor], device, stream=None) -> torch.Tensor:
    need = workspace_bytes(p)
    if workspace is None:
        workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=device)
        if isinstance(stream, torch.cuda.Stream):  # freed on return: keep it until `stream` is done with it
            workspace.record_stream(stream)
    return workspace


def build_tables(p: Params, q: torch.Tensor, cache: PagedKVCache, tables: BlockTables,
                 workspace: Optional[torch.Tensor] = None, stream=None) -> BlockTables:
    ws = _ws(p, workspace, q.device if q is not None else cache.k_pages.device, stream)
    c, t = cache._c(), tables._c()
    _check(lib().cpa_build_tables(ctypes.byref(p), _ptr(q), ctypes.byref(c), ctypes.byref(t),
                                  _ptr(ws), ws.numel(), _stream(stream)))
    return tables


def paged_attention(p: Params, q: torch.Tensor, cache: PagedKVCache, tables: Optional[BlockTables],
                    out: torch.Tensor, workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    ws = _ws(p, workspace, q.device, stream)
    cache._check_v(p)
    c = cache._c()
    t = tables._c() if tables is not None else None
    _check(lib().cpa_paged_attention(ctypes.byref(p), _ptr(q), ctypes.byref(c),
                                     ctypes.byref(t) if t is not None else None, _ptr(out), _ptr(ws),
                                     ws.numel(), _stream(stream)))
    return out


def chunk_step(p: Params, q: torch.Tensor, cache: PagedKVCache, tables: BlockTables, out: torch.Tensor,
               k_chunk: Optional[torch.Tensor] = None, v_chunk: Optional[torch.Tensor] = None,
               workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    ws = _ws(p, workspace, q.device, stream)
    cache._check_v(p)
    c, t = cache._c(), tables._c()
    _check(lib().cpa_chunk_step(ctypes.byref(p), _ptr(q), _ptr(k_chunk), _ptr(v_chunk), ctypes.byref(c),
                                ctypes.byref(t), _ptr(out), _ptr(ws), ws.numel(), _stream(stream)))
    return out


def prepare_chunk(p: Params, q: torch.Tensor, cache: PagedKVCache, tables: BlockTables,
                  k_chunk: Optional[torch.Tensor] = None, v_chunk: Optional[torch.Tensor] = None,
                  workspace: Optional[torch.Tensor] = None, stream=None) -> BlockTables:
    """cpa_prepare_chunk: append (optional) + estimator + tables, the first half of chunk_step."""
    ws = _ws(p, workspace, q.device, stream)
    cache._check_v(p)
    c, t = cache._c(), tables._c()
    _check(lib().cpa_prepare_chunk(ctypes.byref(p), _ptr(q), _ptr(k_chunk), _ptr(v_chunk), ctypes.byref(c),
                                   ctypes.byref(t), _ptr(ws), ws.numel(), _stream(stream)))
    return tables


class PeerOut:
    """Peer mappings for cpa_chunk_step_peer (see cpa.h): W gathered output buffers [B, C, W*Hq, d]
    and W uint32 signal pads, given as raw device addresses valid in this process (torch symmetric
    memory buffer_ptrs, CUDA IPC, or -- in single-GPU tests -- plain tensors on one device). Epochs
    are kept on the device (cpa.h), so a captured CUDA graph of the step can be replayed."""

    def __init__(self, world: int, rank: int, out_ptrs, signal_ptrs, out_token_stride: int = 0,
                 timeout_ms: int = 0, dev_status: Optional[torch.Tensor] = None):
        assert len(out_ptrs) == world and len(signal_ptrs) == world
        self._outs = (ctypes.c_void_p * world)(*[int(x) for x in out_ptrs])
        self._sigs = (ctypes.c_void_p * world)(*[int(x) for x in signal_ptrs])
        self.world, self.rank, self.epoch = world, rank, 0
        self.out_token_stride, self.timeout_ms, self.dev_status = out_token_stride, timeout_ms, dev_status

    def _next(self) -> _PeerOut:
        return _PeerOut(self.world, self.rank, self._outs, self.out_token_stride, self._sigs, 0,
                        self.timeout_ms, _ptr(self.dev_status))


def chunk_step_peer(p: Params, q: torch.Tensor, cache: PagedKVCache, tables: BlockTables, peers: PeerOut,
                    k_chunk: Optional[torch.Tensor] = None, v_chunk: Optional[torch.Tensor] = None,
                    workspace: Optional[torch.Tensor] = None, stream=None) -> None:
    """cpa_chunk_step with the head-output all-gather fused into the attention epilogue (cpa.h)."""
    ws = _ws(p, workspace, q.device, stream)
    cache._check_v(p)
    c, t, pr = cache._c(), tables._c(), peers._next()
    _check(lib().cpa_chunk_step_peer(ctypes.byref(p), _ptr(q), _ptr(k_chunk), _ptr(v_chunk), ctypes.byref(c),
                                     ctypes.byref(t), ctypes.byref(pr), _ptr(ws), ws.numel(), _stream(stream)))


def paged_attention_peer(p: Params, q: torch.Tensor, cache: PagedKVCache, tables: Optional[BlockTables],
                         peers: PeerOut, workspace: Optional[torch.Tensor] = None, stream=None) -> None:
    """cpa_paged_attention with the fused head-output all-gather + barrier (cpa.h)."""
    ws = _ws(p, workspace, q.device, stream)
    cache._check_v(p)
    c, pr = cache._c(), peers._next()
    t = tables._c() if tables is not None else None
    _check(lib().cpa_paged_attention_peer(ctypes.byref(p), _ptr(q), ctypes.byref(c),
                                          ctypes.byref(t) if t is not None else None, ctypes.byref(pr), _ptr(ws),
                                          ws.numel(), _stream(stream)))


def peer_barrier(peers: PeerOut, stream=None) -> None:
    pr = peers._next()
    _check(lib().cpa_peer_barrier(ctypes.byref(pr), _stream(stream)))


def append_kv(p: Params, k_chunk: torch.Tensor, v_chunk: torch.Tensor, cache: PagedKVCache, stream=None):
    cache._check_v(p)
    c = cache._c()
    _check(lib().cpa_append_kv(ctypes.byref(p), _ptr(k_chunk), _ptr(v_chunk), ctypes.byref(c), _stream(stream)))


def paged_attention_copy(p: Params, q: torch.Tensor, cache: PagedKVCache, tables: BlockTables,
                         out: torch.Tensor, workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """NEXT-3 ablation: gather the tabled pages into a compact pool, then attend (see cpa.h)."""
    need = int(lib().cpa_copy_workspace_bytes(ctypes.byref(p)))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=q.device)
    cache._check_v(p)
    c, t = cache._c(), tables._c()
    _check(lib().cpa_paged_attention_copy(ctypes.byref(p), _ptr(q), ctypes.byref(c), ctypes.byref(t), _ptr(out),
                                          _ptr(workspace), workspace.numel(), _stream(stream)))
    return out


def block_sparse_attention(p: Params, q: torch.Tensor, cache: PagedKVCache, mask_bits: torch.Tensor,
                           out: torch.Tensor, stream=None) -> torch.Tensor:
    """NEXT-3 ablation: execute a 2D per-(b,h,q-block) mask [B,Hq,nqb,nwords] directly (see cpa.h)."""
    cache._check_v(p)
    c = cache._c()
    _check(lib().cpa_block_sparse_attention(ctypes.byref(p), _ptr(q), ctypes.byref(c), _ptr(mask_bits), _ptr(out),
                                            None, 0, _stream(stream)))
    return out


def expand_tables(p: Params, tables: BlockTables, mask_bits: torch.Tensor, stream=None) -> torch.Tensor:
    """q-uniform expansion of the tables into a 2D mask [B,Hq,nqb,nwords] (see cpa.h)."""
    t = tables._c()
    _check(lib().cpa_expand_tables(ctypes.byref(p), ctypes.byref(t), _ptr(mask_bits), _stream(stream)))
    return mask_bits


class HostChunkStream:
    """Chunk steps fed from pinned HOST buffers, pipelined over three streams: the H2D copy of step
    i+1's inputs and the D2H copy of step i-1's output overlap step i's kernels (device staging is
    multi-buffered; the cache, tables and workspace are used in stream order on the compute stream).
    Plumbing only -- every step runs cpa_chunk_step (with graphs=True replayed from one captured CUDA
    graph per staging slot). Read a host output only after synchronize().

    Multi-GPU (peers = one PeerOut per slot, gathered = this rank's gathered buffer [B, C, W*Hq, d] of
    each slot): every step runs cpa_chunk_step_peer into its slot's gathered buffers on every rank, and
    the D2H reads this rank's head slice. Three slots, and step i starts only after this rank's D2H of
    step i-2 finished: any rank writing slot (i+1) % 3 at step i+1 has passed barrier i, so every rank
    has finished its D2H of step i-2 == the last reader of that slot (cpa.h reuse rule)."""

    def __init__(self, p: Params, cache: PagedKVCache, tables: BlockTables, q_shape, kv_shape,
                 workspace: Optional[torch.Tensor] = None, device="cuda", graphs: bool = False,
                 peers=None, gathered=None, rank: int = 0):
        self.p, self.cache, self.tables = p, cache, tables
        self.ws = workspace if workspace is not None else _ws(p, None, device)
        self.peers, self.gathered, self.rank = peers, gathered, rank
        self.n = 3 if peers is not None else 2
        if peers is not None:
            assert gathered is not None and len(peers) == self.n and len(gathered) == self.n
        bf = torch.bfloat16
        o_dtype = torch.float32 if p.flags & F_OUT_F32 else bf
        self.q = [torch.empty(q_shape, dtype=bf, device=device) for _ in range(self.n)]
        self.k = [torch.empty(kv_shape, dtype=bf, device=device) for _ in range(self.n)]
        self.v = [torch.empty(kv_shape, dtype=bf, device=device) for _ in range(self.n)]
        if peers is None:
            self.o = [torch.empty(q_shape, dtype=o_dtype, device=device) for _ in range(self.n)]
        else:
            hq = q_shape[2]
            self.o = [g[:, :, rank * hq:(rank + 1) * hq] for g in gathered]
        self.s_in, self.s_comp, self.s_out = (torch.cuda.Stream(device) for _ in range(3))
        self.ev_in = [torch.cuda.Event() for _ in range(self.n)]
        self.ev_comp = [torch.cuda.Event() for _ in range(self.n)]
        self.ev_out = [torch.cuda.Event() for _ in range(self.n)]
        self.i = 0
        self.graphs = None
        if graphs:  # one graph per slot: append + estimator + tables + attention on that slot's buffers
            self.graphs = []
            for s in range(self.n):
                with torch.cuda.stream(self.s_comp):
                    for _ in range(2):
                        self._step(s)
                self.s_comp.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.s_comp):
                    self._step(s)
                self.graphs.append(g)
            torch.cuda.synchronize()

    def _step(self, s: int, with_kv: bool = True, stream=None):
        k, v = (self.k[s], self.v[s]) if with_kv else (None, None)
        if self.peers is not None:
            chunk_step_peer(self.p, self.q[s], self.cache, self.tables, self.peers[s], k, v, workspace=self.ws,
                            stream=stream)
        else:
            chunk_step(self.p, self.q[s], self.cache, self.tables, self.o[s], k, v, workspace=self.ws, stream=stream)

    def submit(self, hq: torch.Tensor, ho: torch.Tensor, hk: Optional[torch.Tensor] = None,
               hv: Optional[torch.Tensor] = None) -> None:
        """Enqueue one chunk step: hq [B,C,Hq,d] (+ hk/hv [B,C,Hkv,d] to append) -> ho [B,C,Hq,d]."""
        s = self.i % self.n
        self.s_in.wait_event(self.ev_comp[s])        # step i-n has finished reading this slot
        with torch.cuda.stream(self.s_in):
            self.q[s].copy_(hq, non_blocking=True)
            if hk is not None:
                self.k[s].copy_(hk, non_blocking=True)
                self.v[s].copy_(hv, non_blocking=True)
            self.ev_in[s].record(self.s_in)
        self.s_comp.wait_event(self.ev_in[s])
        self.s_comp.wait_event(self.ev_out[s])       # D2H of step i-n has finished reading o[s]
        if self.peers is not None and self.i >= 2:
            self.s_comp.wait_event(self.ev_out[(self.i - 2) % self.n])  # cross-rank slot reuse (class doc)
        if self.graphs is not None:  # the captured step always appends the slot's K/V
            assert hk is not None, "graphs=True runs the step with the chunk's K/V"
            with torch.cuda.stream(self.s_comp):
                self.graphs[s].replay()
        else:
            self._step(s, hk is not None, stream=self.s_comp)
        self.ev_comp[s].record(self.s_comp)
        self.s_out.wait_event(self.ev_comp[s])
        with torch.cuda.stream(self.s_out):
            ho.copy_(self.o[s], non_blocking=True)
            self.ev_out[s].record(self.s_out)
        self.i += 1

    def synchronize(self) -> None:
        for st in (self.s_in, self.s_comp, self.s_out):
            st.synchronize()


def last_launch_count() -> int:
    return int(lib().cpa_last_launch_count())
