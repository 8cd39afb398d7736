"""ctypes binding of libbkv (include/bkv.h) over torch tensors.

Argument marshalling only: every step of the hot path runs in the CUDA kernels
of libbkv.so.  There is no CPU or PyTorch fallback -- if the library is missing
or the device is not a CUDA device, calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os
import threading
from dataclasses import dataclass

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libbkv.so")

BKV_DIR_FWD = 0   # RT: left -> right
BKV_DIR_REV = 1   # BE: right -> left


class BkvError(RuntimeError):
    pass


class _Pool(ctypes.Structure):
    _fields_ = [("k", ctypes.c_void_p), ("v", ctypes.c_void_p),
                ("num_blocks", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("block_size", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("stride_block", ctypes.c_int64), ("stride_head", ctypes.c_int64),
                ("stride_slot", ctypes.c_int64)]


class _Map(ctypes.Structure):
    _fields_ = [("block_tables", ctypes.c_void_p), ("bt_stride", ctypes.c_int32),
                ("dirs", ctypes.c_void_p), ("dir_row_stride", ctypes.c_int32),
                ("dir_col_stride", ctypes.c_int32), ("num_seqs", ctypes.c_int32),
                ("fills", ctypes.c_void_p), ("fill_row_stride", ctypes.c_int32),
                ("num_entries", ctypes.c_void_p)]


_lib = None
_lib_lock = threading.Lock()

EXPORTS = ("bkv_kv_append", "bkv_paged_decode_attention", "bkv_decode_workspace_size",
           "bkv_validate_layout_host", "bkv_status_string", "bkv_last_error", "bkv_version",
           "bkv_kv_checkpoint", "bkv_kv_restore", "bkv_paged_decode_attention_ex",
           "bkv_decode_step", "bkv_validate_block_map_host", "bkv_kv_append_checkpoint",
           "bkv_paged_prefill_attention", "bkv_decode_multi_out", "bkv_peer_barrier",
           "bkv_paged_mixed_attention")
BKV_FLAG_PDL = 1   # include/bkv.h: programmatic dependent launch (seq_lens not written by the previous kernel)
BKV_FLAG_KV_EARLY = 2   # planned decode: resident KV not written by the previous kernel either
BKV_FLAG_PEER_MULTICAST = 4   # peer_outs = [one NVLS multicast address] (multimem stores)


def lib():
    """Load libbkv.so (raises if it was not built -- no fallback path exists)."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise BkvError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
                L = ctypes.CDLL(LIB_PATH)
                P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
                L.bkv_kv_append.argtypes = [ctypes.POINTER(_Pool), ctypes.POINTER(_Map), P, P, i32, P, P, P, P]
                L.bkv_kv_append.restype = ctypes.c_int
                L.bkv_kv_append_checkpoint.argtypes = [ctypes.POINTER(_Pool), ctypes.POINTER(_Map), P, P, i32,
                                                       P, P, P, P, P, P, P]
                L.bkv_kv_append_checkpoint.restype = ctypes.c_int
                L.bkv_paged_decode_attention.argtypes = [
                    ctypes.POINTER(_Pool), ctypes.POINTER(_Map), P, i32, P, i64, i64, i32, ctypes.c_float,
                    P, i64, i64, P, ctypes.c_size_t, P]
                L.bkv_paged_decode_attention.restype = ctypes.c_int
                L.bkv_paged_decode_attention_ex.argtypes = [
                    ctypes.POINTER(_Pool), ctypes.POINTER(_Map), P, i32, P, i64, i64, i32, ctypes.c_float,
                    P, i64, i64, P, ctypes.c_size_t, ctypes.c_uint32, P]
                L.bkv_paged_decode_attention_ex.restype = ctypes.c_int
                L.bkv_decode_step.argtypes = [
                    ctypes.POINTER(_Pool), ctypes.POINTER(_Map), P, i32, P, P, P, i64, i64, i32,
                    ctypes.c_float, P, i64, i64, P, ctypes.c_size_t, ctypes.c_uint32, P]
                L.bkv_decode_step.restype = ctypes.c_int
                L.bkv_paged_prefill_attention.argtypes = [
                    ctypes.POINTER(_Pool), ctypes.POINTER(_Map), P, P, i32, P, i64, i64, i32, ctypes.c_float,
                    P, i64, i64, P]
                L.bkv_paged_prefill_attention.restype = ctypes.c_int
                L.bkv_decode_multi_out.argtypes = [
                    ctypes.POINTER(_Pool), ctypes.POINTER(_Map), P, i32, P, P, P, i64, i64, i32, ctypes.c_float,
                    P, P, i32, i64, i64, P, ctypes.c_size_t, ctypes.c_uint32, P]
                L.bkv_decode_multi_out.restype = ctypes.c_int
                L.bkv_peer_barrier.argtypes = [P, i32, i32, P, P, ctypes.c_uint64, P]
                L.bkv_peer_barrier.restype = ctypes.c_int
                L.bkv_paged_mixed_attention.argtypes = [
                    ctypes.POINTER(_Pool), ctypes.POINTER(_Map), P, P, i32, i32, i32, i32, P, i64, i64, i32,
                    ctypes.c_float, P, i64, i64, P, ctypes.c_size_t, ctypes.c_uint32, P]
                L.bkv_paged_mixed_attention.restype = ctypes.c_int
                L.bkv_decode_workspace_size.argtypes = [i32, i32, i32, i32]
                L.bkv_decode_workspace_size.restype = ctypes.c_size_t
                L.bkv_validate_layout_host.argtypes = [P, i32, P, i32, i32, i32, P, i32, i32, i32, P]
                L.bkv_validate_layout_host.restype = ctypes.c_int
                L.bkv_validate_block_map_host.argtypes = [ctypes.POINTER(_Map), P, i32, i32, i32, P]
                L.bkv_validate_block_map_host.restype = ctypes.c_int
                L.bkv_kv_checkpoint.argtypes = [ctypes.POINTER(_Pool), P, i32, P, P, P]
                L.bkv_kv_checkpoint.restype = ctypes.c_int
                L.bkv_kv_restore.argtypes = [ctypes.POINTER(_Pool), P, i32, P, P, P]
                L.bkv_kv_restore.restype = ctypes.c_int
                L.bkv_decode_plan_bytes.argtypes = [i32, i32, i32, i32]
                L.bkv_decode_plan_bytes.restype = ctypes.c_size_t
                L.bkv_decode_plan.argtypes = [P, ctypes.POINTER(_Map), i32, i32, i32, i32, i32, P, ctypes.c_size_t,
                                              ctypes.POINTER(ctypes.c_size_t)]
                L.bkv_decode_plan.restype = ctypes.c_int
                L.bkv_decode_planned.argtypes = [
                    ctypes.POINTER(_Pool), ctypes.POINTER(_Map), P, P, P, P, P, P, i64, i64, i32,
                    ctypes.c_float, P, i64, i64, P, i32, P, ctypes.c_size_t, ctypes.c_uint32, P]
                L.bkv_decode_planned.restype = ctypes.c_int
                L.bkv_reload_dev_switches.argtypes = []
                L.bkv_reload_dev_switches.restype = None
                L.bkv_status_string.argtypes = [ctypes.c_int]
                L.bkv_status_string.restype = ctypes.c_char_p
                L.bkv_last_error.restype = ctypes.c_char_p
                L.bkv_version.restype = ctypes.c_int32
                _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        L = lib()
        raise BkvError(f"{what}: {L.bkv_status_string(rc).decode()} -- {L.bkv_last_error().decode()}")


def _stream_ptr(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dev(t: torch.Tensor, name: str, dtype=None):
    if not t.is_cuda:
        raise BkvError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise BkvError(f"{name} must be {dtype}, got {t.dtype}")
    return t


@dataclass
class KVPool:
    """One layer of one rank's KV block pool: K, V bf16 [num_blocks][H][bs][d] (D1)."""
    k: torch.Tensor
    v: torch.Tensor

    @staticmethod
    def empty(num_blocks, num_kv_heads, block_size, head_dim, device="cuda"):
        shape = (num_blocks, num_kv_heads, block_size, head_dim)
        return KVPool(torch.empty(shape, dtype=torch.bfloat16, device=device),
                      torch.empty(shape, dtype=torch.bfloat16, device=device))

    @property
    def num_blocks(self): return self.k.shape[0]

    @property
    def num_kv_heads(self): return self.k.shape[1]

    @property
    def block_size(self): return self.k.shape[2]

    @property
    def head_dim(self): return self.k.shape[3]

    def c(self) -> _Pool:
        _dev(self.k, "pool.k", torch.bfloat16)
        _dev(self.v, "pool.v", torch.bfloat16)
        if self.k.shape != self.v.shape or self.k.stride() != self.v.stride() or self.k.stride(3) != 1:
            raise BkvError("pool k/v must have equal shapes and strides with contiguous head_dim")
        sb, sh, ss, _ = self.k.stride()
        nb, H, bs, d = self.k.shape
        return _Pool(self.k.data_ptr(), self.v.data_ptr(), nb, H, bs, d, sb, sh, ss)


def block_map(block_tables: torch.Tensor, dirs: torch.Tensor, fills=None, num_entries=None) -> _Map:
    """D2 + D3: int32 block tables [B][M]; uint8 dirs [B] (per request) or [B][M].
    General map: uint8 ``fills`` [B][M] (tokens per entry) and int32
    ``num_entries`` [B]; both None for a dense map."""
    _dev(block_tables, "block_tables", torch.int32)
    _dev(dirs, "dirs", torch.uint8)
    if block_tables.dim() != 2 or block_tables.stride(1) != 1:
        raise BkvError("block_tables must be [B][M] with unit column stride")
    B = block_tables.shape[0]
    if dirs.dim() == 1:
        rs, cs = dirs.stride(0), 0
    else:
        rs, cs = dirs.stride(0), dirs.stride(1)
    if dirs.shape[0] != B:
        raise BkvError("dirs must have one row per request")
    if (fills is None) != (num_entries is None):
        raise BkvError("a general map needs both fills and num_entries")
    if fills is None:
        return _Map(block_tables.data_ptr(), block_tables.stride(0), dirs.data_ptr(), rs, cs, B,
                    None, 0, None)
    _dev(fills, "fills", torch.uint8)
    _dev(num_entries, "num_entries", torch.int32)
    if fills.dim() != 2 or fills.shape[0] != B or fills.stride(1) != 1 or num_entries.shape != (B,):
        raise BkvError("fills must be [B][M] with unit column stride, num_entries [B]")
    return _Map(block_tables.data_ptr(), block_tables.stride(0), dirs.data_ptr(), rs, cs, B,
                fills.data_ptr(), fills.stride(0), num_entries.data_ptr())


def kv_append(pool: KVPool, block_tables, dirs, seq_lens_before, cu_new_tokens, k_new, v_new,
              slot_mapping=None, total_new_tokens=None, stream=None, fills=None, num_entries=None):
    """bkv_kv_append: write new K/V rows [total_new][H][d] into their bidirectional slots."""
    p, m = pool.c(), block_map(block_tables, dirs, fills, num_entries)
    _dev(seq_lens_before, "seq_lens_before", torch.int32)
    _dev(cu_new_tokens, "cu_new_tokens", torch.int32)
    _dev(k_new, "k_new", torch.bfloat16)
    _dev(v_new, "v_new", torch.bfloat16)
    if not (k_new.is_contiguous() and v_new.is_contiguous()):
        raise BkvError("k_new/v_new must be contiguous [total_new][H][d]")
    n = k_new.shape[0] if total_new_tokens is None else int(total_new_tokens)
    sm = 0
    if slot_mapping is not None:
        sm = _dev(slot_mapping, "slot_mapping", torch.int64).data_ptr()
    rc = lib().bkv_kv_append(ctypes.byref(p), ctypes.byref(m), seq_lens_before.data_ptr(),
                             cu_new_tokens.data_ptr(), n, k_new.data_ptr(), v_new.data_ptr(),
                             ctypes.c_void_p(sm), _stream_ptr(stream))
    _check(rc, "bkv_kv_append")


def kv_append_checkpoint(pool: KVPool, block_tables, dirs, seq_lens_before, cu_new_tokens, k_new, v_new,
                         evict_rows, ckpt_k, ckpt_v, slot_mapping=None, total_new_tokens=None,
                         stream=None, fills=None, num_entries=None):
    """bkv_kv_append_checkpoint: kv_append that first copies the live peer rows it overwrites
    (evict_rows[i] >= 0 -> row evict_rows[i] of ckpt_k/ckpt_v, bf16 [rows][H][d]) -- the
    lazy checkpoint of PAPER.md P:726-728, fused into the write."""
    p, m = pool.c(), block_map(block_tables, dirs, fills, num_entries)
    for t, n in ((seq_lens_before, "seq_lens_before"), (cu_new_tokens, "cu_new_tokens"),
                 (evict_rows, "evict_rows")):
        _dev(t, n, torch.int32)
    for t, n in ((k_new, "k_new"), (v_new, "v_new"), (ckpt_k, "ckpt_k"), (ckpt_v, "ckpt_v")):
        if n.startswith("ckpt") and not t.is_cuda:
            if not t.is_pinned():   # pinned host memory is device-addressable under UVA
                raise BkvError(f"{n} must be a CUDA tensor or pinned host memory")
            if t.dtype != torch.bfloat16:
                raise BkvError(f"{n} must be bfloat16")
        else:
            _dev(t, n, torch.bfloat16)
        if not t.is_contiguous():
            raise BkvError(f"{n} must be contiguous")
    n = k_new.shape[0] if total_new_tokens is None else int(total_new_tokens)
    sm = 0 if slot_mapping is None else _dev(slot_mapping, "slot_mapping", torch.int64).data_ptr()
    rc = lib().bkv_kv_append_checkpoint(ctypes.byref(p), ctypes.byref(m), seq_lens_before.data_ptr(),
                                        cu_new_tokens.data_ptr(), n, k_new.data_ptr(), v_new.data_ptr(),
                                        ctypes.c_void_p(sm), evict_rows.data_ptr(), ckpt_k.data_ptr(),
                                        ckpt_v.data_ptr(), _stream_ptr(stream))
    _check(rc, "bkv_kv_append_checkpoint")


def kv_checkpoint(pool: KVPool, slot_ids, k_out=None, v_out=None, stream=None):
    """bkv_kv_checkpoint: rows of physical slots (int64 ids block*bs+slot) -> [n][H][d] buffers
    (device tensors, or device views of pinned host memory).  Returns (k_out, v_out)."""
    p = pool.c()
    _dev(slot_ids, "slot_ids", torch.int64)
    n = slot_ids.numel()
    shape = (n, pool.num_kv_heads, pool.head_dim)
    if k_out is None:
        k_out = torch.empty(shape, dtype=torch.bfloat16, device=pool.k.device)
    if v_out is None:
        v_out = torch.empty(shape, dtype=torch.bfloat16, device=pool.k.device)
    for t, nm in ((k_out, "k_out"), (v_out, "v_out")):
        if not t.is_cuda and not t.is_pinned():   # pinned host memory is device-addressable (UVA)
            raise BkvError(f"{nm} must be a CUDA tensor or pinned host memory")
        if t.dtype != torch.bfloat16 or not t.is_contiguous() or tuple(t.shape) != shape:
            raise BkvError(f"{nm} must be contiguous bfloat16 {list(shape)}")
    rc = lib().bkv_kv_checkpoint(ctypes.byref(p), slot_ids.data_ptr(), n, k_out.data_ptr(), v_out.data_ptr(),
                                 _stream_ptr(stream))
    _check(rc, "bkv_kv_checkpoint")
    return k_out, v_out


def kv_restore(pool: KVPool, slot_ids, k_in, v_in, stream=None):
    """bkv_kv_restore: scatter checkpointed rows back into their slots (swap-in)."""
    p = pool.c()
    _dev(slot_ids, "slot_ids", torch.int64)
    n = slot_ids.numel()
    shape = (n, pool.num_kv_heads, pool.head_dim)
    for t, nm in ((k_in, "k_in"), (v_in, "v_in")):
        if not t.is_cuda and not t.is_pinned():   # pinned host memory is device-addressable (UVA)
            raise BkvError(f"{nm} must be a CUDA tensor or pinned host memory")
        if t.dtype != torch.bfloat16 or not t.is_contiguous() or tuple(t.shape) != shape:
            raise BkvError(f"{nm} must be contiguous bfloat16 {list(shape)}")
    rc = lib().bkv_kv_restore(ctypes.byref(p), slot_ids.data_ptr(), slot_ids.numel(), k_in.data_ptr(),
                              v_in.data_ptr(), _stream_ptr(stream))
    _check(rc, "bkv_kv_restore")


def decode_workspace_size(num_seqs, num_q_heads, num_kv_heads, head_dim) -> int:
    n = lib().bkv_decode_workspace_size(num_seqs, num_q_heads, num_kv_heads, head_dim)
    if n == 0:
        raise BkvError("bkv_decode_workspace_size: " + lib().bkv_last_error().decode())
    return int(n)


_ws_cache = {}
_ws_lock = threading.Lock()


def workspace(num_seqs, num_q_heads, num_kv_heads, head_dim, device=None, stream=None):
    """Zero-initialised workspace cached per (device, stream); grows on demand."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    s = torch.cuda.current_stream(dev) if stream is None else stream
    need = decode_workspace_size(num_seqs, num_q_heads, num_kv_heads, head_dim)
    key = (dev.index, s.cuda_stream)
    with _ws_lock:
        ws = _ws_cache.get(key)
        if ws is None or ws.numel() < need:
            # allocated and zeroed ON the stream that will use it, so its first kernel is
            # ordered after the zero-fill and the allocator ties the block to that stream
            with torch.cuda.stream(s):
                ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=dev)
            _ws_cache[key] = ws
    return ws


def _attn_args(pool, block_tables, dirs, seq_lens, q, softmax_scale, out, max_seq_len, ws, stream,
               fills=None, num_entries=None):
    p, m = pool.c(), block_map(block_tables, dirs, fills, num_entries)
    _dev(seq_lens, "seq_lens", torch.int32)
    _dev(q, "q", torch.bfloat16)
    if q.dim() != 3:
        raise BkvError("q must be [B][Hq][d]")
    B, Hq, d = q.shape
    if q.stride(2) != 1:
        raise BkvError("q must have a unit stride along head_dim")
    if B != block_tables.shape[0] or seq_lens.dim() != 1 or seq_lens.numel() != B:
        raise BkvError(f"q has {B} rows but block_tables has {block_tables.shape[0]} and "
                       f"seq_lens {seq_lens.numel()}: one row per request in each")
    if d != pool.head_dim:
        raise BkvError(f"q head_dim {d} != pool head_dim {pool.head_dim}")
    if out is None:
        out = torch.empty((B, Hq, d), dtype=torch.bfloat16, device=q.device)
    _dev(out, "out", torch.bfloat16)
    if out.dim() != 3 or tuple(out.shape) != (B, Hq, d):
        raise BkvError(f"out must be [B][Hq][d] = {[B, Hq, d]}, got {list(out.shape)}")
    if out.stride(2) != 1:
        raise BkvError("out must have a unit stride along head_dim")
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(d)
    if max_seq_len is None:
        max_seq_len = block_tables.shape[1] * pool.block_size
    if ws is None:
        ws = workspace(B, Hq, pool.num_kv_heads, d, q.device, stream)
    return p, m, out, softmax_scale, max_seq_len, ws


def paged_decode_attention(pool: KVPool, block_tables, dirs, seq_lens, q, softmax_scale=None,
                           out=None, max_seq_len=None, ws=None, stream=None, pdl=False,
                           fills=None, num_entries=None):
    """bkv_paged_decode_attention.  q: bf16 [B][Hq][d] (any strides with unit last stride).
    out: bf16 with the same indexing (allocated [B][Hq][d] if None).  Returns out.
    ``fills``/``num_entries``: general map."""
    p, m, out, scale, msl, ws = _attn_args(pool, block_tables, dirs, seq_lens, q, softmax_scale,
                                           out, max_seq_len, ws, stream, fills, num_entries)
    rc = lib().bkv_paged_decode_attention_ex(
        ctypes.byref(p), ctypes.byref(m), seq_lens.data_ptr(), int(msl), q.data_ptr(),
        q.stride(0), q.stride(1), q.shape[1], float(scale), out.data_ptr(), out.stride(0),
        out.stride(1), ws.data_ptr(), ws.numel(), BKV_FLAG_PDL if pdl else 0, _stream_ptr(stream))
    _check(rc, "bkv_paged_decode_attention")
    return out


def decode_step(pool: KVPool, block_tables, dirs, seq_lens, k_new, v_new, q, softmax_scale=None,
                out=None, max_seq_len=None, ws=None, stream=None, pdl=False, fills=None,
                num_entries=None):
    """bkv_decode_step: append token seq_lens[r]-1 of every request (k_new/v_new contiguous
    bf16 [B][H_kv][d]) and attend over the context including it, in one launch pair.
    Equal to kv_append(before=seq_lens-1, cu=arange(B+1)) + paged_decode_attention."""
    p, m, out, scale, msl, ws = _attn_args(pool, block_tables, dirs, seq_lens, q, softmax_scale,
                                           out, max_seq_len, ws, stream, fills, num_entries)
    _dev(k_new, "k_new", torch.bfloat16)
    _dev(v_new, "v_new", torch.bfloat16)
    shape = (q.shape[0], pool.num_kv_heads, pool.head_dim)
    if tuple(k_new.shape) != shape or tuple(v_new.shape) != shape:
        raise BkvError(f"k_new/v_new must be [B][H_kv][d] = {list(shape)}")
    if not (k_new.is_contiguous() and v_new.is_contiguous()):
        raise BkvError("k_new/v_new must be contiguous")
    rc = lib().bkv_decode_step(
        ctypes.byref(p), ctypes.byref(m), seq_lens.data_ptr(), int(msl), k_new.data_ptr(),
        v_new.data_ptr(), q.data_ptr(), q.stride(0), q.stride(1), q.shape[1], float(scale),
        out.data_ptr(), out.stride(0), out.stride(1), ws.data_ptr(), ws.numel(),
        BKV_FLAG_PDL if pdl else 0, _stream_ptr(stream))
    _check(rc, "bkv_decode_step")
    return out


def paged_prefill_attention(pool: KVPool, block_tables, dirs, seq_lens, cu_q, q, max_q_len=None,
                            softmax_scale=None, out=None, stream=None, fills=None, num_entries=None):
    """bkv_paged_prefill_attention: causal attention of every request's LAST
    n_r = cu_q[r+1]-cu_q[r] tokens over its paged context; q/out bf16 [total][Hq][d]
    (unit last stride).  n_r = 1 rows are decodes, so one call serves a mixed batch.
    ``max_q_len``: host bound of max n_r (sizes the grid); None uses the total row count, a
    valid but looser bound -- pass the scheduler's value, no device reduction is ever run."""
    p, m = pool.c(), block_map(block_tables, dirs, fills, num_entries)
    _dev(seq_lens, "seq_lens", torch.int32)
    _dev(cu_q, "cu_q", torch.int32)
    _dev(q, "q", torch.bfloat16)
    T, Hq, d = q.shape
    if q.stride(2) != 1:
        raise BkvError("q must have a unit stride along head_dim")
    if out is None:
        out = torch.empty((T, Hq, d), dtype=torch.bfloat16, device=q.device)
    _dev(out, "out", torch.bfloat16)
    if out.stride(2) != 1:
        raise BkvError("out must have a unit stride along head_dim")
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(d)
    if max_q_len is None:   # a host upper bound with no device reduction or sync: n_r <= total rows
        max_q_len = T
    rc = lib().bkv_paged_prefill_attention(
        ctypes.byref(p), ctypes.byref(m), seq_lens.data_ptr(), cu_q.data_ptr(), int(max_q_len),
        q.data_ptr(), q.stride(0), q.stride(1), Hq, float(softmax_scale), out.data_ptr(),
        out.stride(0), out.stride(1), _stream_ptr(stream))
    _check(rc, "bkv_paged_prefill_attention")
    return out


def _ptr_array(ptrs):
    vals = [p if isinstance(p, int) else p.data_ptr() for p in ptrs]
    return (ctypes.c_void_p * max(1, len(vals)))(*vals), len(vals)


def decode_multi_out(pool: KVPool, block_tables, dirs, seq_lens, q, out, peer_outs, k_new=None,
                     v_new=None, softmax_scale=None, max_seq_len=None, ws=None, stream=None, pdl=False,
                     fills=None, num_entries=None, multicast=False):
    """bkv_decode_multi_out (fused reassembly): decode attention (or the fused
    decode step when k_new/v_new are given) whose output rows are also stored into every
    pointer of ``peer_outs`` (ints = device-accessible peer addresses, or tensors), with
    ``out``'s strides.  ``multicast``: peer_outs is ONE NVLS multicast address and each row
    is stored once with multimem.st (BKV_FLAG_PEER_MULTICAST).  Returns out."""
    p, m, out, scale, msl, ws = _attn_args(pool, block_tables, dirs, seq_lens, q, softmax_scale,
                                           out, max_seq_len, ws, stream, fills, num_entries)
    arr, n = _ptr_array(peer_outs)
    kp = vp = None
    if k_new is not None:
        _dev(k_new, "k_new", torch.bfloat16)
        _dev(v_new, "v_new", torch.bfloat16)
        kp, vp = k_new.data_ptr(), v_new.data_ptr()
    rc = lib().bkv_decode_multi_out(
        ctypes.byref(p), ctypes.byref(m), seq_lens.data_ptr(), int(msl), kp, vp, q.data_ptr(),
        q.stride(0), q.stride(1), q.shape[1], float(scale), out.data_ptr(), arr, n, out.stride(0),
        out.stride(1), ws.data_ptr(), ws.numel(),
        (BKV_FLAG_PDL if pdl else 0) | (BKV_FLAG_PEER_MULTICAST if multicast else 0), _stream_ptr(stream))
    _check(rc, "bkv_decode_multi_out")
    return out


def peer_barrier(pads, rank, counter, err, timeout_ns=5_000_000_000, stream=None):
    """bkv_peer_barrier: stream-ordered cross-rank completion signal (``pads`` = per-rank
    device-accessible uint32 flag arrays, ints or tensors; counter/err: int32 device tensors)."""
    arr, n = _ptr_array(pads)
    rc = lib().bkv_peer_barrier(arr, n, int(rank), counter.data_ptr(), err.data_ptr(), int(timeout_ns),
                                _stream_ptr(stream))
    _check(rc, "bkv_peer_barrier")


def paged_mixed_attention(pool: KVPool, block_tables, dirs, seq_lens, cu_q, q, num_prefill_seqs,
                          num_prefill_rows, max_q_len=None, max_seq_len=None, softmax_scale=None,
                          out=None, ws=None, stream=None, pdl=False, fills=None, num_entries=None):
    """bkv_paged_mixed_attention (P:762-765 dispatch): requests [0, P) prefill through the causal
    kernel, requests [P, B) decode (one row each, rows after the prefill rows) through the
    split-K decode kernel.  q/out bf16 [total][Hq][d]."""
    p, m = pool.c(), block_map(block_tables, dirs, fills, num_entries)
    for t, n in ((seq_lens, "seq_lens"), (cu_q, "cu_q")):
        _dev(t, n, torch.int32)
    _dev(q, "q", torch.bfloat16)
    T, Hq, d = q.shape
    if out is None:
        out = torch.empty((T, Hq, d), dtype=torch.bfloat16, device=q.device)
    _dev(out, "out", torch.bfloat16)
    if q.stride(2) != 1 or out.stride(2) != 1:
        raise BkvError("q/out must have a unit stride along head_dim")
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(d)
    if max_q_len is None:   # host upper bound, no device op: a prefill's n_r <= the prefill rows
        max_q_len = int(num_prefill_rows)
    if max_seq_len is None:
        max_seq_len = block_tables.shape[1] * pool.block_size
    B = block_tables.shape[0]
    if ws is None:
        ws = workspace(max(1, B - int(num_prefill_seqs)), Hq, pool.num_kv_heads, d, q.device, stream)
    rc = lib().bkv_paged_mixed_attention(
        ctypes.byref(p), ctypes.byref(m), seq_lens.data_ptr(), cu_q.data_ptr(), int(num_prefill_seqs),
        int(num_prefill_rows), int(max_q_len), int(max_seq_len), q.data_ptr(), q.stride(0), q.stride(1), Hq,
        float(softmax_scale), out.data_ptr(), out.stride(0), out.stride(1), ws.data_ptr(), ws.numel(),
        BKV_FLAG_PDL if pdl else 0, _stream_ptr(stream))
    _check(rc, "bkv_paged_mixed_attention")
    return out


def reload_dev_switches():
    """Re-read the BKV_* developer switches (read once per process otherwise)."""
    lib().bkv_reload_dev_switches()


class DecodePlan:
    """A host-built split plan of one decode step (bkv_decode_plan) and its device copy.

    Built from the scheduler's HOST lengths and block map once per step; every layer's
    :func:`decode_planned` call reuses it."""

    def __init__(self, host, dev, nbytes):
        self.host = host          # numpy int32 buffer (the header is read by each call)
        self.dev = dev            # torch uint8 device tensor holding the same bytes (capacity-sized)
        self.nbytes = nbytes      # bytes a step uploads (the layout is fixed; the tail is the entry list)

    @property
    def header(self):
        names = ("magic", "version", "words", "B", "H", "g", "D", "bs", "general", "grid", "warps", "P",
                 "n_segs", "n_tasks", "n_zero", "total", "off_wseg", "off_segs", "off_ctask", "off_tasks",
                 "off_zero", "max_pieces", "max_entries", "off_xrows", "n_xrows", "off_ent", "n_ent")
        return {n: int(self.host[i]) for i, n in enumerate(names)}

    def upload(self, host, stream=None):
        """Copy a later step's plan (same geometry) into this plan's device buffer."""
        t = torch.from_numpy(np.asarray(host).view(np.uint8))
        self.dev[:t.numel()].copy_(t, non_blocking=False)
        self.host = host


def _host_map(block_tables, dirs, fills=None, num_entries=None):
    bt = np.ascontiguousarray(np.asarray(block_tables), dtype=np.int32)
    dd = np.ascontiguousarray(np.asarray(dirs), dtype=np.uint8)
    rs, cs = (1, 0) if dd.ndim == 1 else (dd.shape[1], 1)
    keep = [bt, dd]
    if fills is None:
        m = _Map(bt.ctypes.data, bt.shape[1], dd.ctypes.data, rs, cs, bt.shape[0], None, 0, None)
    else:
        f = np.ascontiguousarray(np.asarray(fills), dtype=np.uint8)
        ne = np.ascontiguousarray(np.asarray(num_entries), dtype=np.int32)
        keep += [f, ne]
        m = _Map(bt.ctypes.data, bt.shape[1], dd.ctypes.data, rs, cs, bt.shape[0], f.ctypes.data, f.shape[1],
                 ne.ctypes.data)
    return m, keep


def decode_plan_host(seq_lens, block_tables, dirs, num_kv_heads, num_q_heads, head_dim, block_size,
                     fills=None, num_entries=None, num_sms=0):
    """bkv_decode_plan on host arrays (lengths and the step's block map) -> numpy int32 plan
    (capacity-sized view; the first ``nbytes`` bytes are the step's upload, see .nbytes of
    :class:`DecodePlan`).  ``num_sms`` = 0 plans for the current device (needs a GPU)."""
    ln = np.ascontiguousarray(np.asarray(seq_lens), dtype=np.int32)
    m, keep = _host_map(block_tables, dirs, fills, num_entries)
    cap = lib().bkv_decode_plan_bytes(m.num_seqs, int(num_kv_heads), m.bt_stride, int(num_sms))
    if cap == 0:
        raise BkvError("bkv_decode_plan_bytes: " + lib().bkv_last_error().decode())
    buf = np.zeros((cap + 15) // 4 + 4, dtype=np.int32)
    off = (-buf.ctypes.data) % 16 // 4            # 16-byte aligned view
    view = buf[off:off + cap // 4]
    used = ctypes.c_size_t(0)
    rc = lib().bkv_decode_plan(ln.ctypes.data, ctypes.byref(m), int(num_kv_heads), int(num_q_heads),
                               int(head_dim), int(block_size), int(num_sms), view.ctypes.data, view.nbytes,
                               ctypes.byref(used))
    del keep
    _check(rc, "bkv_decode_plan")
    return view   # (a view: keeps the aligned buffer alive)


def plan_used_bytes(host):
    """Bytes of a host plan a step must upload (header words: off_ent + n_ent entries)."""
    return 4 * (int(host[25]) + int(host[26]))


def decode_plan(seq_lens_host, block_tables_host, dirs_host, pool_or_geom, num_q_heads, fills_host=None,
                num_entries_host=None, device=None, stream=None):
    """Build the step's plan on the host and copy it to a device buffer of the plan capacity.

    ``pool_or_geom``: a KVPool (geometry taken from it) or a tuple (num_kv_heads, head_dim, block_size)."""
    if isinstance(pool_or_geom, KVPool):
        H, d, bs = pool_or_geom.num_kv_heads, pool_or_geom.head_dim, pool_or_geom.block_size
        device = pool_or_geom.k.device if device is None else device
    else:
        H, d, bs = pool_or_geom
    host = decode_plan_host(seq_lens_host, block_tables_host, dirs_host, H, num_q_heads, d, bs, fills_host,
                            num_entries_host)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    t = torch.from_numpy(host.view(np.uint8))
    s = torch.cuda.current_stream(dev) if stream is None else stream
    with torch.cuda.stream(s):
        d_t = torch.empty(t.numel() + 16, dtype=torch.uint8, device=dev)
        off = (-d_t.data_ptr()) % 16
        d_t = d_t[off:off + t.numel()]
        n = plan_used_bytes(host)
        d_t[:n].copy_(t[:n])   # pageable source: complete on return
    return DecodePlan(host, d_t, n)


def decode_planned(pool: KVPool, block_tables, dirs, seq_lens, plan: DecodePlan, q, k_new=None, v_new=None,
                   softmax_scale=None, out=None, peer_outs=(), ws=None, stream=None, pdl=False, fills=None,
                   num_entries=None, kv_early=False, multicast=False):
    """bkv_decode_planned: one layer's decode attention (or fused decode step when k_new/v_new
    are given) with the step's host-built plan (the decode kernel + the cross-CTA merge
    kernel).  Returns out.  ``kv_early`` (with ``pdl``): BKV_FLAG_KV_EARLY -- the preceding
    kernel does not write this pool's resident KV, so the first KV tiles are requested (and
    the next few prefetched into L2) before the grid wait.  ``multicast``: ``peer_outs`` is
    ONE NVLS multicast address (BKV_FLAG_PEER_MULTICAST)."""
    p, m, out, scale, _, ws = _attn_args(pool, block_tables, dirs, seq_lens, q, softmax_scale,
                                         out, None, ws, stream, fills, num_entries)
    if plan.dev.device != q.device:
        raise BkvError("plan was copied to another device")
    kp = vp = None
    if (k_new is None) != (v_new is None):
        raise BkvError("k_new and v_new must both be given or both be None")
    if k_new is not None:
        _dev(k_new, "k_new", torch.bfloat16)
        _dev(v_new, "v_new", torch.bfloat16)
        shape = (q.shape[0], pool.num_kv_heads, pool.head_dim)
        if tuple(k_new.shape) != shape or tuple(v_new.shape) != shape:
            raise BkvError(f"k_new/v_new must be [B][H_kv][d] = {list(shape)}")
        if not (k_new.is_contiguous() and v_new.is_contiguous()):
            raise BkvError("k_new/v_new must be contiguous")
        kp, vp = k_new.data_ptr(), v_new.data_ptr()
    arr, n = _ptr_array(list(peer_outs))
    rc = lib().bkv_decode_planned(
        ctypes.byref(p), ctypes.byref(m), seq_lens.data_ptr(), plan.host.ctypes.data, plan.dev.data_ptr(),
        kp, vp, q.data_ptr(), q.stride(0), q.stride(1), q.shape[1], float(scale), out.data_ptr(),
        out.stride(0), out.stride(1), arr if n else None, n, ws.data_ptr(), ws.numel(),
        (BKV_FLAG_PDL if pdl else 0) | (BKV_FLAG_KV_EARLY if (pdl and kv_early) else 0)
        | (BKV_FLAG_PEER_MULTICAST if multicast else 0), _stream_ptr(stream))
    _check(rc, "bkv_decode_planned")
    return out


def validate_layout_host(block_tables, dirs, seq_lens, num_blocks, block_size, require_nonempty=True):
    """Host validator (I1-I4) on CPU tensors / numpy arrays.  Returns (ok, info[5])."""
    bt = np.ascontiguousarray(np.asarray(block_tables), dtype=np.int32)
    dd = np.ascontiguousarray(np.asarray(dirs), dtype=np.uint8)
    ln = np.ascontiguousarray(np.asarray(seq_lens), dtype=np.int32)
    rs, cs = (1, 0) if dd.ndim == 1 else (dd.shape[1], 1)
    info = np.zeros(5, dtype=np.int64)
    rc = lib().bkv_validate_layout_host(bt.ctypes.data, bt.shape[1], dd.ctypes.data, rs, cs,
                                        ln.shape[0], ln.ctypes.data, int(num_blocks), int(block_size),
                                        int(bool(require_nonempty)), info.ctypes.data)
    if rc not in (0, 4):
        _check(rc, "bkv_validate_layout_host")
    return rc == 0, [int(x) for x in info]


def validate_block_map_host(block_tables, dirs, seq_lens, num_blocks, block_size, fills=None,
                            num_entries=None, require_nonempty=True):
    """bkv_validate_block_map_host on host arrays (dense, or general with fills/num_entries).
    Returns (ok, info[5])."""
    bt = np.ascontiguousarray(np.asarray(block_tables), dtype=np.int32)
    dd = np.ascontiguousarray(np.asarray(dirs), dtype=np.uint8)
    ln = np.ascontiguousarray(np.asarray(seq_lens), dtype=np.int32)
    rs, cs = (1, 0) if dd.ndim == 1 else (dd.shape[1], 1)
    keep = [bt, dd, ln]
    if fills is None:
        m = _Map(bt.ctypes.data, bt.shape[1], dd.ctypes.data, rs, cs, ln.shape[0], None, 0, None)
    else:
        f = np.ascontiguousarray(np.asarray(fills), dtype=np.uint8)
        ne = np.ascontiguousarray(np.asarray(num_entries), dtype=np.int32)
        keep += [f, ne]
        m = _Map(bt.ctypes.data, bt.shape[1], dd.ctypes.data, rs, cs, ln.shape[0], f.ctypes.data,
                 f.shape[1], ne.ctypes.data)
    info = np.zeros(5, dtype=np.int64)
    rc = lib().bkv_validate_block_map_host(ctypes.byref(m), ln.ctypes.data, int(num_blocks),
                                           int(block_size), int(bool(require_nonempty)), info.ctypes.data)
    del keep
    if rc not in (0, 4):
        _check(rc, "bkv_validate_block_map_host")
    return rc == 0, [int(x) for x in info]
