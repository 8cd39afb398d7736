"""Counter-based bf16 value generator with bit-identical numpy and torch versions.

Every K/V/Q element is a pure function of (seed, kind, layer, request, index),
so a rank holding a head shard, the CPU oracle and the GPU path all draw the
same numbers without shipping tensors around (SURVEY §8(d) "all GPU data
derives from (seed, config, layer, global kv_head)").

Distribution: Irwin-Hall sum of four 12-bit uniforms, centred, times 2^-11
(mean 0, std ~1.15, |x| <= 4), rounded to bf16 with round-to-nearest-even done
in integer arithmetic so both backends agree bit for bit.  SURVEY Q15: parity
inputs use unit-scale V; peaked logits come from scaling Q by a power of two
(``scale_log2``), which is exact in bf16.
"""
from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF
BF16_NAN = 0x7FC0          # quiet-NaN bf16 pattern used to poison non-owned slots
KIND_K, KIND_V, KIND_Q, KIND_QP = 1, 2, 3, 4


def _mul32_np(x, c: int):
    x = x.astype(np.uint64)
    lo = (x & np.uint64(0xFFFF)) * np.uint64(c)
    hi = (((x >> np.uint64(16)) * np.uint64(c & 0xFFFF)) & np.uint64(0xFFFF)) << np.uint64(16)
    return (lo + hi) & np.uint64(M32)


def _mix32_np(x):
    x = x.astype(np.uint64)
    x = x ^ (x >> np.uint64(16))
    x = _mul32_np(x, 0x7FEB352D)
    x = x ^ (x >> np.uint64(15))
    x = _mul32_np(x, 0x846CA68B)
    x = x ^ (x >> np.uint64(16))
    return x


def key32(*parts: int) -> int:
    """Fold integer parts (each < 2^32) into one 32-bit stream key."""
    x = np.array([0x811C9DC5], dtype=np.uint64)
    for p in parts:
        p = int(p)
        assert 0 <= p <= M32, p
        x = _mix32_np((x ^ np.uint64(p)) + np.uint64(0x9E3779B9) & np.uint64(M32))
    return int(x[0])


def _bits_from_hash_np(base: int, idx: np.ndarray, scale_log2: int) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.uint64)
    assert idx.size == 0 or int(idx.max()) <= M32
    h1 = _mix32_np((np.uint64(base) + _mul32_np(idx, 0x9E3779B1)) & np.uint64(M32))
    h2 = _mix32_np(h1 ^ np.uint64(0x85EBCA6B))
    m = np.uint64(0xFFF)
    c = ((h1 & m) + ((h1 >> np.uint64(12)) & m) + (h2 & m) + ((h2 >> np.uint64(12)) & m)).astype(np.int64) - 8190
    f = c.astype(np.float32) * np.float32(2.0 ** (scale_log2 - 11))   # exact: |c| < 2^13, power-of-2 scale
    u = f.view(np.uint32).astype(np.uint64)
    bias = np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))
    return ((u + bias) >> np.uint64(16)).astype(np.uint16)


def hash_bf16_np(base: int, idx, scale_log2: int = 0) -> np.ndarray:
    """bf16 bit patterns (uint16) for counter indices ``idx`` of stream ``base``."""
    return _bits_from_hash_np(base, np.asarray(idx), scale_log2)


# ---------------------------------------------------------------- torch twin
def _mul32_t(x, c: int):
    lo = (x & 0xFFFF) * c
    hi = (((x >> 16) * (c & 0xFFFF)) & 0xFFFF) << 16
    return (lo + hi) & M32


def _mix32_t(x):
    x = x ^ (x >> 16)
    x = _mul32_t(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32_t(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def hash_bf16_torch(base: int, idx, scale_log2: int = 0):
    """torch twin of :func:`hash_bf16_np`; ``idx`` is an int64 tensor (any device).

    Returns a torch.bfloat16 tensor with the same bits as the numpy version.
    """
    import torch
    h1 = _mix32_t((idx * 0 + base + _mul32_t(idx, 0x9E3779B1)) & M32)
    h2 = _mix32_t(h1 ^ 0x85EBCA6B)
    c = (h1 & 0xFFF) + ((h1 >> 12) & 0xFFF) + (h2 & 0xFFF) + ((h2 >> 12) & 0xFFF) - 8190
    f = c.to(torch.float32) * (2.0 ** (scale_log2 - 11))
    u = f.view(torch.int32).to(torch.int64) & M32
    bias = 0x7FFF + ((u >> 16) & 1)
    b = ((u + bias) >> 16).to(torch.int32)
    b = torch.where(b >= 0x8000, b - 0x10000, b).to(torch.int16)
    return b.view(torch.bfloat16)


# ------------------------------------------------------- named value streams
def _stream(seed: int, kind: int, layer: int, req: int) -> int:
    return key32(seed, kind, layer, req)


def dense_kv_np(seed: int, layer: int, req: int, L: int, heads, d: int, h_total: int,
                t0: int = 0):
    """Dense logical-order K and V of request ``req``: uint16 [L][len(heads)][d].

    ``heads`` are GLOBAL kv-head indices; element (t, h, i) is counter
    ((t0+t)*h_total + h)*d + i of the request's K (resp. V) stream.
    """
    heads = np.asarray(list(heads), dtype=np.int64)
    t = np.arange(t0, t0 + L, dtype=np.int64)[:, None, None]
    idx = (t * h_total + heads[None, :, None]) * d + np.arange(d, dtype=np.int64)[None, None, :]
    k = hash_bf16_np(_stream(seed, KIND_K, layer, req), idx)
    v = hash_bf16_np(_stream(seed, KIND_V, layer, req), idx)
    return k, v


def q_np(seed: int, layer: int, req: int, heads, d: int, scale_log2: int = 0):
    """Query rows of request ``req`` for GLOBAL q-heads ``heads``: uint16 [len(heads)][d]."""
    heads = np.asarray(list(heads), dtype=np.int64)
    idx = heads[:, None] * d + np.arange(d, dtype=np.int64)[None, :]
    return hash_bf16_np(_stream(seed, KIND_Q, layer, req), idx, scale_log2)


def dense_kv_torch(seed: int, layer: int, req: int, L: int, heads, d: int, h_total: int,
                   device, t0: int = 0):
    import torch
    heads = torch.as_tensor(list(heads), dtype=torch.int64, device=device)
    t = torch.arange(t0, t0 + L, dtype=torch.int64, device=device)[:, None, None]
    idx = (t * h_total + heads[None, :, None]) * d + torch.arange(d, dtype=torch.int64, device=device)[None, None, :]
    k = hash_bf16_torch(_stream(seed, KIND_K, layer, req), idx)
    v = hash_bf16_torch(_stream(seed, KIND_V, layer, req), idx)
    return k, v


def q_torch(seed: int, layer: int, req: int, heads, d: int, device, scale_log2: int = 0):
    import torch
    heads = torch.as_tensor(list(heads), dtype=torch.int64, device=device)
    idx = heads[:, None] * d + torch.arange(d, dtype=torch.int64, device=device)[None, :]
    return hash_bf16_torch(_stream(seed, KIND_Q, layer, req), idx, scale_log2)


def q_rows_np(seed: int, layer: int, req: int, n: int, heads, d: int, h_total: int,
              scale_log2: int = 0):
    """Query rows of a request's last ``n`` tokens (mixed prefill + decode):
    uint16 [n][len(heads)][d]; element (i, h, c) is counter (i*h_total + h)*d + c of the
    request's prefill-query stream (GLOBAL q-head indices)."""
    heads = np.asarray(list(heads), dtype=np.int64)
    i = np.arange(n, dtype=np.int64)[:, None, None]
    idx = (i * h_total + heads[None, :, None]) * d + np.arange(d, dtype=np.int64)[None, None, :]
    return hash_bf16_np(_stream(seed, KIND_QP, layer, req), idx, scale_log2)


def q_rows_torch(seed: int, layer: int, req: int, n: int, heads, d: int, h_total: int, device,
                 scale_log2: int = 0):
    import torch
    heads = torch.as_tensor(list(heads), dtype=torch.int64, device=device)
    i = torch.arange(n, dtype=torch.int64, device=device)[:, None, None]
    idx = (i * h_total + heads[None, :, None]) * d + torch.arange(d, dtype=torch.int64, device=device)[None, None, :]
    return hash_bf16_torch(_stream(seed, KIND_QP, layer, req), idx, scale_log2)
