"""CPU oracle for BROS bidirectional paged decode attention -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It wraps ``bkv_oracle.c``
(plain C, fp64) through ctypes and shares nothing with the CUDA path.

Function-level citations live in ``bkv_oracle.c``.  Parity pins: DESIGN.md
"Oracle pins".  Nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bkv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -fopenmp).  Returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, dbl = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        L.bkvo_bf16_to_f64.argtypes = [ctypes.c_uint16]
        L.bkvo_bf16_to_f64.restype = dbl
        L.bkvo_slot_in_block.argtypes = [i32, i64, i32]
        L.bkvo_slot_in_block.restype = i32
        L.bkvo_validate.argtypes = [i32, P, i32, P, i32, i32, P, i32, i32, i32, P]
        L.bkvo_validate.restype = i32
        L.bkvo_append.argtypes = [P, P, i64, i64, i64, i32, i32, i32,
                                  i32, P, i32, P, i32, i32, P, P, P, P, P]
        L.bkvo_append.restype = None
        L.bkvo_gather.argtypes = [P, P, i64, i64, i64, i32, i32, i32,
                                  P, i32, P, i32, i32, i32, i64, P, P]
        L.bkvo_gather.restype = None
        L.bkvo_attention.argtypes = [P, P, i64, i64, i64, i32, i32, i32,
                                     P, i32, P, i32, i32, P, i32, i32, P, i32, dbl, P]
        L.bkvo_attention.restype = None
        L.bkvo_checkpoint.argtypes = [P, P, i64, i64, i64, i32, i32, i32, P, i32, P, P]
        L.bkvo_checkpoint.restype = None
        L.bkvo_restore.argtypes = [P, P, i64, i64, i64, i32, i32, i32, P, i32, P, P]
        L.bkvo_restore.restype = None
        L.bkvo_overwritten_peers.argtypes = [i32, P, i32, P, i32, i32, P, P, P, i32, i32, P, P, P, i32]
        L.bkvo_overwritten_peers.restype = i32
        L.bkvo_validate_f.argtypes = [i32, P, i32, P, i32, i32, P, i32, P, P, i32, i32, i32, P]
        L.bkvo_validate_f.restype = i32
        L.bkvo_append_f.argtypes = [P, P, i64, i64, i64, i32, i32, i32,
                                    i32, P, i32, P, i32, i32, P, i32, P, P, P, P, P]
        L.bkvo_append_f.restype = None
        L.bkvo_gather_f.argtypes = [P, P, i64, i64, i64, i32, i32, i32,
                                    P, i32, P, i32, i32, P, i32, i32, i64, P, P]
        L.bkvo_gather_f.restype = None
        L.bkvo_attention_f.argtypes = [P, P, i64, i64, i64, i32, i32, i32,
                                       P, i32, P, i32, i32, P, i32, P, i32, i32, P, i32, dbl, P]
        L.bkvo_attention_f.restype = None
        L.bkvo_prefill_attention.argtypes = [P, P, i64, i64, i64, i32, i32, i32,
                                             P, i32, P, i32, i32, P, i32, i32, P, P, P, i32, dbl, P]
        L.bkvo_prefill_attention.restype = None
        L.bkvo_num_threads.restype = i32
        L.bkvo_set_num_threads.argtypes = [i32]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _dirs(dirs):
    d = _c(dirs, np.uint8)
    if d.ndim == 1:          # one flag per request (reading Q5: col_stride 0)
        return d, 1, 0
    return d, d.shape[1], 1


def _pool_geom(K):
    assert K.dtype == np.uint16 and K.ndim == 4 and K.strides[3] == 2
    sb, sh, ss = (s // 2 for s in K.strides[:3])
    nblk, H, bs, d = K.shape
    return sb, sh, ss, H, d, bs


def bf16_to_f64(bits):
    """Vectorised exact bf16 -> float64 (the bf16 pattern is the top half of a float32)."""
    b = np.asarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def slot_in_block(direction: int, t: int, bs: int) -> int:
    return lib().bkvo_slot_in_block(int(direction), int(t), int(bs))


def _fills(fills, num_entries, B):
    """General map: uint8 fills [B][M] + int32 num_entries [B]."""
    f = _c(fills, np.uint8)
    ne = _c(num_entries, np.int32)
    assert f.ndim == 2 and f.shape[0] == B and ne.shape == (B,)
    return f, f.shape[1], ne


def validate(block_tables, dirs, lens, num_blocks: int, bs: int, require_nonempty=True,
             fills=None, num_entries=None):
    """Return (code, info): 0 ok, 1 I4 range, 2 I1 slot collision, 3 I2 sharing.
    With ``fills``/``num_entries`` the map is a general one (bkvo_validate_f)."""
    bt = _c(block_tables, np.int32)
    d, rs, cs = _dirs(dirs)
    ln = _c(lens, np.int32)
    info = np.zeros(4, dtype=np.int64)
    if fills is not None:
        f, frs, ne = _fills(fills, num_entries, int(ln.shape[0]))
        rc = lib().bkvo_validate_f(int(ln.shape[0]), _ptr(bt), int(bt.shape[1]), _ptr(d), rs, cs,
                                   _ptr(f), frs, _ptr(ne), _ptr(ln), int(num_blocks), int(bs),
                                   int(bool(require_nonempty)), _ptr(info))
        return int(rc), tuple(int(x) for x in info)
    rc = lib().bkvo_validate(int(ln.shape[0]), _ptr(bt), int(bt.shape[1]), _ptr(d), rs, cs,
                             _ptr(ln), int(num_blocks), int(bs), int(bool(require_nonempty)),
                             _ptr(info))
    return int(rc), tuple(int(x) for x in info)


def new_pool(num_blocks: int, H: int, bs: int, d: int, fill: int = 0):
    """Host KV pool pair, uint16 bf16 bits, layout [block][head][slot][d]."""
    K = np.full((num_blocks, H, bs, d), fill, dtype=np.uint16)
    return K, K.copy()


def append(K, V, block_tables, dirs, before, cu_new, k_new, v_new, fills=None, num_entries=None):
    """In-place append into host pools; returns int64 slot_mapping [total_new]."""
    sb, sh, ss, H, d, bs = _pool_geom(K)
    assert V.shape == K.shape and V.strides == K.strides
    bt = _c(block_tables, np.int32)
    dd, rs, cs = _dirs(dirs)
    bf = _c(before, np.int32)
    cu = _c(cu_new, np.int32)
    kn = _c(k_new, np.uint16).reshape(-1, H, d)
    vn = _c(v_new, np.uint16).reshape(-1, H, d)
    assert kn.shape[0] == cu[-1]
    sm = np.zeros(int(cu[-1]), dtype=np.int64)
    if fills is not None:
        f, frs, _ = _fills(fills, num_entries, int(bf.shape[0]))
        lib().bkvo_append_f(_ptr(K), _ptr(V), sb, sh, ss, H, d, bs, int(bf.shape[0]), _ptr(bt),
                            int(bt.shape[1]), _ptr(dd), rs, cs, _ptr(f), frs, _ptr(bf), _ptr(cu),
                            _ptr(kn), _ptr(vn), _ptr(sm))
        return sm
    lib().bkvo_append(_ptr(K), _ptr(V), sb, sh, ss, H, d, bs, int(bf.shape[0]), _ptr(bt),
                      int(bt.shape[1]), _ptr(dd), rs, cs, _ptr(bf), _ptr(cu), _ptr(kn), _ptr(vn),
                      _ptr(sm))
    return sm


def gather(K, V, block_tables, dirs, r: int, L: int, fills=None, num_entries=None):
    """Dense logical-order (K_r, V_r), uint16 [L][H][d]."""
    sb, sh, ss, H, d, bs = _pool_geom(K)
    bt = _c(block_tables, np.int32)
    dd, rs, cs = _dirs(dirs)
    ko = np.zeros((L, H, d), dtype=np.uint16)
    vo = np.zeros((L, H, d), dtype=np.uint16)
    if fills is not None:
        f, frs, _ = _fills(fills, num_entries, int(bt.shape[0]))
        lib().bkvo_gather_f(_ptr(K), _ptr(V), sb, sh, ss, H, d, bs, _ptr(bt), int(bt.shape[1]),
                            _ptr(dd), rs, cs, _ptr(f), frs, int(r), int(L), _ptr(ko), _ptr(vo))
        return ko, vo
    lib().bkvo_gather(_ptr(K), _ptr(V), sb, sh, ss, H, d, bs, _ptr(bt), int(bt.shape[1]),
                      _ptr(dd), rs, cs, int(r), int(L), _ptr(ko), _ptr(vo))
    return ko, vo


def attention(K, V, block_tables, dirs, lens, q, scale: float, r_range=None, fills=None,
              num_entries=None):
    """fp64 decode attention, out float64 [B][Hq][d] (rows outside r_range stay 0)."""
    sb, sh, ss, H, d, bs = _pool_geom(K)
    bt = _c(block_tables, np.int32)
    dd, rs, cs = _dirs(dirs)
    ln = _c(lens, np.int32)
    qq = _c(q, np.uint16)
    B, Hq, dq = qq.shape
    assert dq == d and Hq % H == 0
    out = np.zeros((B, Hq, d), dtype=np.float64)
    r0, r1 = (0, B) if r_range is None else r_range
    if fills is not None:
        f, frs, _ = _fills(fills, num_entries, B)
        lib().bkvo_attention_f(_ptr(K), _ptr(V), sb, sh, ss, H, d, bs, _ptr(bt), int(bt.shape[1]),
                               _ptr(dd), rs, cs, _ptr(f), frs, _ptr(ln), int(r0), int(r1), _ptr(qq),
                               int(Hq), float(scale), _ptr(out))
        return out
    lib().bkvo_attention(_ptr(K), _ptr(V), sb, sh, ss, H, d, bs, _ptr(bt), int(bt.shape[1]),
                         _ptr(dd), rs, cs, _ptr(ln), int(r0), int(r1), _ptr(qq), int(Hq),
                         float(scale), _ptr(out))
    return out


def prefill_attention(K, V, block_tables, dirs, lens, cu_q, q, scale: float, fills=None,
                      num_entries=None):
    """fp64 causal attention of each request's LAST n = cu_q[r+1]-cu_q[r] tokens over its
    paged context (mixed prefill + decode).  q uint16 [total][Hq][d];
    returns float64 [total][Hq][d]."""
    sb, sh, ss, H, d, bs = _pool_geom(K)
    bt = _c(block_tables, np.int32)
    dd, rs, cs = _dirs(dirs)
    ln = _c(lens, np.int32)
    cu = _c(cu_q, np.int32)
    qq = _c(q, np.uint16)
    T, Hq, dq = qq.shape
    B = int(ln.shape[0])
    assert dq == d and Hq % H == 0 and cu.shape == (B + 1,) and cu[-1] == T
    out = np.zeros((T, Hq, d), dtype=np.float64)
    f, frs = None, 0
    if fills is not None:
        f, frs, _ = _fills(fills, num_entries, B)
    lib().bkvo_prefill_attention(_ptr(K), _ptr(V), sb, sh, ss, H, d, bs, _ptr(bt), int(bt.shape[1]),
                                 _ptr(dd), rs, cs, _ptr(f), frs, B, _ptr(ln), _ptr(cu), _ptr(qq),
                                 int(Hq), float(scale), _ptr(out))
    return out


def checkpoint(K, V, slot_ids):
    """Rows of the given physical slots -> (k, v) uint16 [n][H][d] (lazy checkpoint)."""
    sb, sh, ss, H, d, bs = _pool_geom(K)
    sl = _c(slot_ids, np.int64)
    ko = np.zeros((sl.shape[0], H, d), np.uint16)
    vo = np.zeros((sl.shape[0], H, d), np.uint16)
    lib().bkvo_checkpoint(_ptr(K), _ptr(V), sb, sh, ss, H, d, bs, _ptr(sl), int(sl.shape[0]), _ptr(ko), _ptr(vo))
    return ko, vo


def restore(K, V, slot_ids, k_in, v_in):
    """In-place scatter of checkpointed rows back into their slots (swap-in)."""
    sb, sh, ss, H, d, bs = _pool_geom(K)
    sl = _c(slot_ids, np.int64)
    lib().bkvo_restore(_ptr(K), _ptr(V), sb, sh, ss, H, d, bs, _ptr(sl), int(sl.shape[0]),
                       _ptr(_c(k_in, np.uint16)), _ptr(_c(v_in, np.uint16)))


def overwritten_peers(block_tables, dirs, live_lens, before, n_new, num_blocks, bs, cap=1 << 16):
    """Live peer tokens an append would overwrite: list of (request, token, slot id)."""
    bt = _c(block_tables, np.int32)
    d, rs, cs = _dirs(dirs)
    ll, bf, nn = _c(live_lens, np.int32), _c(before, np.int32), _c(n_new, np.int32)
    vr = np.zeros(cap, np.int32)
    vt = np.zeros(cap, np.int64)
    vs = np.zeros(cap, np.int64)
    k = lib().bkvo_overwritten_peers(int(ll.shape[0]), _ptr(bt), int(bt.shape[1]), _ptr(d), rs, cs, _ptr(ll),
                                     _ptr(bf), _ptr(nn), int(num_blocks), int(bs), _ptr(vr), _ptr(vt), _ptr(vs), cap)
    k = min(k, cap)
    return [(int(vr[i]), int(vt[i]), int(vs[i])) for i in range(k)]


def num_threads() -> int:
    return int(lib().bkvo_num_threads())


def set_num_threads(n: int) -> None:
    lib().bkvo_set_num_threads(int(n))
