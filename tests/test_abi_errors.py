"""Argument errors of the C ABI are reported synchronously, before any launch or device
query (include/bkv.h "Conventions") -- checked here without a GPU by calling the raw
entry points with fake, never-dereferenced device addresses."""
import ctypes

import pytest

import paper_2504_09590_b200 as bkv
from paper_2504_09590_b200.bkv import _Map, _Pool

OK, INVALID, UNSUPPORTED = 0, 1, 2
FAKE = 0x10000            # 16-byte aligned, never touched: every case fails before use


def pool(d=128, bs=16, H=2, nblk=8):
    return _Pool(FAKE, FAKE, nblk, H, bs, d, H * bs * d, bs * d, d)


def bmap(B=4, fills=False):
    return _Map(FAKE, 8, FAKE, 8, 1, B, FAKE if fills else None, 8 if fills else 0, FAKE if fills else None)


def decode(p, m, Hq=2, q=FAKE, scale=0.1, max_len=64, flags=0, ws_bytes=1 << 30):
    L = bkv.lib()
    return L.bkv_paged_decode_attention_ex(ctypes.byref(p), ctypes.byref(m), FAKE, max_len, q, 256, 128, Hq,
                                           scale, FAKE, 256, 128, FAKE, ws_bytes, flags, None)


def err():
    return bkv.lib().bkv_last_error().decode()


def test_decode_argument_errors():
    assert decode(pool(d=96), bmap()) == UNSUPPORTED and "head_dim" in err()
    assert decode(pool(bs=8), bmap()) == UNSUPPORTED and "block_size" in err()
    assert decode(pool(), bmap(B=2049)) == UNSUPPORTED and "num_seqs" in err()
    assert decode(pool(H=129), bmap()) == UNSUPPORTED and "num_kv_heads" in err()
    assert decode(pool(), bmap(), Hq=3) == INVALID and "multiple" in err()
    assert decode(pool(H=1), bmap(), Hq=17) == UNSUPPORTED and "group" in err()
    assert decode(pool(), bmap(), q=FAKE + 2) == INVALID and "aligned" in err()
    assert decode(pool(), bmap(), scale=float("nan")) == INVALID and "scale" in err()
    assert decode(pool(), bmap(), max_len=8 * 16 + 1) == INVALID and "max_seq_len" in err()
    assert decode(pool(), bmap(), flags=8) == INVALID and "flags" in err()
    # BKV_FLAG_PEER_MULTICAST without exactly one peer output (the plain call has none)
    assert decode(pool(), bmap(), flags=4) == INVALID and "MULTICAST" in err()
    p = pool()
    p.k = None
    assert decode(p, bmap()) == INVALID
    m = bmap(fills=True)
    m.num_entries = None
    assert decode(pool(), m) == INVALID and "num_entries" in err()
    assert decode(pool(), bmap(B=0)) == OK          # empty batch: no-op


def test_append_and_prefill_argument_errors():
    L = bkv.lib()
    p, m = pool(), bmap()
    rc = L.bkv_kv_append(ctypes.byref(p), ctypes.byref(m), FAKE, FAKE, 4, None, FAKE, None, None)
    assert rc == INVALID and "NULL" in err()
    rc = L.bkv_kv_append(ctypes.byref(p), ctypes.byref(m), FAKE, FAKE, 4, FAKE + 8, FAKE, None, None)
    assert rc == INVALID and "aligned" in err()
    mg = _Map(FAKE, 20000, FAKE, 20000, 1, 4, FAKE, 20000, FAKE)
    rc = L.bkv_kv_append(ctypes.byref(p), ctypes.byref(mg), FAKE, FAKE, 4, FAKE, FAKE, None, None)
    assert rc == UNSUPPORTED and "bt_stride" in err()
    rc = L.bkv_kv_append_checkpoint(ctypes.byref(p), ctypes.byref(m), FAKE, FAKE, 4, FAKE, FAKE, None,
                                    None, FAKE, FAKE, None)
    assert rc == INVALID and "evict_rows" in err()
    rc = L.bkv_paged_prefill_attention(ctypes.byref(p), ctypes.byref(m), FAKE, FAKE, -1, FAKE, 256, 128, 2,
                                       0.1, FAKE, 256, 128, None)
    assert rc == INVALID and "max_q_len" in err()
    rc = L.bkv_paged_prefill_attention(ctypes.byref(p), ctypes.byref(m), FAKE, FAKE, 4, FAKE, 250, 128, 2,
                                       0.1, FAKE, 256, 128, None)
    assert rc == INVALID and "aligned" in err()


def test_reassembly_argument_errors():
    L = bkv.lib()
    p, m = pool(), bmap()
    peers = (ctypes.c_void_p * 9)(*([FAKE] * 9))
    rc = L.bkv_decode_multi_out(ctypes.byref(p), ctypes.byref(m), FAKE, 64, None, None, FAKE, 256, 128, 2,
                                0.1, FAKE, peers, 9, 256, 128, FAKE, 1 << 30, 0, None)
    assert rc == UNSUPPORTED and "n_peers" in err()
    rc = L.bkv_decode_multi_out(ctypes.byref(p), ctypes.byref(m), FAKE, 64, FAKE, None, FAKE, 256, 128, 2,
                                0.1, FAKE, peers, 1, 256, 128, FAKE, 1 << 30, 0, None)
    assert rc == INVALID and "k_new" in err()
    pads = (ctypes.c_void_p * 2)(FAKE, FAKE)
    assert L.bkv_peer_barrier(pads, 0, 0, FAKE, FAKE, 1000, None) == UNSUPPORTED
    assert L.bkv_peer_barrier(pads, 2, 2, FAKE, FAKE, 1000, None) == INVALID
    assert L.bkv_peer_barrier(pads, 2, 0, None, FAKE, 1000, None) == INVALID


def test_status_strings_cover_every_code():
    L = bkv.lib()
    names = [L.bkv_status_string(c).decode() for c in range(6)]
    assert names == ["BKV_OK", "BKV_ERR_INVALID_ARGUMENT", "BKV_ERR_UNSUPPORTED",
                     "BKV_ERR_WORKSPACE_TOO_SMALL", "BKV_ERR_LAYOUT", "BKV_ERR_CUDA"]
    assert L.bkv_version() == 300
