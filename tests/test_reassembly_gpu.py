"""Fused reassembly: bkv_decode_multi_out + bkv_peer_barrier.

On one GPU the "peers" are extra local buffers: the same code path stores each
output row into every pointer it is given (on a multi-GPU box those pointers
are peers' symmetric-memory buffers reached over NVLink).  Checked: every peer
copy is bit-identical to the local output (single- and multi-split requests,
attention-only and fused-step modes), the TP head-slice layout reassembles the
global head-major output exactly like the all-gather would, and the peer
barrier completes (world 1), honours a pre-signalled peer, and times out
instead of hanging when a peer never arrives.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2504_09590_b200 as bkv
from synth import make_case
from dataclasses import replace

from tests._cases import dense_case, default_scale, oracle_pool
from tests.test_fused_step import _prefilled, _step_rows
from tests.test_gpu_parity import DEV, check_close, gpu_map, gpu_pool_from_dense, t_u16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,min_split", [("tiny_gqa", None), ("tiny_gqa", "1"), ("tiny", "1"), ("tiny", None)])
def test_multi_out_copies_are_bitwise_local(cfg, min_split, monkeypatch):
    if min_split:
        monkeypatch.setenv("BKV_MIN_SPLIT", min_split)      # force split-K + merge for every request
        monkeypatch.setenv("BKV_UNITS_PER_WARP", "64")
    case = make_case(cfg, 31)
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    K, V, _ = oracle_pool(case, ks, vs, sh.num_kv_heads)
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, default_scale(sh.head_dim))
    pool, _ = gpu_pool_from_dense(case, ks, vs, sh.num_kv_heads)
    bt, dirs, lens = gpu_map(lay)
    out = torch.full((lay.batch, sh.num_q_heads, sh.head_dim), 3.0, dtype=torch.bfloat16, device=DEV)
    peers = [torch.full_like(out, -1.0) for _ in range(3)]
    bkv.decode_multi_out(pool, bt, dirs, lens, t_u16(q), out, peers)
    torch.cuda.synchronize()
    check_close(out, ref, cfg)
    for pb in peers:
        assert torch.equal(pb.view(torch.int16), out.view(torch.int16))


def test_multi_out_fused_step_and_tp_slices():
    """Two 'ranks' of a TP2 split of tiny_gqa each write their head slice into both
    global head-major buffers; both buffers end up equal to the oracle's full output."""
    case = make_case("tiny_gqa", 32)
    sh, lay = case.shape, case.layout
    B, d, tp = lay.batch, sh.head_dim, 2
    g_bufs = [torch.zeros((sh.num_q_heads, B, d), dtype=torch.bfloat16, device=DEV) for _ in range(tp)]
    ks_all, vs_all, q_all = dense_case(case)
    K, V, _ = oracle_pool(case, ks_all, vs_all, sh.num_kv_heads)
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q_all, default_scale(d))
    hq_loc, hkv_loc = sh.num_q_heads // tp, sh.num_kv_heads // tp
    bt, dirs, lens = gpu_map(lay)
    for rank in range(tp):
        kvh = list(range(rank * hkv_loc, (rank + 1) * hkv_loc))
        qh = list(range(rank * hq_loc, (rank + 1) * hq_loc))
        ks, vs, q = dense_case(case, kv_heads=kvh, q_heads=qh)
        # pool holds tokens [0, L-1); the fused step appends token L-1
        sub = replace(case, shape=replace(sh, num_q_heads=hq_loc, num_kv_heads=hkv_loc))
        K0, V0 = _prefilled(sub, ks, vs, (lay.lens - 1).astype(np.int32))
        pool = bkv.KVPool(t_u16(K0), t_u16(V0))
        kr, vr = _step_rows(ks, vs, lay.lens, hkv_loc, d)
        local = g_bufs[rank][rank * hq_loc:(rank + 1) * hq_loc]            # my slice, head-major
        peers = [gb[rank * hq_loc:(rank + 1) * hq_loc].data_ptr() for k, gb in enumerate(g_bufs) if k != rank]
        bkv.decode_multi_out(pool, bt, dirs, lens, t_u16(q), local.permute(1, 0, 2), peers,
                             k_new=t_u16(kr), v_new=t_u16(vr))
    torch.cuda.synchronize()
    assert torch.equal(g_bufs[0].view(torch.int16), g_bufs[1].view(torch.int16))
    check_close(g_bufs[0].permute(1, 0, 2), ref, "tp2 slices")


def test_peer_barrier_world1_prearrived_and_timeout():
    pads = torch.zeros(2, dtype=torch.int32, device=DEV)
    counter = torch.zeros(1, dtype=torch.int32, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    for _ in range(3):                                   # world 1: signal self, wait self
        bkv.peer_barrier([pads.data_ptr()], 0, counter, err)
    torch.cuda.synchronize()
    assert counter.item() == 3 and err.item() == 0 and pads[0].item() == 3
    # world 2, rank 0: the peer's flag in my pad is already ahead -> no wait
    mine = torch.zeros(2, dtype=torch.int32, device=DEV)
    peer = torch.zeros(2, dtype=torch.int32, device=DEV)
    mine[1] = 10
    c2 = torch.zeros(1, dtype=torch.int32, device=DEV)
    bkv.peer_barrier([mine.data_ptr(), peer.data_ptr()], 0, c2, err)
    torch.cuda.synchronize()
    assert err.item() == 0 and peer[0].item() == 1 and mine[0].item() == 1
    # a peer that never arrives: bounded wait, error flag, no hang
    mine2 = torch.zeros(2, dtype=torch.int32, device=DEV)
    c3 = torch.zeros(1, dtype=torch.int32, device=DEV)
    bkv.peer_barrier([mine2.data_ptr(), peer.data_ptr()], 0, c3, err, timeout_ns=2_000_000)
    torch.cuda.synchronize()
    assert err.item() == 1
