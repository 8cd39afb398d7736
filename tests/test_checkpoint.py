"""Lazy checkpointing.

CPU: the oracle's checkpoint/restore and overwritten-peer detection are pinned
to the paper's a3/B8 example and to a flat-array replay.
GPU: bkv_kv_checkpoint / bkv_kv_restore match the oracle bit for bit.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from synth import build_layout
from synth.values import BF16_NAN

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _a3b8(bs):
    """RT request B (forward) and BE request a (reversed) sharing B's last block."""
    c = [c for c in json.load(open(os.path.join(GOLD, "a3_b8_collision.json")))["cases"]
         if c["bs"] == bs and c["expect_code"] == 2][0]
    M = max(len(c["B_bt"]), len(c["a_bt"]))
    bt = np.full((2, M), -1, np.int32)
    bt[0, :len(c["B_bt"])] = c["B_bt"]
    bt[1, :len(c["a_bt"])] = c["a_bt"]
    return c, bt, np.array([0, 1], np.uint8)


@pytest.mark.parametrize("bs", [12, 4])
def test_a3_b8_lazy_checkpoint_oracle(bs):
    """B holds 8 tokens, a holds 4; appending B8 must checkpoint exactly a3,
    overwrite it, and a later restore brings a3 back bitwise."""
    c, bt, dirs = _a3b8(bs)
    H, d = 2, 8
    K, V = oracle.new_pool(c["num_blocks"], H, bs, d, fill=0)
    rng = np.random.default_rng(0)
    dense_B = rng.integers(1, 60000, (9, H, d)).astype(np.uint16)
    dense_a = rng.integers(1, 60000, (4, H, d)).astype(np.uint16)
    # resident state before the step: B tokens 0..7, a tokens 0..3 (fills 8 + 4 = 12 / bs slots used)
    oracle.append(K, V, bt[:1], dirs[:1], np.zeros(1, np.int32), np.array([0, 8], np.int32), dense_B[:8], dense_B[:8])
    oracle.append(K, V, bt[1:], dirs[1:], np.zeros(1, np.int32), np.array([0, 4], np.int32), dense_a, dense_a)
    # the step appends B8: which live peer token does it overwrite?
    victims = oracle.overwritten_peers(bt, dirs, live_lens=[8, 4], before=[8, 4], n_new=[1, 0],
                                       num_blocks=c["num_blocks"], bs=bs)
    assert [(r, t) for r, t, _ in victims] == [(1, 3)]            # exactly a3
    sid = victims[0][2]
    assert sid == c["B_bt"][-1] * bs + c["collision_slot"]
    ck, cv = oracle.checkpoint(K, V, [sid])
    assert np.array_equal(ck[0], dense_a[3]) and np.array_equal(cv[0], dense_a[3])
    sm = oracle.append(K, V, bt[:1], dirs[:1], np.array([8], np.int32), np.array([0, 1], np.int32),
                       dense_B[8:9], dense_B[8:9])
    assert sm.tolist() == [sid]
    kB, _ = oracle.gather(K, V, bt[:1], dirs[:1], 0, 9)
    assert np.array_equal(kB, dense_B)
    # B finishes and releases; a is scheduled again: swap a3 back in
    oracle.restore(K, V, [sid], ck, cv)
    ka, va = oracle.gather(K, V, bt[1:], dirs[1:], 0, 4)
    assert np.array_equal(ka, dense_a) and np.array_equal(va, dense_a)


def test_overwritten_peers_flat_array_replay():
    """Random shared-tail layouts, RT tails grown past their share: every reported
    victim is exactly a live BE token on the RT token's slot (flat slot-owner replay)."""
    rng = np.random.default_rng(3)
    bs = 16
    lens = rng.integers(1, 120, 16)
    is_be = np.arange(16) % 2 == 1
    lay = build_layout(lens, is_be, bs, rng, spare_blocks=2)
    # grow every RT request by up to 6 tokens inside its last block (overlap allowed now)
    grow = np.where(~is_be, np.minimum(6, (-lens) % bs), 0).astype(np.int32)
    victims = oracle.overwritten_peers(lay.block_tables, lay.dirs, lay.lens, lay.lens, grow,
                                       lay.num_blocks, bs)
    owner = {}
    for r in range(16):
        for t in range(lens[r]):
            e, j = divmod(t, bs)
            slot = bs - 1 - j if is_be[r] else j
            owner[int(lay.block_tables[r, e]) * bs + slot] = (r, t)
    expect = []
    for r in range(16):
        for j in range(grow[r]):
            t = lens[r] + j
            e, jj = divmod(t, bs)
            sid = int(lay.block_tables[r, e]) * bs + jj
            if sid in owner and owner[sid][0] != r:
                expect.append((owner[sid][0], owner[sid][1], sid))
    assert victims == expect


@pytest.mark.gpu
def test_gpu_checkpoint_restore_bitwise():
    import paper_2504_09590_b200 as bkv
    rng = np.random.default_rng(5)
    for H, d, bs in ((2, 128, 16), (4, 64, 32)):
        nblk = 64
        K = rng.integers(0, 65535, (nblk, H, bs, d)).astype(np.uint16)
        V = rng.integers(0, 65535, (nblk, H, bs, d)).astype(np.uint16)

        def g(a):
            return torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16)

        def u(t):
            return t.view(torch.int16).cpu().numpy().view(np.uint16)

        pool = bkv.KVPool(g(K), g(V))
        sids = rng.choice(nblk * bs, 300, replace=False).astype(np.int64)
        ck, cv = oracle.checkpoint(K, V, sids)
        gk, gv = bkv.kv_checkpoint(pool, torch.from_numpy(sids).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(u(gk), ck) and np.array_equal(u(gv), cv)
        # overwrite, then restore: the pool is back to its original bytes
        pool.k[:] = 0
        pool.v.view(torch.int16).fill_(np.int16(np.uint16(BF16_NAN).view(np.int16)))
        bkv.kv_restore(pool, torch.from_numpy(sids).cuda(), gk, gv)
        torch.cuda.synchronize()
        Ko = np.zeros_like(K)
        Vo = np.full_like(V, BF16_NAN)
        oracle.restore(Ko, Vo, sids, ck, cv)
        assert np.array_equal(u(pool.k), Ko) and np.array_equal(u(pool.v), Vo)


def _grown_rt_case(seed, bs=16, H=2, d=128, B=16):
    """Shared-tail layout whose RT requests then grow INTO their BE peer's slots."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 120, B)
    is_be = np.arange(B) % 2 == 1
    lay = build_layout(lens, is_be, bs, rng, spare_blocks=2)
    grow = np.where(~is_be, np.minimum(6, (-lens) % bs), 0).astype(np.int32)
    K = rng.integers(0, 65535, (lay.num_blocks, H, bs, d)).astype(np.uint16)
    V = rng.integers(0, 65535, (lay.num_blocks, H, bs, d)).astype(np.uint16)
    n = int(grow.sum())
    kn = rng.integers(0, 65535, (n, H, d)).astype(np.uint16)
    vn = rng.integers(0, 65535, (n, H, d)).astype(np.uint16)
    cu = np.concatenate([[0], np.cumsum(grow)]).astype(np.int32)
    return lay, grow, K, V, kn, vn, cu


def test_fused_checkpoint_reference_is_checkpoint_then_append():
    """CPU side of the fused call's definition: the victims the oracle reports are exactly
    the slots whose old bytes differ after the append; checkpointing them first keeps them."""
    lay, grow, K, V, kn, vn, cu = _grown_rt_case(7, d=8)
    before = lay.lens.astype(np.int32)
    victims = oracle.overwritten_peers(lay.block_tables, lay.dirs, lay.lens, before, grow, lay.num_blocks, 16)
    assert len(victims) > 0
    sids = [s for _, _, s in victims]
    ck, cv = oracle.checkpoint(K, V, sids)
    K2, V2 = K.copy(), V.copy()
    sm = oracle.append(K2, V2, lay.block_tables, lay.dirs, before, cu, kn, vn)
    assert set(sids) <= set(sm.tolist())
    kk, vv = oracle.checkpoint(K, V, sm)          # old contents of every written slot
    assert np.array_equal(ck, kk[[sm.tolist().index(s) for s in sids]])


@pytest.mark.gpu
@pytest.mark.parametrize("seed,d", [(7, 128), (8, 64)])
def test_gpu_append_checkpoint_fused_bitwise(seed, d):
    """bkv_kv_append_checkpoint == oracle checkpoint(victims) + oracle append, bit for bit."""
    import paper_2504_09590_b200 as bkv
    lay, grow, K, V, kn, vn, cu = _grown_rt_case(seed, d=d)
    H = K.shape[1]
    before = lay.lens.astype(np.int32)
    victims = oracle.overwritten_peers(lay.block_tables, lay.dirs, lay.lens, before, grow, lay.num_blocks, 16)
    sids = [s for _, _, s in victims]
    assert len(sids) > 0
    ck, cv = oracle.checkpoint(K, V, sids)
    Ko, Vo = K.copy(), V.copy()
    sm = oracle.append(Ko, Vo, lay.block_tables, lay.dirs, before, cu, kn, vn)
    evict = np.array([sids.index(s) if s in sids else -1 for s in sm.tolist()], np.int32)

    def g(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16).copy()).cuda().view(torch.bfloat16)

    def u(t):
        return t.view(torch.int16).cpu().numpy().view(np.uint16)

    pool = bkv.KVPool(g(K), g(V))
    n_ck = len(sids) + 3                       # spare rows must stay untouched
    gk = torch.full((n_ck, H, d), 7.0, dtype=torch.bfloat16, device="cuda")
    gv = torch.full((n_ck, H, d), 7.0, dtype=torch.bfloat16, device="cuda")
    gsm = torch.zeros(len(sm), dtype=torch.int64, device="cuda")
    bkv.kv_append_checkpoint(pool, torch.from_numpy(lay.block_tables).cuda(), torch.from_numpy(lay.dirs).cuda(),
                             torch.from_numpy(before).cuda(), torch.from_numpy(cu).cuda(), g(kn), g(vn),
                             torch.from_numpy(evict).cuda(), gk, gv, slot_mapping=gsm)
    torch.cuda.synchronize()
    assert np.array_equal(u(pool.k), Ko) and np.array_equal(u(pool.v), Vo)
    assert np.array_equal(gsm.cpu().numpy(), sm)
    assert np.array_equal(u(gk)[:len(sids)], ck) and np.array_equal(u(gv)[:len(sids)], cv)
    assert (gk[len(sids):].float() == 7.0).all() and (gv[len(sids):].float() == 7.0).all()
    # swap-in after the RT request finished: the peer's tokens come back bitwise
    bkv.kv_restore(pool, torch.tensor(sids, dtype=torch.int64, device="cuda"), gk[:len(sids)], gv[:len(sids)])
    torch.cuda.synchronize()
    oracle.restore(Ko, Vo, sids, ck, cv)
    assert np.array_equal(u(pool.k), Ko)


@pytest.mark.gpu
def test_gpu_append_checkpoint_into_pinned_host_memory():
    """The checkpoint rows may land directly in pinned host memory (UVA: the pinned
    pointer is valid on the device) -- the D2H checkpoint of P:726 with no staging copy."""
    import paper_2504_09590_b200 as bkv
    H, d = 2, 64
    lay, grow, K, V, kn, vn, cu = _grown_rt_case(9, d=d, H=H)
    before = lay.lens.astype(np.int32)
    victims = oracle.overwritten_peers(lay.block_tables, lay.dirs, lay.lens, before, grow, lay.num_blocks, 16)
    sids = [s for _, _, s in victims]
    ck, cv = oracle.checkpoint(K, V, sids)
    Ko, Vo = K.copy(), V.copy()
    sm = oracle.append(Ko, Vo, lay.block_tables, lay.dirs, before, cu, kn, vn)
    evict = np.array([sids.index(s) if s in sids else -1 for s in sm.tolist()], np.int32)

    def g(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16).copy()).cuda().view(torch.bfloat16)

    hk = torch.zeros((len(sids), H, d), dtype=torch.bfloat16).pin_memory()
    hv = torch.zeros((len(sids), H, d), dtype=torch.bfloat16).pin_memory()
    pool = bkv.KVPool(g(K), g(V))
    bkv.kv_append_checkpoint(pool, torch.from_numpy(lay.block_tables).cuda(), torch.from_numpy(lay.dirs).cuda(),
                             torch.from_numpy(before).cuda(), torch.from_numpy(cu).cuda(), g(kn), g(vn),
                             torch.from_numpy(evict).cuda(), hk, hv)
    torch.cuda.synchronize()
    assert np.array_equal(hk.view(torch.int16).numpy().view(np.uint16), ck)
    assert np.array_equal(hv.view(torch.int16).numpy().view(np.uint16), cv)
    assert np.array_equal(pool.k.view(torch.int16).cpu().numpy().view(np.uint16), Ko)
