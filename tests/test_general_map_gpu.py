"""GPU parity of the general block map through the C ABI.

Same seeded inputs on both sides (synth.build_general_layout: FindBlock /
FindPreemptBlock stand-in); the oracle side is bkvo_*_f.
Append and slot map bit-exact; attention within the north_star tolerance;
the fused decode step bit-identical to append + attention.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2504_09590_b200 as bkv
from synth import make_case
from synth.values import BF16_NAN
from synth.workload import Shape
from tests._cases import dense_case, ragged, default_scale
from tests.test_general_map import oracle_general_pool
from tests.test_gpu_parity import DEV, check_close, t_u16, u16

pytestmark = pytest.mark.gpu


def gmap(lay):
    return (torch.from_numpy(lay.block_tables).to(DEV), torch.from_numpy(lay.dirs).to(DEV),
            torch.from_numpy(lay.lens.astype(np.int32)).to(DEV),
            torch.from_numpy(lay.fills).to(DEV), torch.from_numpy(lay.num_entries).to(DEV))


def gpu_general_pool(case, ks, vs, H, lens=None, fill=BF16_NAN):
    sh, lay = case.shape, case.layout
    lens = lay.lens if lens is None else lens
    pool = bkv.KVPool.empty(lay.num_blocks, H, sh.block_size, sh.head_dim, DEV)
    pool.k.view(torch.int16).fill_(np.int16(np.uint16(fill).view(np.int16)))
    pool.v.view(torch.int16).fill_(np.int16(np.uint16(fill).view(np.int16)))
    before = np.zeros(lay.batch, np.int32)
    kn, vn, cu = ragged(ks, vs, lens, before)
    bt, dirs, _, fills, nent = gmap(lay)
    sm = torch.zeros(kn.shape[0], dtype=torch.int64, device=DEV)
    bkv.kv_append(pool, bt, dirs, torch.from_numpy(before).to(DEV), torch.from_numpy(cu).to(DEV),
                  t_u16(kn), t_u16(vn), slot_mapping=sm, fills=fills, num_entries=nent)
    return pool, sm


@pytest.mark.parametrize("cfg,seed,share", [("tiny", 0, 0.6), ("tiny", 1, 1.0), ("tiny_gqa", 2, 0.8),
                                            ("llama70b", 3, 0.6)])
def test_general_append_bitwise(cfg, seed, share):
    case = make_case(cfg, seed, general=True, share_prob=share)
    sh = case.shape
    heads = [6] if cfg == "llama70b" else None
    ks, vs, _ = dense_case(case, kv_heads=heads, q_heads=[0])
    H = 1 if heads else sh.num_kv_heads
    Ko, Vo, smo = oracle_general_pool(case, ks, vs, H)
    pool, sm = gpu_general_pool(case, ks, vs, H)
    torch.cuda.synchronize()
    assert np.array_equal(u16(pool.k), Ko) and np.array_equal(u16(pool.v), Vo)
    assert np.array_equal(sm.cpu().numpy(), smo)


def test_general_ragged_append_on_prefilled_pool_bs32():
    """Prefill a prefix, then append the rest of each request as ragged chunks."""
    sh = Shape("g32", 4, 2, 128, 32, 24, 0.5, "uniform", 700, 1, 1, uniform_max=700)
    case = make_case(sh, 8, general=True, share_prob=0.9)
    lay = case.layout
    ks, vs, _ = dense_case(case)
    rng = np.random.default_rng(1)
    before = (lay.lens * rng.random(lay.batch)).astype(np.int32)
    Ko, Vo, _ = oracle_general_pool(case, ks, vs, 2, lens=before)
    pool = bkv.KVPool(t_u16(Ko.copy()), t_u16(Vo.copy()))
    kd, vd, cud = ragged(ks, vs, lay.lens, before)
    smo = oracle.append(Ko, Vo, lay.block_tables, lay.dirs, before, cud, kd, vd,
                        fills=lay.fills, num_entries=lay.num_entries)
    bt, dirs, _, fills, nent = gmap(lay)
    sm = torch.zeros(kd.shape[0], dtype=torch.int64, device=DEV)
    bkv.kv_append(pool, bt, dirs, torch.from_numpy(before).to(DEV), torch.from_numpy(cud).to(DEV),
                  t_u16(kd), t_u16(vd), slot_mapping=sm, fills=fills, num_entries=nent)
    torch.cuda.synchronize()
    assert np.array_equal(u16(pool.k), Ko) and np.array_equal(u16(pool.v), Vo)
    assert np.array_equal(sm.cpu().numpy(), smo)


@pytest.mark.parametrize("cfg,seed,qs,share", [("tiny", 0, 0, 0.6), ("tiny", 5, 3, 1.0),
                                               ("tiny_gqa", 2, 0, 0.8), ("tiny_gqa", 7, 4, 1.0)])
def test_general_attention_parity(cfg, seed, qs, share):
    case = make_case(cfg, seed, general=True, share_prob=share, q_scale_log2=qs)
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    K, V, _ = oracle_general_pool(case, ks, vs, sh.num_kv_heads)
    sc = default_scale(sh.head_dim)
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, sc,
                           fills=lay.fills, num_entries=lay.num_entries)
    pool, _ = gpu_general_pool(case, ks, vs, sh.num_kv_heads)
    bt, dirs, lens, fills, nent = gmap(lay)
    o = bkv.paged_decode_attention(pool, bt, dirs, lens, t_u16(q), sc, fills=fills, num_entries=nent)
    torch.cuda.synchronize()
    check_close(o, ref, cfg)
    # poison (P5(vi)): zero instead of NaN in every non-owned slot -> bitwise equal output
    pool0, _ = gpu_general_pool(case, ks, vs, sh.num_kv_heads, fill=0)
    o0 = bkv.paged_decode_attention(pool0, bt, dirs, lens, t_u16(q), sc, fills=fills, num_entries=nent)
    torch.cuda.synchronize()
    assert torch.equal(o.view(torch.int16), o0.view(torch.int16))


@pytest.mark.parametrize("hq,hkv,d,bs", [(8, 1, 128, 16), (5, 5, 128, 16), (6, 2, 64, 32)])
def test_general_attention_long_ragged(hq, hkv, d, bs):
    """Long requests (many splits) with partly filled entries everywhere."""
    sh = Shape("gl", hq, hkv, d, bs, 12, 0.5, "uniform", 3000, 1, 1, uniform_max=3000)
    case = make_case(sh, hq + bs, general=True, share_prob=1.0, q_scale_log2=2)
    lay = case.layout
    ks, vs, q = dense_case(case)
    K, V, _ = oracle_general_pool(case, ks, vs, hkv)
    sc = default_scale(d)
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, sc,
                           fills=lay.fills, num_entries=lay.num_entries)
    pool, _ = gpu_general_pool(case, ks, vs, hkv)
    bt, dirs, lens, fills, nent = gmap(lay)
    o = bkv.paged_decode_attention(pool, bt, dirs, lens, t_u16(q), sc, fills=fills, num_entries=nent)
    torch.cuda.synchronize()
    check_close(o, ref, str((hq, hkv, d, bs)))


@pytest.mark.parametrize("cfg,seed", [("tiny", 3), ("tiny_gqa", 4), ("llama70b", 5)])
def test_general_fused_decode_step(cfg, seed):
    """bkv_decode_step on a general map: token L-1 is the last token of the last entry."""
    case = make_case(cfg, seed, general=True, share_prob=0.8)
    sh, lay = case.shape, case.layout
    kv = [2] if cfg == "llama70b" else None
    qh = list(range(16, 24)) if cfg == "llama70b" else None
    ks, vs, q = dense_case(case, kv_heads=kv, q_heads=qh)
    H = 1 if kv else sh.num_kv_heads
    d, B = sh.head_dim, lay.batch
    lens = lay.lens.astype(np.int32)
    before = (lens - 1).astype(np.int32)
    K0, V0, _ = oracle_general_pool(case, ks, vs, H, lens=before)
    Ko, Vo = K0.copy(), V0.copy()
    kd, vd, cu = ragged(ks, vs, lens, before)
    oracle.append(Ko, Vo, lay.block_tables, lay.dirs, before, cu, kd, vd,
                  fills=lay.fills, num_entries=lay.num_entries)
    sc = default_scale(d)
    ref = oracle.attention(Ko, Vo, lay.block_tables, lay.dirs, lens, q, sc,
                           fills=lay.fills, num_entries=lay.num_entries)
    bt, dirs, lens_t, fills, nent = gmap(lay)
    pool = bkv.KVPool(t_u16(K0.copy()), t_u16(V0.copy()))
    o = bkv.decode_step(pool, bt, dirs, lens_t, t_u16(kd), t_u16(vd), t_u16(q), sc,
                        fills=fills, num_entries=nent)
    pool2 = bkv.KVPool(t_u16(K0.copy()), t_u16(V0.copy()))
    bkv.kv_append(pool2, bt, dirs, torch.from_numpy(before).to(DEV), torch.from_numpy(cu).to(DEV),
                  t_u16(kd), t_u16(vd), fills=fills, num_entries=nent)
    o2 = bkv.paged_decode_attention(pool2, bt, dirs, lens_t, t_u16(q), sc, fills=fills, num_entries=nent)
    torch.cuda.synchronize()
    assert np.array_equal(u16(pool.k), Ko) and np.array_equal(u16(pool.v), Vo)
    check_close(o, ref, cfg)
    assert torch.equal(o.view(torch.int16), o2.view(torch.int16))


def test_dense_map_as_general_is_bitwise_dense():
    """A general map whose non-last entries are full gives bitwise the dense-map output."""
    case = make_case("tiny_gqa", 11)
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    from tests.test_gpu_parity import gpu_pool_from_dense, gpu_map
    pool, _ = gpu_pool_from_dense(case, ks, vs, sh.num_kv_heads)
    bt, dirs, lens = gpu_map(lay)
    nb = lay.nblocks().astype(np.int32)
    fills = np.zeros(lay.block_tables.shape, np.uint8)
    for r in range(lay.batch):
        for e in range(nb[r]):
            fills[r, e] = min(sh.block_size, int(lay.lens[r]) - e * sh.block_size)
    o1 = bkv.paged_decode_attention(pool, bt, dirs, lens, t_u16(q))
    o2 = bkv.paged_decode_attention(pool, bt, dirs, lens, t_u16(q), fills=torch.from_numpy(fills).to(DEV),
                                    num_entries=torch.from_numpy(nb).to(DEV))
    torch.cuda.synchronize()
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))


@pytest.mark.parametrize("cfg,seed", [("tiny_gqa", 6), ("llama70b", 7)])
def test_general_fused_step_streamk(cfg, seed, monkeypatch):
    """The stream-K split plan (forced on) over general maps with the fused append:
    segments follow entry counts, the new token's entry is owned by exactly one range."""
    monkeypatch.setenv("BKV_STREAMK", "2")
    test_general_fused_decode_step(cfg, seed)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("streamk", ["0", "2"])
def test_general_fused_step_fuzz(seed, streamk, monkeypatch):
    """Seeded random geometries on FindBlock-style general maps through the fused decode
    step (pool bit-exact, output vs the oracle, equal to append + attention), both plans."""
    monkeypatch.setenv("BKV_STREAMK", streamk)
    rng = np.random.default_rng(2000 + seed)
    hkv = int(rng.choice([1, 2, 4]))
    g = int(rng.choice([1, 2, 4, 8]))
    d = int(rng.choice([64, 128]))
    bs = int(rng.choice([16, 32]))
    B = int(rng.integers(2, 40))
    sh = Shape(f"gfuzz{seed}", hkv * g, hkv, d, bs, B, 0.5, "uniform", 1200, 1, 1, uniform_max=1200)
    test_general_fused_decode_step(sh, seed)
