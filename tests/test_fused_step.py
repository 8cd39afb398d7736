"""GPU parity of the fused decode step (include/bkv.h bkv_decode_step).

bkv_decode_step(pool, map, seq_lens, k_new, v_new, q) is DEFINED as
kv_append(before = seq_lens - 1, one token per request) followed by the
attention over seq_lens.  Checked three ways on the same seeded inputs:
  * the pool after the call equals the ORACLE's append bit for bit
    (§5.1, P:711 slot rule),
  * the output is within the north_star tolerance of the oracle's attention,
  * the output is bitwise the unfused two-call path's.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2504_09590_b200 as bkv
from synth import make_case, build_layout
from synth.values import BF16_NAN
from synth.workload import Case, Shape
from tests._cases import dense_case, ragged, default_scale
from tests.test_gpu_parity import DEV, check_close, gpu_map, t_u16, u16

pytestmark = pytest.mark.gpu


def _prefilled(case, ks, vs, lens_before, per_request=False):
    """Host pool holding tokens [0, lens_before[r]) of every request (oracle append)."""
    sh, lay = case.shape, case.layout
    B = lay.batch
    K, V = oracle.new_pool(lay.num_blocks, sh.num_kv_heads, sh.block_size, sh.head_dim, BF16_NAN)
    kn, vn, cu = ragged(ks, vs, lens_before, np.zeros(B, np.int32))
    dirs = lay.dirs_per_request if per_request else lay.dirs
    oracle.append(K, V, lay.block_tables, dirs, np.zeros(B, np.int32), cu, kn, vn)
    return K, V


def _step_rows(ks, vs, lens, H, d):
    """Rows of token L-1 per request as [B][H][d] (zeros where L == 0)."""
    B = len(lens)
    kr = np.zeros((B, H, d), np.uint16)
    vr = np.zeros((B, H, d), np.uint16)
    for r in range(B):
        if lens[r] > 0:
            kr[r] = ks[r][lens[r] - 1]
            vr[r] = vs[r][lens[r] - 1]
    return kr, vr


def _check_step(case, per_request=False, pdl=False, tag=""):
    sh, lay = case.shape, case.layout
    B, H, d = lay.batch, sh.num_kv_heads, sh.head_dim
    ks, vs, q = dense_case(case)
    lens = lay.lens.astype(np.int32)
    before = np.maximum(lens - 1, 0).astype(np.int32)
    K0, V0 = _prefilled(case, ks, vs, before, per_request)
    # oracle: append token L-1 (requests with L == 0 get nothing), then attention
    Ko, Vo = K0.copy(), V0.copy()
    has = (lens > 0).astype(np.int32)
    cu = np.concatenate([[0], np.cumsum(has)]).astype(np.int32)
    kd, vd, _ = ragged(ks, vs, lens, before)
    dirs_h = lay.dirs_per_request if per_request else lay.dirs
    oracle.append(Ko, Vo, lay.block_tables, dirs_h, before, cu, kd, vd)
    ref = oracle.attention(Ko, Vo, lay.block_tables, dirs_h, lens, q, default_scale(d))

    bt, dirs, lens_t = gpu_map(lay, per_request)
    kr, vr = _step_rows(ks, vs, lens, H, d)
    # fused
    pool = bkv.KVPool(t_u16(K0.copy()), t_u16(V0.copy()))
    o = bkv.decode_step(pool, bt, dirs, lens_t, t_u16(kr), t_u16(vr), t_u16(q), pdl=pdl)
    # unfused: kv_append + attention on a second copy
    pool2 = bkv.KVPool(t_u16(K0.copy()), t_u16(V0.copy()))
    bkv.kv_append(pool2, bt, dirs, torch.from_numpy(before).to(DEV), torch.from_numpy(cu).to(DEV),
                  t_u16(kd), t_u16(vd))
    o2 = bkv.paged_decode_attention(pool2, bt, dirs, lens_t, t_u16(q))
    torch.cuda.synchronize()
    assert np.array_equal(u16(pool.k), Ko) and np.array_equal(u16(pool.v), Vo), tag
    check_close(o, ref, tag)
    assert torch.equal(o.view(torch.int16), o2.view(torch.int16)), tag
    return o


@pytest.mark.parametrize("cfg,seed", [("tiny", 0), ("tiny", 1), ("tiny_gqa", 2), ("tiny_gqa", 3)])
def test_fused_step_small(cfg, seed):
    _check_step(make_case(cfg, seed), tag=cfg)


@pytest.mark.parametrize("hq,hkv,d,bs", [(16, 1, 128, 16), (12, 1, 64, 32), (6, 2, 64, 16),
                                         (3, 3, 64, 32), (5, 5, 128, 32), (32, 2, 128, 16),
                                         (8, 1, 128, 16)])
def test_fused_step_geometries(hq, hkv, d, bs):
    sh = Shape("g", hq, hkv, d, bs, 20, 0.5, "uniform", 900, 1, 1, uniform_max=900)
    _check_step(make_case(sh, hq * 7 + d + bs), tag=f"{hq}/{hkv}/{d}/{bs}")


@pytest.mark.parametrize("direction", [0, 1])
def test_fused_step_edge_lengths(direction):
    """New token on every position class: first/last slot of a block, the first
    and second 16-slot half of a bs=32 block, a context of one token."""
    lens = [1, 2, 15, 16, 17, 31, 32, 33, 47, 48, 63, 64, 65, 255, 256, 257, 1000, 2049]
    for (hq, hkv, d, bs, seed) in ((8, 2, 128, 16, 4), (4, 4, 64, 32, 5), (16, 2, 128, 32, 6)):
        sh = Shape("edge", hq, hkv, d, bs, len(lens), 0.5, "uniform", 4096, 1, 1)
        case = make_case(sh, seed, lens=lens, is_be=[bool(direction)] * len(lens))
        _check_step(case, tag=f"dir{direction} {hq}/{hkv}/{d}/{bs}")


def test_fused_step_shared_tails_per_request_dirs_and_pdl():
    case = make_case("tiny_gqa", 9)
    _check_step(case, per_request=True, tag="per-request")
    _check_step(make_case("tiny", 10), pdl=True, tag="pdl")


def test_fused_step_empty_request_untouched():
    sh = Shape("z", 8, 1, 128, 16, 4, 0.5, "uniform", 64, 1, 1)
    lay = build_layout([0, 5, 0, 40], [False, True, True, False], 16, np.random.default_rng(0), spare_blocks=2)
    o = _check_step(Case(sh, lay, 3), tag="empty")
    assert (u16(o)[[0, 2]] == 0).all()


def test_fused_steps_in_sequence_grow_context():
    """Several decode iterations back to back (lengths +1 each step, PDL on):
    after each step the pool is the oracle's append of every token so far."""
    sh = Shape("seq", 16, 2, 128, 16, 12, 0.5, "uniform", 300, 1, 1, uniform_max=300)
    n_steps = 5
    lens = np.random.default_rng(17).integers(n_steps + 1, 300, size=12)
    case = make_case(sh, 17, lens=lens)
    lay = case.layout
    B, H, d = lay.batch, sh.num_kv_heads, sh.head_dim
    # the layout is built for the FINAL lengths; run steps L-n+1 .. L
    final = lay.lens.astype(np.int32)
    assert (final > n_steps).all()
    ks, vs, q = dense_case(case)
    start = final - n_steps
    K, V = _prefilled(case, ks, vs, start)
    pool = bkv.KVPool(t_u16(K.copy()), t_u16(V.copy()))
    bt, dirs, _ = gpu_map(lay)
    outs = []
    for s in range(1, n_steps + 1):
        cur = (start + s).astype(np.int32)
        kr, vr = _step_rows(ks, vs, cur, H, d)
        outs.append(bkv.decode_step(pool, bt, dirs, torch.from_numpy(cur).to(DEV), t_u16(kr), t_u16(vr),
                                    t_u16(q), pdl=True))
    torch.cuda.synchronize()
    Ko, Vo = _prefilled(case, ks, vs, final)
    # slots beyond start but never written stay NaN on both sides; live slots must match
    assert np.array_equal(u16(pool.k), Ko) and np.array_equal(u16(pool.v), Vo)
    ref = oracle.attention(Ko, Vo, lay.block_tables, lay.dirs, final, q, default_scale(d))
    check_close(outs[-1], ref, "last step")


def test_fused_step_argument_errors():
    pool = bkv.KVPool.empty(4, 2, 16, 64, DEV)
    bt = torch.zeros(1, 1, dtype=torch.int32, device=DEV)
    dirs = torch.zeros(1, dtype=torch.uint8, device=DEV)
    lens = torch.ones(1, dtype=torch.int32, device=DEV)
    q = torch.zeros(1, 2, 64, dtype=torch.bfloat16, device=DEV)
    kn = torch.zeros(1, 2, 64, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(bkv.BkvError, match="k_new/v_new"):
        bkv.decode_step(pool, bt, dirs, lens, kn[:, :1], kn[:, :1], q)
    with pytest.raises(bkv.BkvError, match="multiple"):
        bkv.decode_step(pool, bt, dirs, lens, kn, kn, torch.zeros(1, 3, 64, dtype=torch.bfloat16, device=DEV))
