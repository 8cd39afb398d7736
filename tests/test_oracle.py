"""Pins of the CPU oracle against the paper and against mathematics (-m "not gpu").

Each test says what it pins.  None of them re-types the oracle's formula:
expectations are hand-derived fixtures (tests/golden, with citations), closed
forms, invariants, or torch's float64 scaled_dot_product_attention on dense
(unpaged) arrays.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from synth import CONFIGS, make_case, build_layout, dense_kv_np
from synth.values import BF16_NAN
from tests._cases import dense_case, oracle_pool, ragged, default_scale

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ bf16 bits
def test_bf16_decode_exact():
    # IEEE: 0x3F80 = 1.0, 0xC000 = -2.0, 0x3EAB ~ 0.333984375, 0x0001 smallest subnormal
    assert oracle.lib().bkvo_bf16_to_f64(0x3F80) == 1.0
    assert oracle.lib().bkvo_bf16_to_f64(0xC000) == -2.0
    assert oracle.lib().bkvo_bf16_to_f64(0x3EAB) == 0.333984375
    assert oracle.lib().bkvo_bf16_to_f64(0x0001) == 2.0 ** -133
    assert np.isnan(oracle.lib().bkvo_bf16_to_f64(BF16_NAN))


# ------------------------------------------------------- slot map: P:711 fixture
def _fixture_layout(fx, per_request):
    reqs = fx["requests"]
    M = max(len(r["block_table"]) for r in reqs)
    bt = np.full((len(reqs), M), -1, np.int32)
    dirs2 = np.zeros((len(reqs), M), np.uint8)
    for i, r in enumerate(reqs):
        bt[i, :len(r["block_table"])] = r["block_table"]
        dirs2[i, :len(r["block_table"])] = r["dir"]
    dirs1 = np.array([r["dir"] for r in reqs], np.uint8)
    lens = np.array([r["len"] for r in reqs], np.int32)
    return bt, (dirs1 if per_request else dirs2), lens


@pytest.mark.parametrize("per_request", [False, True])
def test_p711_slot_mapping_golden(per_request):
    """Pins the slot map (reading Q3) to hand-derived slots."""
    fx = _load("p711_layout.json")
    bs, nblk = fx["block_size"], fx["num_blocks"]
    bt, dirs, lens = _fixture_layout(fx, per_request)
    assert oracle.validate(bt, dirs, lens, nblk, bs) == (0, (0, 0, 0, 0))
    H, d = 2, 8
    K, V = oracle.new_pool(nblk, H, bs, d, fill=0)
    total = int(lens.sum())
    # token payload encodes (request, t, head): every row is distinct
    k_new = (np.arange(total * H * d, dtype=np.int64) % 60000 + 1).astype(np.uint16).reshape(total, H, d)
    v_new = (k_new ^ 0x5555).astype(np.uint16)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    sm = oracle.append(K, V, bt, dirs, np.zeros(len(lens), np.int32), cu, k_new, v_new)
    for i, r in enumerate(fx["requests"]):
        assert sm[cu[i]:cu[i + 1]].tolist() == fx["expected_slot_mapping"][r["name"]], r["name"]
    # the rows landed exactly there, and nowhere else
    touched = np.zeros((nblk, bs), bool)
    for i in range(total):
        blk, slot = divmod(int(sm[i]), bs)
        assert np.array_equal(K[blk, :, slot, :], k_new[i]) and np.array_equal(V[blk, :, slot, :], v_new[i])
        touched[blk, slot] = True
    assert not K.transpose(0, 2, 1, 3)[~touched].any() and not V.transpose(0, 2, 1, 3)[~touched].any()


def test_p711_single_token_slots():
    # j-th token of an RT block at slot j, of a BE block at slot bs-1-j (Q3)
    for bs in (4, 12, 16, 32):
        for t in range(3 * bs):
            assert oracle.slot_in_block(0, t, bs) == t % bs
            assert oracle.slot_in_block(1, t, bs) == bs - 1 - t % bs


def test_decode_step_append_golden():
    """Decode step (1 new token per request, reading Q7) lands on the fixture's last slots."""
    fx = _load("p711_layout.json")
    bs, nblk = fx["block_size"], fx["num_blocks"]
    bt, dirs, lens = _fixture_layout(fx, False)
    K, V = oracle.new_pool(nblk, 1, bs, 4, fill=0)
    B = len(lens)
    kn = np.arange(1, B * 4 + 1, dtype=np.uint16).reshape(B, 1, 4)
    sm = oracle.append(K, V, bt, dirs, lens - 1, np.arange(B + 1, dtype=np.int32), kn, kn)
    assert sm.tolist() == [fx["expected_slot_mapping"][r["name"]][-1] for r in fx["requests"]]


# --------------------------------------------------- a3/B8 collision rule
def test_a3_b8_collision_rule():
    """Pins validator I1 to the paper's worked example."""
    fx = _load("a3_b8_collision.json")
    for c in fx["cases"]:
        M = max(len(c["B_bt"]), len(c["a_bt"]))
        bt = np.full((2, M), -1, np.int32)
        bt[0, :len(c["B_bt"])] = c["B_bt"]
        bt[1, :len(c["a_bt"])] = c["a_bt"]
        dirs = np.array([0, 1], np.uint8)
        lens = np.array([c["B_len"], c["a_len"]], np.int32)
        code, info = oracle.validate(bt, dirs, lens, c["num_blocks"], c["bs"])
        assert code == c["expect_code"], c
        if code == 2:
            assert list(info) == c["expect_info"]
            assert oracle.slot_in_block(0, 8, c["bs"]) == c["collision_slot"]
            assert oracle.slot_in_block(1, 3, c["bs"]) == c["collision_slot"]


def test_validator_rejects_bad_layouts():
    bs = 16
    bt = np.array([[0, 1], [2, -1]], np.int32)
    dirs = np.array([[0, 0], [1, 0]], np.uint8)
    lens = np.array([20, 5], np.int32)
    assert oracle.validate(bt, dirs, lens, 3, bs)[0] == 0
    # I4: block id out of range
    assert oracle.validate(np.array([[0, 3], [2, -1]], np.int32), dirs, lens, 3, bs)[0] == 1
    # I4: direction flag not in {0, 1}
    assert oracle.validate(bt, np.array([[0, 2], [1, 0]], np.uint8), lens, 3, bs)[0] == 1
    # I4: length beyond the block table / empty context for attention (Q8)
    assert oracle.validate(bt, dirs, np.array([33, 5], np.int32), 3, bs)[0] == 1
    assert oracle.validate(bt, dirs, np.array([20, 0], np.int32), 3, bs)[0] == 1
    assert oracle.validate(bt, dirs, np.array([20, 0], np.int32), 3, bs, require_nonempty=False)[0] == 0
    # I2: two RT requests on one block ("one RT request and one BE request")
    assert oracle.validate(np.array([[0, 1], [1, -1]], np.int32), np.array([[0, 0], [0, 0]], np.uint8),
                           np.array([20, 2], np.int32), 3, bs)[0] == 3
    # RT + BE sharing block 1 with 4 + 12 = 16 slots is fine; 4 + 13 collides (I1)
    bt2 = np.array([[0, 1], [1, -1]], np.int32)
    d2 = np.array([[0, 0], [1, 1]], np.uint8)
    assert oracle.validate(bt2, d2, np.array([20, 12], np.int32), 3, bs)[0] == 0
    assert oracle.validate(bt2, d2, np.array([20, 13], np.int32), 3, bs)[0] == 2


# ---------------------------------------------- append/gather identity (P1)
@pytest.mark.parametrize("cfg,seed", [("tiny", 0), ("tiny", 1), ("tiny_gqa", 2), ("opt13b", 3)])
def test_gather_after_append_is_identity(cfg, seed):
    """Appending dense tokens then gathering returns them bitwise (random block ids,
    both directions, shared RT/BE tails) -- pins append, gather and the slot map together."""
    case = make_case(cfg, seed)
    sh, lay = case.shape, case.layout
    if cfg == "opt13b":   # keep the CPU test small: 4 heads of the real geometry
        heads = [0, 17, 33, 39]
    else:
        heads = list(range(sh.num_kv_heads))
    assert oracle.validate(lay.block_tables, lay.dirs, lay.lens, lay.num_blocks, sh.block_size)[0] == 0
    ks, vs, _ = dense_case(case, kv_heads=heads, q_heads=[0])
    K, V, sm = oracle_pool(case, ks, vs, len(heads))
    assert lay.n_shared > 0 or cfg == "opt13b"
    for r in range(lay.batch):
        k, v = oracle.gather(K, V, lay.block_tables, lay.dirs, r, int(lay.lens[r]))
        assert np.array_equal(k, ks[r]) and np.array_equal(v, vs[r])
    # every non-resident slot still holds the poison pattern
    owned = np.zeros((lay.num_blocks, sh.block_size), bool)
    for s in sm:
        owned[s // sh.block_size, s % sh.block_size] = True
    assert len(set(sm.tolist())) == len(sm)
    assert (K.transpose(0, 2, 1, 3)[~owned] == BF16_NAN).all()
    assert (V.transpose(0, 2, 1, 3)[~owned] == BF16_NAN).all()


def test_multistep_append_stress():
    """SPEC S:286-style flat-array stress: many steps of ragged prefill chunks and
    single-token decodes for mixed RT/BE requests sharing tails; after every step
    each request's resident prefix reads back exactly (every appended token reachable
    exactly once, P:711 + BASELINE north_star)."""
    rng = np.random.default_rng(7)
    bs, H, d = 16, 2, 8
    B = 24
    final = rng.integers(1, 200, B)
    is_be = rng.random(B) < 0.5
    lay = build_layout(final, is_be, bs, rng, spare_blocks=5)
    assert oracle.validate(lay.block_tables, lay.dirs, lay.lens, lay.num_blocks, bs)[0] == 0
    dense = [np.stack([np.full((H, d), (r << 10 | t) & 0xFFFF, np.uint16) for t in range(final[r])])
             for r in range(B)]
    K, V = oracle.new_pool(lay.num_blocks, H, bs, d, fill=BF16_NAN)
    cur = np.zeros(B, np.int64)
    n_tokens = 0
    while (cur < final).any():
        step_new = np.where(rng.random(B) < 0.3, rng.integers(1, 40, B), 1)
        step_new = np.minimum(step_new, final - cur)
        after = cur + step_new
        kn, vn, cu = ragged(dense, dense, after, cur)
        sm = oracle.append(K, V, lay.block_tables, lay.dirs, cur.astype(np.int32), cu, kn, vn)
        assert len(set(sm.tolist())) == len(sm)
        n_tokens += len(sm)
        cur = after
        for r in range(B):
            k, _ = oracle.gather(K, V, lay.block_tables, lay.dirs, r, int(cur[r]))
            assert np.array_equal(k, dense[r][:cur[r]])
    assert n_tokens == final.sum()


# -------------------------------------------- attention: library routine (P2)
def _sdpa_f64(q, k, v, scale, g):
    """torch float64 SDPA on dense arrays; GQA via repeat_interleave (reading Q9)."""
    qt = torch.from_numpy(oracle.bf16_to_f64(q))[:, None, :]          # [Hq, 1, d]
    kt = torch.from_numpy(oracle.bf16_to_f64(k)).permute(1, 0, 2)      # [H, L, d]
    vt = torch.from_numpy(oracle.bf16_to_f64(v)).permute(1, 0, 2)
    kt = kt.repeat_interleave(g, dim=0)
    vt = vt.repeat_interleave(g, dim=0)
    return torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, scale=scale)[:, 0, :].numpy()


@pytest.mark.parametrize("cfg,seed,qs", [("tiny", 0, 0), ("tiny", 5, 3), ("tiny_gqa", 1, 0), ("tiny_gqa", 4, 4)])
def test_attention_matches_torch_sdpa_f64(cfg, seed, qs):
    case = make_case(cfg, seed, q_scale_log2=qs)
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    K, V, _ = oracle_pool(case, ks, vs, sh.num_kv_heads)
    scale = default_scale(sh.head_dim)
    out = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, scale)
    for r in range(lay.batch):
        ref = _sdpa_f64(q[r], ks[r], vs[r], scale, sh.group)
        np.testing.assert_allclose(out[r], ref, rtol=0, atol=1e-12)


# -------------------------------------------------- attention: closed forms (P3)
def _one_request_pool(k, v, bs, direction, seed=0):
    L, H, d = k.shape
    rng = np.random.default_rng(seed)
    lay = build_layout([L], [bool(direction)], bs, rng, spare_blocks=2)
    K, V = oracle.new_pool(lay.num_blocks, H, bs, d, fill=BF16_NAN)
    oracle.append(K, V, lay.block_tables, lay.dirs, np.zeros(1, np.int32),
                  np.array([0, L], np.int32), k, v)
    return K, V, lay


@pytest.mark.parametrize("direction", [0, 1])
def test_closed_forms(direction):
    bs, H, d = 16, 2, 32
    k, v = dense_kv_np(3, 0, 0, 37, [0, 1], d, 2)
    q = dense_kv_np(4, 0, 0, 1, [0, 1, 2, 3], d, 4)[0]              # [1][4][d]: 4 q heads, g = 2
    # (i) L = 1: out = v_0 exactly
    K, V, lay = _one_request_pool(k[:1], v[:1], bs, direction)
    out = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, 0.125)
    for h in range(4):
        assert np.array_equal(out[0, h], oracle.bf16_to_f64(v[0, h // 2]))
    # (ii) scale = 0: uniform weights, out = mean of V over tokens
    K, V, lay = _one_request_pool(k, v, bs, direction)
    out = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, 0.0)
    for h in range(4):
        np.testing.assert_allclose(out[0, h], oracle.bf16_to_f64(v[:, h // 2]).mean(0), atol=1e-13)
    # (iii) all keys equal: out = mean of V at any scale
    ke = np.repeat(k[:1], 37, axis=0)
    K, V, lay = _one_request_pool(ke, v, bs, direction)
    out = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, 0.7)
    for h in range(4):
        np.testing.assert_allclose(out[0, h], oracle.bf16_to_f64(v[:, h // 2]).mean(0), atol=1e-13)
    # (iv) all value rows equal: out = that row
    ve = np.repeat(v[5:6], 37, axis=0)
    K, V, lay = _one_request_pool(k, ve, bs, direction)
    out = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, 0.3)
    for h in range(4):
        np.testing.assert_allclose(out[0, h], oracle.bf16_to_f64(ve[0, h // 2]), atol=1e-14)
    # (v) one dominant key: out -> its value row
    kd = np.zeros_like(k)
    kd[11] = q[0, ::2]       # token 11 aligned with q heads 0 and 2 (kv heads 0, 1 via g = 2)
    K, V, lay = _one_request_pool(kd, v, bs, direction)
    out = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, 50.0)
    np.testing.assert_allclose(out[0, 0], oracle.bf16_to_f64(v[11, 0]), atol=1e-9)
    np.testing.assert_allclose(out[0, 2], oracle.bf16_to_f64(v[11, 1]), atol=1e-9)


def test_empty_context_gives_zeros():
    # reading Q8: L = 0 is invalid for attention; if met, the output is 0, never NaN
    K, V = oracle.new_pool(2, 1, 16, 8, fill=BF16_NAN)
    out = oracle.attention(K, V, np.array([[0]], np.int32), np.array([0], np.uint8),
                           np.array([0], np.int32), np.ones((1, 1, 8), np.uint16), 1.0)
    assert (out == 0).all()


# ------------------------------------------------ metamorphic invariants (P5)
def test_mirror_and_relabel_invariance():
    """Same logical tokens stored with the opposite direction, and with physical
    blocks relabelled, give bitwise-identical oracle outputs (attention is over the
    request's token set; paging only moves bytes -- SURVEY §8(c))."""
    case = make_case("tiny_gqa", 11)
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    K, V, _ = oracle_pool(case, ks, vs, sh.num_kv_heads)
    scale = default_scale(sh.head_dim)
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, scale)
    # mirror: flip every request's direction, no tail sharing (would collide otherwise)
    rng = np.random.default_rng(99)
    lay2 = build_layout(lay.lens, ~lay.is_be, sh.block_size, rng, share_tails=False, spare_blocks=7)
    K2, V2 = oracle.new_pool(lay2.num_blocks, sh.num_kv_heads, sh.block_size, sh.head_dim, fill=BF16_NAN)
    kn, vn, cu = ragged(ks, vs, lay.lens, np.zeros(lay.batch, np.int64))
    oracle.append(K2, V2, lay2.block_tables, lay2.dirs, np.zeros(lay.batch, np.int32), cu, kn, vn)
    out2 = oracle.attention(K2, V2, lay2.block_tables, lay2.dirs, lay2.lens, q, scale)
    assert np.array_equal(ref, out2)


def test_gqa_equals_mha_with_repeated_heads():
    """Reading Q9 (kv = h // g): a GQA batch equals MHA over kv heads repeated g times."""
    case = make_case("tiny_gqa", 6)
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    K, V, _ = oracle_pool(case, ks, vs, sh.num_kv_heads)
    scale = default_scale(sh.head_dim)
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, scale)
    Kr = np.repeat(K, sh.group, axis=1)
    Vr = np.repeat(V, sh.group, axis=1)
    out = oracle.attention(Kr, Vr, lay.block_tables, lay.dirs, lay.lens, q, scale)
    assert np.array_equal(ref, out)
