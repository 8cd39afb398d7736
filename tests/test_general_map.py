"""CPU pins of the general block map (include/bkv.h bkv_block_map).

FindBlock/FindPreemptBlock let ANY block-table entry be
partly filled; the general map carries per-entry fill counts.  Pins:
  * hand-derived golden slot map of a P:711/P:717/P:720 scenario and its
    a3/B8-style collision,
  * reduction: a general map with every non-last entry full is the dense map
    (slot map, gather and attention identical),
  * identity: gather after append returns the dense per-request arrays,
  * brute force: fp64 attention on the dense arrays (torch SDPA, float64),
  * the C ABI's host validator agrees with the oracle's on mutated maps.
No GPU needed (the libbkv host validator is plain host code).
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from synth import CONFIGS, make_case, build_general_layout
from synth.values import BF16_NAN
from tests._cases import dense_case, ragged, default_scale

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _fixture():
    with open(os.path.join(GOLD, "p717_general_map.json")) as f:
        fx = json.load(f)
    reqs = fx["requests"]
    B, M = len(reqs), max(len(r["block_table"]) for r in reqs)
    bt = np.full((B, M), -1, np.int32)
    fills = np.zeros((B, M), np.uint8)
    dirs = np.zeros((B, M), np.uint8)
    for i, r in enumerate(reqs):
        n = len(r["block_table"])
        bt[i, :n] = r["block_table"]
        fills[i, :n] = r["fills"]
        dirs[i, :n] = r["dir"]
    lens = np.array([r["len"] for r in reqs], np.int32)
    nent = np.array([len(r["block_table"]) for r in reqs], np.int32)
    return fx, bt, dirs, fills, nent, lens


def oracle_general_pool(case, ks, vs, n_heads, fill=BF16_NAN, lens=None):
    """Host pool holding tokens [0, lens[r]) of every request of a general-map case."""
    sh, lay = case.shape, case.layout
    lens = lay.lens if lens is None else lens
    K, V = oracle.new_pool(lay.num_blocks, n_heads, sh.block_size, sh.head_dim, fill)
    before = np.zeros(lay.batch, np.int32)
    kn, vn, cu = ragged(ks, vs, lens, before)
    sm = oracle.append(K, V, lay.block_tables, lay.dirs, before, cu, kn, vn,
                       fills=lay.fills, num_entries=lay.num_entries)
    return K, V, sm


def test_p717_general_slot_mapping_golden():
    fx, bt, dirs, fills, nent, lens = _fixture()
    bs = fx["block_size"]
    assert oracle.validate(bt, dirs, lens, fx["num_blocks"], bs, fills=fills, num_entries=nent)[0] == 0
    H, d = 1, 8
    K, V = oracle.new_pool(fx["num_blocks"], H, bs, d, 0)
    B = len(lens)
    rows = np.arange(1, int(lens.sum()) + 1, dtype=np.uint16)
    kn = np.repeat(rows[:, None, None], d, axis=2).astype(np.uint16)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    sm = oracle.append(K, V, bt, dirs, np.zeros(B, np.int32), cu, kn, kn, fills=fills, num_entries=nent)
    for i, r in enumerate(fx["requests"]):
        assert sm[cu[i]:cu[i + 1]].tolist() == fx["expected_slot_mapping"][r["name"]], r["name"]
    # every appended row sits exactly at its slot id, no other slot written
    flat = K.reshape(-1, d)[:, 0]
    assert sorted(np.flatnonzero(flat).tolist()) == sorted(sm.tolist())
    assert (flat[sm] == rows).all()


def test_p717_general_collision_rule():
    fx, bt, dirs, fills, nent, lens = _fixture()
    c = [r["name"] for r in fx["requests"]].index("C")
    lens2, fills2 = lens.copy(), fills.copy()
    lens2[c] = fx["collision"]["C_len"]
    fills2[c, 0] = fx["collision"]["C_len"]
    rc, info = oracle.validate(bt, dirs, lens2, fx["num_blocks"], fx["block_size"], fills=fills2, num_entries=nent)
    assert rc == 2 and list(info) == fx["collision"]["expected_info"]
    lens2[c] -= 1
    fills2[c, 0] -= 1
    assert oracle.validate(bt, dirs, lens2, fx["num_blocks"], fx["block_size"], fills=fills2, num_entries=nent)[0] == 0


def _dense_as_general(lay):
    nb = lay.nblocks().astype(np.int32)
    fills = np.zeros(lay.block_tables.shape, np.uint8)
    for r in range(lay.batch):
        for e in range(nb[r]):
            fills[r, e] = min(lay.block_size, int(lay.lens[r]) - e * lay.block_size)
    return fills, nb


@pytest.mark.parametrize("cfg,seed", [("tiny", 0), ("tiny_gqa", 1), ("opt13b", 2)])
def test_full_entries_reduce_to_dense_map(cfg, seed):
    case = make_case(cfg, seed)
    sh, lay = case.shape, case.layout
    heads = [0, 1] if cfg == "opt13b" else None
    ks, vs, q = dense_case(case, kv_heads=heads, q_heads=heads)
    H = len(heads) if heads else sh.num_kv_heads
    fills, nb = _dense_as_general(lay)
    B = lay.batch
    kn, vn, cu = ragged(ks, vs, lay.lens, np.zeros(B, np.int32))
    K1, V1 = oracle.new_pool(lay.num_blocks, H, sh.block_size, sh.head_dim, BF16_NAN)
    K2, V2 = K1.copy(), V1.copy()
    s1 = oracle.append(K1, V1, lay.block_tables, lay.dirs, np.zeros(B, np.int32), cu, kn, vn)
    s2 = oracle.append(K2, V2, lay.block_tables, lay.dirs, np.zeros(B, np.int32), cu, kn, vn,
                       fills=fills, num_entries=nb)
    assert np.array_equal(s1, s2) and np.array_equal(K1, K2) and np.array_equal(V1, V2)
    assert oracle.validate(lay.block_tables, lay.dirs, lay.lens, lay.num_blocks, sh.block_size,
                           fills=fills, num_entries=nb)[0] == 0
    if cfg != "opt13b":
        sc = default_scale(sh.head_dim)
        a1 = oracle.attention(K1, V1, lay.block_tables, lay.dirs, lay.lens, q, sc)
        a2 = oracle.attention(K1, V1, lay.block_tables, lay.dirs, lay.lens, q, sc, fills=fills, num_entries=nb)
        assert np.array_equal(a1, a2)


@pytest.mark.parametrize("cfg,seed,share", [("tiny", 0, 0.6), ("tiny", 3, 1.0), ("tiny_gqa", 1, 0.8),
                                            ("opt13b", 2, 0.6)])
def test_general_gather_after_append_is_identity(cfg, seed, share):
    case = make_case(cfg, seed, general=True, share_prob=share)
    sh, lay = case.shape, case.layout
    assert lay.general and (lay.fills[:, 0] > 0).all()
    assert oracle.validate(lay.block_tables, lay.dirs, lay.lens, lay.num_blocks, sh.block_size,
                           fills=lay.fills, num_entries=lay.num_entries)[0] == 0
    # a general map has partly filled NON-LAST entries (the point of f3)
    nonlast_partial = sum(int((lay.fills[r, :lay.num_entries[r] - 1] < sh.block_size).sum())
                          for r in range(lay.batch))
    assert nonlast_partial > 0
    heads = [3] if cfg == "opt13b" else None
    ks, vs, _ = dense_case(case, kv_heads=heads, q_heads=heads)
    H = 1 if heads else sh.num_kv_heads
    K, V, sm = oracle_general_pool(case, ks, vs, H)
    assert len(set(sm.tolist())) == sm.size   # every token on its own slot
    for r in range(lay.batch):
        kg, vg = oracle.gather(K, V, lay.block_tables, lay.dirs, r, int(lay.lens[r]),
                               fills=lay.fills, num_entries=lay.num_entries)
        assert np.array_equal(kg, ks[r]) and np.array_equal(vg, vs[r])


def _sdpa_f64(q, k, v, scale, g):
    qf = oracle.bf16_to_f64(q)[:, None, :]
    kf = np.repeat(oracle.bf16_to_f64(k), g, axis=1).transpose(1, 0, 2)
    vf = np.repeat(oracle.bf16_to_f64(v), g, axis=1).transpose(1, 0, 2)
    o = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(qf), torch.from_numpy(kf), torch.from_numpy(vf), scale=scale)
    return o[:, 0, :].numpy()


@pytest.mark.parametrize("cfg,seed,qs", [("tiny", 4, 0), ("tiny_gqa", 5, 3)])
def test_general_attention_matches_sdpa_f64(cfg, seed, qs):
    case = make_case(cfg, seed, general=True, q_scale_log2=qs)
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    K, V, _ = oracle_general_pool(case, ks, vs, sh.num_kv_heads)
    sc = default_scale(sh.head_dim)
    out = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, sc,
                           fills=lay.fills, num_entries=lay.num_entries)
    for r in range(lay.batch):
        ref = _sdpa_f64(q[r], ks[r], vs[r], sc, sh.group)
        assert np.abs(out[r] - ref).max() < 1e-12


def _mutations(lay, rng):
    """(name, block_tables, fills, num_entries, lens) variants that break one invariant."""
    B = lay.batch
    r = int(rng.integers(B))
    f = lay.fills.copy(); f[r, 0] = 0
    yield "fill0", lay.block_tables, f, lay.num_entries, lay.lens
    f = lay.fills.copy(); f[r, 0] = lay.block_size + 1
    yield "fill_big", lay.block_tables, f, lay.num_entries, lay.lens
    ln = lay.lens.copy(); ln[r] += 1
    yield "len_sum", lay.block_tables, lay.fills, lay.num_entries, ln
    ne = lay.num_entries.copy(); ne[r] = lay.block_tables.shape[1] + 1
    yield "nent", lay.block_tables, lay.fills, ne, lay.lens
    # two requests of the same class on one block (I2), or an overlap (I1)
    a, b = 0, 1
    bt = lay.block_tables.copy(); bt[b, 0] = bt[a, 0]
    yield "share", bt, lay.fills, lay.num_entries, lay.lens


def test_host_validator_agrees_with_oracle():
    import paper_2504_09590_b200 as bkv   # host-only entry point of libbkv (no GPU used)
    rng = np.random.default_rng(0)
    for seed in range(12):
        case = make_case("tiny", seed, general=True, share_prob=0.9)
        lay = case.layout
        ok, _ = bkv.validate_block_map_host(lay.block_tables, lay.dirs, lay.lens, lay.num_blocks, 16,
                                            lay.fills, lay.num_entries)
        assert ok
        for name, bt, f, ne, ln in _mutations(lay, rng):
            rc, oi = oracle.validate(bt, lay.dirs, ln, lay.num_blocks, 16, fills=f, num_entries=ne)
            ok, info = bkv.validate_block_map_host(bt, lay.dirs, ln, lay.num_blocks, 16, f, ne)
            assert rc != 0 and not ok and info[0] == rc, (name, rc, info)


def test_general_layout_generator_statistics():
    """Every generated general map is valid, sums to the lengths, and shares blocks."""
    for cfg in ("opt13b", "llama70b"):
        case = make_case(cfg, 0, general=True)
        lay = case.layout
        assert (lay.fills.astype(np.int64).sum(1) == lay.lens).all()
        assert lay.n_shared > 0
        assert oracle.validate(lay.block_tables, lay.dirs, lay.lens, lay.num_blocks, lay.block_size,
                               fills=lay.fills, num_entries=lay.num_entries)[0] == 0
