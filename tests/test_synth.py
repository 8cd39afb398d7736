"""Input-generator checks (host only): determinism, numpy/torch bit-equality,
length statistics vs Table "Workload statistics"."""
import numpy as np
import torch

from synth import CONFIGS, make_case, hash_bf16_np, hash_bf16_torch, key32, dense_kv_np, dense_kv_torch
from synth.workload import _lognormal, _MOMENTS, draw_lengths


def test_hash_numpy_torch_bit_identical():
    idx = np.arange(0, 200000, 7, dtype=np.int64)
    for base in (key32(1, 2, 3), key32(0), key32(2 ** 32 - 1, 5)):
        for sl in (0, 3):
            a = hash_bf16_np(base, idx, sl)
            b = hash_bf16_torch(base, torch.from_numpy(idx), sl).view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(a, b)
    k1, v1 = dense_kv_np(5, 2, 7, 33, [1, 3], 64, 4)
    k2, v2 = dense_kv_torch(5, 2, 7, 33, [1, 3], 64, 4, "cpu")
    assert np.array_equal(k1, k2.view(torch.int16).numpy().view(np.uint16))
    assert np.array_equal(v1, v2.view(torch.int16).numpy().view(np.uint16))


def test_hash_value_distribution():
    x = hash_bf16_np(key32(9), np.arange(400000))
    f = (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    assert abs(f.mean()) < 0.01 and 1.1 < f.std() < 1.2 and np.abs(f).max() <= 4.0


def test_lognormal_moments_match_table():
    rng = np.random.default_rng(0)
    for name, (pm, ps, om, os_) in _MOMENTS.items():
        p = _lognormal(rng, pm, ps, 400000)
        o = _lognormal(rng, om, os_, 400000)
        assert abs(p.mean() / pm - 1) < 0.03 and abs(p.std() / ps - 1) < 0.08, name
        assert abs(o.mean() / om - 1) < 0.03 and abs(o.std() / os_ - 1) < 0.08, name


def test_be_lengths_and_mix():
    rng = np.random.default_rng(1)
    sh = CONFIGS["llama70b"]
    L, is_be = draw_lengths(sh, rng)
    assert is_be.sum() == sh.batch // 2
    # BE: prompt U[512,1024] + U{1..output<=128}
    assert L[is_be].min() >= 513 and L[is_be].max() <= 1024 + 128
    assert 700 < L[is_be].mean() < 950
    assert L.min() >= 1 and L.max() <= sh.max_ctx


def test_layout_determinism_and_sharing():
    a = make_case("llama70b", 3)
    b = make_case("llama70b", 3)
    assert np.array_equal(a.layout.block_tables, b.layout.block_tables)
    assert np.array_equal(a.layout.lens, b.layout.lens)
    assert a.layout.n_shared > 0.5 * min((~a.layout.is_be).sum(), a.layout.is_be.sum())
    # SPEC S:230-style sizing: 20 tokens at bs 16 -> 2 entries (16 + 4)
    c = make_case("tiny", 0, lens=[20], is_be=[False])
    assert (c.layout.block_tables[0] >= 0).sum() == 2
