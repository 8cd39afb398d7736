"""CPU pins of the mixed prefill + decode attention oracle.

oracle.prefill_attention: request r's LAST n_r tokens are queries, query i sits
at logical position L - n + i and attends causally.
Pins: n = 1 reduces to the (separately pinned) decode oracle bit for bit;
float64 torch SDPA with an explicit bottom-right causal mask on the dense
per-request arrays (brute force, no paging); n = L is plain causal
self-attention (SDPA is_causal).  Dense and general maps.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import make_case, q_rows_np
from tests._cases import dense_case, oracle_pool, ragged, default_scale
from tests.test_general_map import oracle_general_pool


def query_counts(lens, rng, decode_frac=0.5, full=False):
    """Mixed batch: some requests decode (n = 1), the others prefill a random suffix."""
    lens = np.asarray(lens)
    if full:
        return lens.astype(np.int32)
    n = np.where(rng.random(lens.shape[0]) < decode_frac, 1,
                 np.maximum(1, (rng.random(lens.shape[0]) * lens).astype(np.int64)))
    return np.minimum(n, lens).astype(np.int32)


def queries(q_tok, n):
    """Stack per-request query rows [n_r][Hq][d] -> ([total][Hq][d], cu_q)."""
    cu = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
    return np.concatenate(q_tok) if len(q_tok) else None, cu


def make_q(case, n, Hq, rng=None, scale_log2=0, heads=None):
    """Seeded query rows (synth.q_rows_np) of every request's last n_r tokens."""
    sh = case.shape
    heads = list(range(sh.num_q_heads)) if heads is None else list(heads)
    rows = [q_rows_np(case.seed, case.layer, r, int(n[r]), heads, sh.head_dim, sh.num_q_heads, scale_log2)
            for r in range(case.layout.batch)]
    return queries(rows, n)


def pools(case, general):
    sh = case.shape
    ks, vs, _ = dense_case(case)
    if general:
        K, V, _ = oracle_general_pool(case, ks, vs, sh.num_kv_heads)
    else:
        K, V, _ = oracle_pool(case, ks, vs, sh.num_kv_heads)
    return ks, vs, K, V


def run_oracle(case, K, V, cu, q, general):
    lay = case.layout
    kw = dict(fills=lay.fills, num_entries=lay.num_entries) if general else {}
    return oracle.prefill_attention(K, V, lay.block_tables, lay.dirs, lay.lens, cu, q,
                                    default_scale(case.shape.head_dim), **kw)


@pytest.mark.parametrize("cfg,general", [("tiny", False), ("tiny_gqa", False), ("tiny_gqa", True)])
def test_single_query_is_decode_attention(cfg, general):
    case = make_case(cfg, 3, general=general)
    sh, lay = case.shape, case.layout
    ks, vs, K, V = pools(case, general)
    _, _, q = dense_case(case)
    cu = np.arange(lay.batch + 1, dtype=np.int32)
    out = run_oracle(case, K, V, cu, q, general)
    kw = dict(fills=lay.fills, num_entries=lay.num_entries) if general else {}
    dec = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, default_scale(sh.head_dim), **kw)
    assert np.array_equal(out, dec)


def _sdpa_causal_suffix(qr, k, v, scale, g):
    """float64 SDPA: queries are the last n of L tokens (bottom-right causal mask)."""
    n, L = qr.shape[0], k.shape[0]
    qf = torch.from_numpy(oracle.bf16_to_f64(qr)).permute(1, 0, 2)           # [Hq][n][d]
    kf = torch.from_numpy(np.repeat(oracle.bf16_to_f64(k), g, axis=1)).permute(1, 0, 2)
    vf = torch.from_numpy(np.repeat(oracle.bf16_to_f64(v), g, axis=1)).permute(1, 0, 2)
    pos = torch.arange(L - n, L)[:, None]
    mask = torch.arange(L)[None, :] <= pos
    o = torch.nn.functional.scaled_dot_product_attention(qf, kf, vf, attn_mask=mask, scale=scale)
    return o.permute(1, 0, 2).numpy()


@pytest.mark.parametrize("cfg,seed,general,full", [("tiny", 0, False, False), ("tiny", 1, True, False),
                                                   ("tiny_gqa", 2, False, False), ("tiny_gqa", 3, True, False),
                                                   ("tiny", 4, False, True), ("tiny_gqa", 5, True, True)])
def test_prefill_matches_sdpa_f64(cfg, seed, general, full):
    case = make_case(cfg, seed, general=general)
    sh, lay = case.shape, case.layout
    rng = np.random.default_rng(seed)
    n = query_counts(lay.lens, rng, full=full)
    ks, vs, K, V = pools(case, general)
    q, cu = make_q(case, n, sh.num_q_heads, rng, scale_log2=1)
    out = run_oracle(case, K, V, cu, q, general)
    sc = default_scale(sh.head_dim)
    for r in range(lay.batch):
        ref = _sdpa_causal_suffix(q[cu[r]:cu[r + 1]], ks[r], vs[r], sc, sh.group)
        assert np.abs(out[cu[r]:cu[r + 1]] - ref).max() < 1e-12, r
